"""Precision plans for emulated mixed-precision MMA (reference: emulation.py).

A wide operand is split into 8- or 4-bit chunks (lower chunks unsigned, top
chunk signed); chunk products recombine with weights 2**(w*(i+j)) (Table IV,
PAPER.md:337-373). The plan is the *contract* (supported pairs, tile k, the
accumulation bound); on B200 the kernels execute every chunk product as an
int8 IMMA (16-bit -> u8 low + s8 high byte, 4-bit -> sign-extended s8, see
DESIGN.md), which is exact and gives identical results.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Tuple

from .errors import OverflowRiskError, UnsupportedPrecisionError

SPMM = "spmm"
SDDMM = "sddmm"

EMULATED = {
    SPMM: {(16, 16), (16, 8), (16, 4), (12, 4), (8, 4)},
    SDDMM: {(16, 16)},
}
NATIVE = {
    SPMM: {(8, 8), (4, 4)},
    SDDMM: {(8, 8), (4, 4)},
}

INT32_MIN = -(1 << 31)
INT32_MAX = (1 << 31) - 1


@dataclass(frozen=True)
class TileShape:
    """Native warp tile of the reference model: 8x8x16 (8-bit) or 8x8x32 (4-bit)."""

    m: int
    n: int
    k: int
    operand_width_lhs: int
    operand_width_rhs: int

    @property
    def elems_per_lane(self) -> int:
        return self.k // 4


INT8_TILE = TileShape(8, 8, 16, 8, 8)
INT4_TILE = TileShape(8, 8, 32, 4, 4)


def native_tile(width: int) -> TileShape:
    if width == 8:
        return INT8_TILE
    if width == 4:
        return INT4_TILE
    raise ValueError(f"no native tile for {width}-bit operands")


def supported_pairs(op_kind: str):
    return sorted(EMULATED[op_kind] | NATIVE[op_kind])


@dataclass(frozen=True)
class EmulationScheme:
    lhs_bits: int
    rhs_bits: int
    op_kind: str
    native_width: int
    lhs_chunks: int
    rhs_chunks: int
    lhs_signed: Tuple[bool, ...]
    rhs_signed: Tuple[bool, ...]

    @property
    def tile(self) -> TileShape:
        return native_tile(self.native_width)

    @property
    def native(self) -> bool:
        return self.lhs_chunks == 1 and self.rhs_chunks == 1

    def weight(self, lhs_chunk: int, rhs_chunk: int) -> int:
        return 1 << (self.native_width * (lhs_chunk + rhs_chunk))

    @property
    def weights(self) -> Tuple[int, ...]:
        return tuple(self.weight(i, j) for i in range(self.lhs_chunks)
                     for j in range(self.rhs_chunks))

    @property
    def device_chunk_products(self) -> int:
        """int8 IMMA products the B200 kernels issue per output (16-bit = 2 chunks)."""
        lc = 2 if self.lhs_bits >= 12 else 1
        rc = 2 if self.rhs_bits >= 12 else 1
        return lc * rc


def plan(lhs_bits: int, rhs_bits: int, op_kind: str = SPMM) -> EmulationScheme:
    """Chunking plan (emulation.py:67-85): w = 8 iff both widths divide by 8."""
    if op_kind not in (SPMM, SDDMM):
        raise ValueError(f"op_kind must be {SPMM!r} or {SDDMM!r}")
    pair = (lhs_bits, rhs_bits)
    if pair not in EMULATED[op_kind] and pair not in NATIVE[op_kind]:
        names = ["L%d-R%d" % p for p in supported_pairs(op_kind)]
        raise UnsupportedPrecisionError(
            f"L{lhs_bits}-R{rhs_bits} is not supported for {op_kind} (supported: {names})")
    w = 8 if lhs_bits % 8 == 0 and rhs_bits % 8 == 0 else 4
    lc, rc = lhs_bits // w, rhs_bits // w
    return EmulationScheme(lhs_bits, rhs_bits, op_kind, w, lc, rc,
                           tuple(i == lc - 1 for i in range(lc)),
                           tuple(j == rc - 1 for j in range(rc)))


def precision_name(lhs_bits: int, rhs_bits: int) -> str:
    return f"L{lhs_bits}-R{rhs_bits}"


def parse_precision(name: str) -> Tuple[int, int]:
    try:
        l, r = name.upper().split("-")
        return int(l.lstrip("L")), int(r.lstrip("R"))
    except Exception:
        raise ValueError(f"precision name must look like 'L8-R4', got {name!r}") from None


def check_accumulation_bound(k: int, chunk_width: int) -> None:
    """K * (2**w - 1)**2 must fit int32 (emulation.py:108-113)."""
    worst = (1 << chunk_width) - 1
    if k * worst * worst > INT32_MAX:
        raise OverflowRiskError(
            f"reduction size {k} risks int32 overflow for {chunk_width}-bit chunk products")
