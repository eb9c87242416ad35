"""SpMM and SDDMM entry points (reference: kernels.py) backed by libmcube (sm_100a).

Same names, signatures, validation and error behaviour as the reference:
`SpmmProblem` / `SddmmProblem` validate at construction (kernels.py:58-118),
`spmm` / `spmm_pipelined` / `sddmm` run the CUDA kernels through the C ABI
(include/mcube.h) and raise OverflowRiskError where the reference does.
Host (numpy) inputs give numpy outputs; CUDA torch inputs give CUDA tensors.
The optional Python epilogue is applied to the finished int32 output, exactly
like the reference (kernels.py:286-290, :428-430).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Union

import numpy as np

from . import _device as D
from . import _native as N
from . import emulation
from .emulation import EmulationScheme, check_accumulation_bound
from .errors import ShuffleStateError
from .qint import COL_MAJOR, ROW_MAJOR, PackedMatrix
from .sparse_format import BcrsMatrix, SrBcrsMatrix, bcrs_to_srbcrs

Epilogue = Callable[[object], object]


@dataclass(frozen=True)
class TilingConfig:
    """BS_n in {64, 128}; BS_m = V and BS_k = tile k are derived (kernels.py:40-55).

    On B200 the CTA shape is chosen by the kernel (64-column warp tiles, a
    4-stage cp.async ring); these fields are validated and kept for API parity.
    """

    bs_n: int = 64
    warps_per_block: int = 2
    pipeline: bool = False
    bs_m: Optional[int] = None
    bs_k: Optional[int] = None

    def __post_init__(self):
        if self.bs_n not in (64, 128):
            raise ValueError(f"BS_n must be 64 or 128, got {self.bs_n}")
        if self.warps_per_block < 1:
            raise ValueError("need at least one warp per block")


@dataclass(frozen=True, eq=False)
class SpmmProblem:
    lhs: SrBcrsMatrix
    rhs: PackedMatrix
    config: TilingConfig = field(default_factory=TilingConfig)
    epilogue: Optional[Epilogue] = None

    def __post_init__(self):
        if self.rhs.layout != ROW_MAJOR:
            raise ValueError("SpMM RHS must be row-major")
        if self.lhs.scalar_cols != self.rhs.rows:
            raise ValueError(f"K mismatch: lhs has {self.lhs.scalar_cols} columns, "
                             f"rhs {self.rhs.rows} rows")
        scheme = self.scheme
        if self.rhs.bit_width == 4 and not self.lhs.shuffled:
            raise ShuffleStateError("4-bit RHS requires shuffled LHS column indices")
        if self.rhs.bit_width != 4 and self.lhs.shuffled:
            raise ShuffleStateError("shuffled LHS indices are only valid with a 4-bit RHS")
        if self.config.bs_m is not None and self.config.bs_m != self.lhs.vector_length:
            raise ValueError("BS_m must equal the vector length")
        bs_k = scheme.tile.k
        if self.config.bs_k is not None and self.config.bs_k != bs_k:
            raise ValueError(f"BS_k must equal the tile reduction {bs_k}")
        if self.lhs.stride % bs_k:
            raise ValueError(f"format stride {self.lhs.stride} must be a multiple of the tile k {bs_k}")

    @property
    def scheme(self) -> EmulationScheme:
        lhs_bits = getattr(self.lhs.values, "bit_width", 32)
        return emulation.plan(lhs_bits, self.rhs.bit_width, emulation.SPMM)


@dataclass(frozen=True, eq=False)
class SddmmProblem:
    a: PackedMatrix
    b: PackedMatrix
    out_pattern: BcrsMatrix
    out_format: str = "bcrs"
    config: TilingConfig = field(default_factory=TilingConfig)
    epilogue: Optional[Epilogue] = None

    def __post_init__(self):
        if self.a.layout != ROW_MAJOR:
            raise ValueError("SDDMM A must be row-major")
        if self.b.layout != COL_MAJOR:
            raise ValueError("SDDMM B must be column-major")
        if self.a.cols != self.b.rows:
            raise ValueError(f"K mismatch: {self.a.cols} vs {self.b.rows}")
        if self.out_pattern.scalar_rows != self.a.rows:
            raise ValueError("pattern rows must match A rows")
        if self.out_pattern.scalar_cols != self.b.cols:
            raise ValueError("pattern columns must match B columns")
        if self.out_format not in ("bcrs", "sr-bcrs"):
            raise ValueError("out_format must be 'bcrs' or 'sr-bcrs'")
        _ = self.scheme

    @property
    def scheme(self) -> EmulationScheme:
        return emulation.plan(self.a.bit_width, self.b.bit_width, emulation.SDDMM)


def _finish(out, host: bool, epilogue):
    if host:
        out = out.cpu().numpy()
    return epilogue(out) if epilogue is not None else out


def spmm_device(p: SpmmProblem, out=None, stream=None, check_status: bool = True):
    """Launch the SpMM kernel; returns the int32 CUDA tensor (no epilogue)."""
    t = D.torch()
    scheme = p.scheme
    check_accumulation_bound(p.lhs.scalar_cols, scheme.native_width)
    lib = N.lib()
    lhs, _k1 = D.srbcrs_struct(p.lhs)
    rhs, _k2 = D.dense_struct(p.rhs)
    if out is None:
        out = t.empty((p.lhs.scalar_rows, p.rhs.cols), dtype=t.int32, device="cuda")
    status = D.fresh_status() if check_status else D.status_word()
    s = N.stream_ptr(stream)
    # moderate sparsity: the library densifies the LHS into a workspace and runs an exact
    # tcgen05 GEMM (mc_spmm_workspace reports 0 when the gather kernels are used)
    need = N.ctypes.c_size_t(0)
    N.check(lib.mc_spmm_workspace(lhs, rhs, N.ctypes.byref(need)))
    ws = t.empty(int(need.value), dtype=t.uint8, device=out.device) if need.value else None
    N.check(lib.mc_spmm_ws(lhs, rhs, p.config.bs_n, N.ptr(out), N.ptr(status), N.ptr(ws),
                           int(need.value), s))
    if check_status:
        D.fetch_status(status, stream)
    return out


def spmm(p: SpmmProblem):
    """Dense M x N int32 product of the SR-BCRS LHS and the dense RHS (kernels.py:293-298)."""
    if p.config.pipeline:
        out, _ = spmm_pipelined(p)
        return out
    out = spmm_device(p)
    return _finish(out, D.any_host(p.lhs, p.rhs), p.epilogue)


def alg1_trace(steps: int) -> List[tuple]:
    """The Alg. 1 stage order (kernels.py:343-364) for one block."""
    t: List[tuple] = [("load_lhs", 0), ("sync",), ("prefetch_rhs", 0)]
    for i in range(1, steps):
        t += [("store_rhs", i - 1), ("load_lhs", i), ("sync",), ("prefetch_rhs", i),
              ("mma", i - 1), ("sync",)]
    t += [("store_rhs", steps - 1), ("sync",), ("mma", steps - 1)]
    return t


def spmm_pipelined(p: SpmmProblem):
    """SpMM plus the logical Alg. 1 schedule per thread block (kernels.py:301-311).

    The device kernel runs the prefetch pipeline as a 4-stage cp.async ring;
    the returned traces describe the reference's logical stage order for each
    (vector row, BS_n column block) with stored_count(r) / BS_k steps.
    """
    if not p.config.pipeline:
        raise ValueError("pipeline is off in this configuration")
    out = spmm_device(p)
    bs_k = p.scheme.tile.k
    bs_n = p.config.bs_n
    traces = []
    begin = np.asarray(D.torch().as_tensor(p.lhs.row_begin).cpu()) if D.is_torch(p.lhs.row_begin) \
        else p.lhs.row_begin
    end = np.asarray(D.torch().as_tensor(p.lhs.row_end).cpu()) if D.is_torch(p.lhs.row_end) \
        else p.lhs.row_end
    for r in range(p.lhs.vector_rows):
        true = int(end[r] - begin[r])
        steps = (-(-true // p.lhs.stride) * p.lhs.stride) // bs_k
        if steps == 0:
            continue
        trace = alg1_trace(steps)
        for c in range(0, p.rhs.cols, bs_n):
            traces.append(((r, c // bs_n), list(trace)))
    return _finish(out, D.any_host(p.lhs, p.rhs), p.epilogue), traces


def sddmm_device(p: SddmmProblem, out=None, stream=None, check_status: bool = True):
    """Launch the SDDMM kernel; returns the int32 block values (CUDA tensor)."""
    t = D.torch()
    scheme = p.scheme
    check_accumulation_bound(p.a.cols, scheme.native_width)
    lib = N.lib()
    a, _k1 = D.dense_struct(p.a)
    b, _k2 = D.dense_struct(p.b)
    pat, _k3 = D.bcrs_struct(p.out_pattern)
    v = p.out_pattern.vector_length
    if out is None:
        out = t.empty(p.out_pattern.n_blocks * v, dtype=t.int32, device="cuda")
    status = D.fresh_status() if check_status else D.status_word()
    s = N.stream_ptr(stream)
    N.check(lib.mc_sddmm(a, b, pat, N.ptr(out), N.ptr(status), s))
    if check_status:
        D.fetch_status(status, stream)
    return out


def sddmm(p: SddmmProblem) -> Union[BcrsMatrix, SrBcrsMatrix]:
    """Dense x dense sampled at the block pattern (kernels.py:367-435)."""
    host = D.any_host(p.a, p.b) or not D.on_device(p.out_pattern.row_offsets)
    values = sddmm_device(p)
    if host:
        values = values.cpu().numpy()
    if p.epilogue is not None:
        values = p.epilogue(values)
    pat = p.out_pattern
    out = BcrsMatrix(pat.scalar_rows, pat.scalar_cols, pat.vector_length, pat.row_offsets,
                     pat.col_indices, values)
    if p.out_format == "sr-bcrs":
        return bcrs_to_srbcrs(out, p.scheme.tile.k)
    return out
