"""Numpy restatement of the reference Magicube (`qsparse`) hot path.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py. Never imported by the
product package.

Every function cites the reference function it restates
(paths relative to /root/reference/pkg/src/qsparse/). The restatement keeps
the reference's *semantics* -- chunk plans, sentinel handling, the int32
overflow checks at the same intermediate points, the fp16/fp64 rounding chain
of the attention pipeline -- but computes chunk products with exact float64
BLAS gathers instead of the reference's per-warp tile simulation. Chunk
products are bounded by K*255*255 < 2**53, so float64 is exact.
"""

from __future__ import annotations

import hashlib
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "SENTINEL", "SHUFFLE_PERM", "SHUFFLE_PERM_INV", "INT32_MIN", "INT32_MAX",
    "OracleOverflow", "pack_bits", "unpack_bits", "chunk_split", "plan",
    "check_bound", "chunk_groups", "safe_magnitudes", "cell_seed",
    "synthetic_bcrs", "bcrs_dense", "srbcrs_from_bcrs", "shuffle_idx",
    "unshuffle_idx", "srbcrs_dense", "spmm", "sddmm", "fp16_round", "quantize",
    "attention", "build_spmm_case", "build_sddmm_case", "build_attention_case",
]

SENTINEL = 0xFFFFFFFF                    # sparse_format.py:25
SHUFFLE_PERM = (0, 2, 4, 6, 1, 3, 5, 7)  # tile_engine.py:35
SHUFFLE_PERM_INV = (0, 4, 1, 5, 2, 6, 3, 7)
INT32_MIN = -(1 << 31)                   # tile_engine.py:29-30
INT32_MAX = (1 << 31) - 1

SPMM_PAIRS = {(16, 16), (16, 8), (16, 4), (12, 4), (8, 4), (8, 8), (4, 4)}  # emulation.py:23-30
SDDMM_PAIRS = {(16, 16), (8, 8), (4, 4)}


class OracleOverflow(ArithmeticError):
    """Raised where the reference raises OverflowRiskError."""


class OracleUnsupported(ValueError):
    """Raised where the reference raises UnsupportedPrecisionError."""


# --------------------------------------------------------------------------
# bit packing (qint.py:41-82): LSB-first uint32 words, sign-extending unpack
# --------------------------------------------------------------------------

def pack_bits(values, bits: int) -> np.ndarray:
    """qint.pack_values (qint.py:41-62): two's complement, LSB-first, zero tail."""
    v = np.asarray(values, dtype=np.int64).ravel()
    n_words = (v.size * bits + 31) // 32
    if v.size == 0:
        return np.zeros(n_words, dtype=np.uint32)
    raw = (v & ((1 << bits) - 1)).astype(np.uint64)
    bitmat = ((raw[:, None] >> np.arange(bits, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)
    flat = bitmat.ravel()
    pad = n_words * 32 - flat.size
    if pad:
        flat = np.concatenate([flat, np.zeros(pad, dtype=np.uint8)])
    return np.packbits(flat, bitorder="little").view("<u4").astype(np.uint32)


def unpack_bits(words, count: int, bits: int, signed: bool = True) -> np.ndarray:
    """qint.unpack_values (qint.py:65-82)."""
    if count == 0:
        return np.zeros(0, dtype=np.int64)
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32)).view(np.uint8)
    b = np.unpackbits(w, bitorder="little")[: count * bits].reshape(count, bits)
    v = (b.astype(np.int64) << np.arange(bits, dtype=np.int64)).sum(axis=1)
    if signed:
        v -= (v >> (bits - 1)) << bits
    return v


def chunk_split(values, src_bits: int, width: int, signed: bool = True) -> List[np.ndarray]:
    """qint.chunk_values (qint.py:209-225): low chunks unsigned, top chunk signed."""
    v = np.asarray(values, dtype=np.int64)
    n = src_bits // width
    mask = (1 << width) - 1
    out = [(v >> (width * i)) & mask for i in range(n)]
    if signed:
        top = out[-1]
        out[-1] = top - ((top >> (width - 1)) << width)
    return out


# --------------------------------------------------------------------------
# emulation plan (emulation.py:67-113)
# --------------------------------------------------------------------------

def plan(lhs_bits: int, rhs_bits: int, op: str = "spmm") -> Dict[str, object]:
    """emulation.plan: native width 8 iff both widths divide by 8, else 4."""
    pairs = SPMM_PAIRS if op == "spmm" else SDDMM_PAIRS
    if (lhs_bits, rhs_bits) not in pairs:
        raise OracleUnsupported(f"L{lhs_bits}-R{rhs_bits} unsupported for {op}")
    w = 8 if (lhs_bits % 8 == 0 and rhs_bits % 8 == 0) else 4
    lc, rc = lhs_bits // w, rhs_bits // w
    return {"width": w, "lhs_chunks": lc, "rhs_chunks": rc,
            "tile_k": 16 if w == 8 else 32}


def check_bound(k: int, width: int) -> None:
    """emulation.check_accumulation_bound (emulation.py:108-113)."""
    worst = (1 << width) - 1
    if k * worst * worst > INT32_MAX:
        raise OracleOverflow(f"K={k} risks int32 overflow at {width}-bit chunks")


def chunk_groups(n_chunks: int, v: int) -> List[List[int]]:
    """kernels._chunk_groups (kernels.py:121-128): stacking groups for V<8."""
    per = max(1, 8 // v) if v < 8 else 1
    return [list(range(b, min(b + per, n_chunks))) for b in range(0, n_chunks, per)]


def _recombine(acc: Dict[Tuple[int, int], np.ndarray], lc: int, rc: int, w: int,
               v: int, what: str) -> np.ndarray:
    """kernels._SpmmBlock.result + tile_engine.redistribute_stacked checks
    (kernels.py:265-275, tile_engine.py:221-248, kernels.py:286-290)."""
    out = None
    for j in range(rc):
        for grp in chunk_groups(lc, v):
            comb = sum((1 << (w * c)) * acc[(c, j)] for c in grp)
            if comb.size and (comb.min() < INT32_MIN or comb.max() > INT32_MAX):
                raise OracleOverflow("stacked recombination exceeds int32")
            term = (1 << (w * j)) * comb
            out = term if out is None else out + term
    if out.size and (out.min() < INT32_MIN or out.max() > INT32_MAX):
        raise OracleOverflow(f"{what} output exceeds int32")
    return out.astype(np.int32)


# --------------------------------------------------------------------------
# input generation (bench.py:70-136, sparse_format.py:453-476)
# --------------------------------------------------------------------------

def safe_magnitudes(lhs_bits: int, rhs_bits: int, k: int, op: str) -> Tuple[int, int]:
    """bench.safe_magnitudes (bench.py:70-83)."""
    w = plan(lhs_bits, rhs_bits, op)["width"]
    limit = (1 << 31) - 1
    kk = max(k, 1)
    root = int(math.isqrt(limit // kk))
    mag_l = min((1 << (lhs_bits - 1)) - 1, root, limit // (kk * ((1 << w) - 1)))
    mag_r = min((1 << (rhs_bits - 1)) - 1, root)
    return max(mag_l, 1), max(mag_r, 1)


def cell_seed(sweep_seed: int, coords: tuple) -> int:
    """bench._cell_seed (bench.py:86-90): sha256 of the coordinate repr."""
    key = repr((sweep_seed,) + tuple(coords)).encode()
    return int.from_bytes(hashlib.sha256(key).digest()[:4], "little")


def synthetic_bcrs(rows: int, cols: int, v: int, sparsity: float, seed: int,
                   bit_width: int = 8, max_magnitude: Optional[int] = None):
    """sparse_format.generate_synthetic (sparse_format.py:453-476).

    Returns (row_offsets int64, col_indices uint32, values int64 block-major).
    Reproduces the reference RNG call sequence exactly.
    """
    if not 0 <= sparsity < 1:
        raise ValueError("sparsity must be in [0, 1)")
    rng = np.random.default_rng(seed)
    per_row = int((1 - sparsity) * cols)
    nrows = rows // v
    cap = max_magnitude if max_magnitude is not None else (1 << (bit_width - 1)) - 1
    picks = [np.sort(rng.choice(cols, size=per_row, replace=False)) for _ in range(nrows)]
    col_idx = (np.concatenate(picks) if picks else np.zeros(0)).astype(np.uint32)
    offsets = np.arange(nrows + 1, dtype=np.int64) * per_row
    n = col_idx.size * v
    mags = rng.integers(1, cap + 1, size=n)
    signs = rng.choice((-1, 1), size=n)
    return offsets, col_idx, (mags * signs).astype(np.int64)


def bcrs_dense(rows: int, cols: int, v: int, offsets, col_idx, values) -> np.ndarray:
    """sparse_format.bcrs_to_dense (sparse_format.py:273-281)."""
    vals = np.asarray(values)
    dtype = vals.dtype if vals.dtype.kind == "f" else np.int64
    d = np.zeros((rows, cols), dtype=dtype)
    offs = np.asarray(offsets, dtype=np.int64)
    counts = np.diff(offs)
    vrow = np.repeat(np.arange(counts.size), counts)
    c = np.asarray(col_idx, dtype=np.int64)
    blk = vals.reshape(-1, v) if vals.size else vals.reshape(0, v)
    for lane in range(v):
        d[vrow * v + lane, c] = blk[:, lane]
    return d


def srbcrs_from_bcrs(offsets, col_idx, values, v: int, stride: int):
    """sparse_format.bcrs_to_srbcrs (sparse_format.py:284-315), vectorised.

    Returns (row_begin, row_end, col_indices(sentinel padded), values(stride
    layout: element (lane, j) of stride s at s*V*S + lane*S + j)).
    """
    offs = np.asarray(offsets, dtype=np.int64)
    true = np.diff(offs)
    stored = -(-true // stride) * stride
    begin = np.concatenate([[0], np.cumsum(stored)[:-1]]).astype(np.int64) if true.size \
        else np.zeros(0, dtype=np.int64)
    end = begin + true
    total = int(stored.sum())
    idx = np.full(total, SENTINEL, dtype=np.uint32)
    vals_in = np.asarray(values)
    vals = np.zeros(total * v, dtype=vals_in.dtype if vals_in.dtype.kind == "f" else np.int64)
    nblk = int(offs[-1]) if offs.size else 0
    if nblk:
        row = np.repeat(np.arange(true.size), true)
        local = np.arange(nblk) - offs[row]
        pos = begin[row] + local
        idx[pos] = np.asarray(col_idx, dtype=np.uint32)[:nblk]
        s_base = (begin[row] + (local // stride) * stride) * v
        j = local % stride
        blk = vals_in.reshape(-1, v)
        for lane in range(v):
            vals[s_base + lane * stride + j] = blk[:, lane]
    return begin, end, idx, vals


def shuffle_idx(col_idx) -> np.ndarray:
    """sparse_format.shuffle_indices (sparse_format.py:373-385): new[p] = old[P[p]]."""
    idx = np.asarray(col_idx, dtype=np.uint32).reshape(-1, 8)
    return idx[:, list(SHUFFLE_PERM)].reshape(-1)


def unshuffle_idx(col_idx) -> np.ndarray:
    """SrBcrsMatrix.unshuffled_indices (sparse_format.py:222-230)."""
    idx = np.asarray(col_idx, dtype=np.uint32).reshape(-1, 8)
    out = np.empty_like(idx)
    out[:, list(SHUFFLE_PERM)] = idx
    return out.reshape(-1)


def _stored_matrix(begin, end, stride):
    true = np.asarray(end, dtype=np.int64) - np.asarray(begin, dtype=np.int64)
    return -(-true // stride) * stride


def srbcrs_dense(rows, cols, v, stride, begin, end, col_idx, values, shuffled=False):
    """sparse_format.srbcrs_to_dense (sparse_format.py:318-337): padding ignored."""
    idx = unshuffle_idx(col_idx) if shuffled else np.asarray(col_idx, dtype=np.uint32)
    vals = np.asarray(values)
    d = np.zeros((rows, cols), dtype=vals.dtype if vals.dtype.kind == "f" else np.int64)
    for r in range(len(begin)):
        b0, true = int(begin[r]), int(end[r] - begin[r])
        for j in range(true):
            p = b0 + j
            base = (p // stride) * v * stride + (p % stride)
            d[r * v:(r + 1) * v, int(idx[p])] = vals[base + np.arange(v) * stride]
    return d


# --------------------------------------------------------------------------
# SpMM (kernels.py:278-340)
# --------------------------------------------------------------------------

def spmm(begin, end, col_idx, values, v: int, stride: int, shuffled: bool,
         lhs_bits: int, rhs_dense: np.ndarray, rhs_bits: int, k: int,
         rows: Optional[Sequence[int]] = None) -> np.ndarray:
    """kernels.spmm semantics (kernels.py:293-340).

    Every stored slot contributes value * B[idx] (a sentinel index gathers a
    zero row, kernels.py:224-236); chunk products at the plan width are
    recombined with the reference's stacked-group and final int32 checks.
    `rows` restricts the computation to a subset of vector rows (used for
    bounded CPU baselines); the result then has len(rows)*V rows.
    """
    p = plan(lhs_bits, rhs_bits, "spmm")
    w, lc, rc = p["width"], p["lhs_chunks"], p["rhs_chunks"]
    check_bound(k, w)
    begin = np.asarray(begin, dtype=np.int64)
    end = np.asarray(end, dtype=np.int64)
    idx = unshuffle_idx(col_idx) if shuffled else np.asarray(col_idx, dtype=np.uint32)
    vals = np.asarray(values, dtype=np.int64)
    b = np.asarray(rhs_dense, dtype=np.int64)
    n = b.shape[1]
    b_chunks = [c.astype(np.float64) for c in
                (chunk_split(b, rhs_bits, w) if rc > 1 else [b])]
    # one zero row appended: sentinel slots gather it (kernels.py:231-234)
    b_chunks = [np.vstack([c, np.zeros((1, n))]) for c in b_chunks]
    stored = _stored_matrix(begin, end, stride)
    sel = range(len(begin)) if rows is None else rows
    out_rows = []
    for r in sel:
        cnt = int(stored[r])
        acc = {(c, j): np.zeros((v, n), dtype=np.int64) for c in range(lc) for j in range(rc)}
        if cnt:
            pos = int(begin[r]) + np.arange(cnt)
            ridx = idx[pos].astype(np.int64)
            ridx = np.where(idx[pos] == SENTINEL, k, ridx)
            vblk = vals[(pos // stride)[None, :] * v * stride
                        + np.arange(v)[:, None] * stride + (pos % stride)[None, :]]
            a_chunks = chunk_split(vblk, lhs_bits, w) if lc > 1 else [vblk]
            for c in range(lc):
                ac = a_chunks[c].astype(np.float64)
                for j in range(rc):
                    acc[(c, j)] = (ac @ b_chunks[j][ridx]).astype(np.int64)
        out_rows.append(acc)
    if not out_rows:
        return np.zeros((0, n), dtype=np.int32)
    stacked = {key: np.concatenate([a[key] for a in out_rows], axis=0) for key in out_rows[0]}
    return _recombine(stacked, lc, rc, w, v, "SpMM")


# --------------------------------------------------------------------------
# SDDMM (kernels.py:367-435)
# --------------------------------------------------------------------------

def sddmm(a_dense: np.ndarray, b_dense: np.ndarray, offsets, col_idx, v: int,
          lhs_bits: int, rhs_bits: int) -> np.ndarray:
    """kernels.sddmm semantics: int32 values, block-major, V per block."""
    p = plan(lhs_bits, rhs_bits, "sddmm")
    w, lc, rc = p["width"], p["lhs_chunks"], p["rhs_chunks"]
    a = np.asarray(a_dense, dtype=np.int64)
    b = np.asarray(b_dense, dtype=np.int64)
    check_bound(a.shape[1], w)
    a_ch = [c.astype(np.float64) for c in (chunk_split(a, lhs_bits, w) if lc > 1 else [a])]
    b_ch = [c.astype(np.float64) for c in (chunk_split(b, rhs_bits, w) if rc > 1 else [b])]
    offs = np.asarray(offsets, dtype=np.int64)
    cols = np.asarray(col_idx, dtype=np.int64)
    nblk = int(offs[-1]) if offs.size else 0
    acc = {(c, j): np.zeros((nblk, v), dtype=np.int64) for c in range(lc) for j in range(rc)}
    for r in range(offs.size - 1):
        lo, hi = int(offs[r]), int(offs[r + 1])
        if hi == lo:
            continue
        cc = cols[lo:hi]
        for c in range(lc):
            arow = a_ch[c][r * v:(r + 1) * v]
            for j in range(rc):
                acc[(c, j)][lo:hi] = (arow @ b_ch[j][:, cc]).T.astype(np.int64)
    return _recombine(acc, lc, rc, w, v, "SDDMM").reshape(-1)


# --------------------------------------------------------------------------
# quantized sparse attention (attention.py:40-187)
# --------------------------------------------------------------------------

def fp16_round(x) -> np.ndarray:
    """attention._fp16_round (attention.py:63-65)."""
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def quantize(x, bits: int) -> Tuple[np.ndarray, float]:
    """attention.quantize (attention.py:40-56): symmetric absmax, ties-to-even."""
    arr = np.asarray(x, dtype=np.float64)
    if not np.isfinite(arr).all():
        raise ValueError("input must be finite")
    qmax = (1 << (bits - 1)) - 1
    absmax = float(np.abs(arr).max()) if arr.size else 0.0
    scale = absmax / qmax if absmax > 0 else 1.0
    q = np.clip(np.rint(arr / scale), -qmax, qmax).astype(np.int64)
    return q, scale


def _row_softmax(vals: np.ndarray, offsets, v: int) -> np.ndarray:
    """attention._row_softmax (attention.py:108-127), same numpy op order."""
    out = np.zeros_like(vals)
    offs = np.asarray(offsets, dtype=np.int64)
    for r in range(offs.size - 1):
        lo, hi = int(offs[r]), int(offs[r + 1])
        if hi == lo:
            continue
        rows = vals[lo * v:hi * v].reshape(hi - lo, v).T
        shifted = np.exp(rows - rows.max(axis=1, keepdims=True))
        probs = fp16_round(shifted / shifted.sum(axis=1, keepdims=True))
        out[lo * v:hi * v] = probs.T.reshape(-1)
    return out


def attention(q, k, vmat, offsets, col_idx, seq_len: int, head_dim: int,
              softmax_bits: int, qkv_bits: int) -> Dict[str, np.ndarray]:
    """attention.sparse_attention (attention.py:130-187) for one head.

    Returns the integer stages and the fp16-rounded output:
    scores_int (block-major int32), scores (fp16-rounded f64), probs,
    probs_int (block-major), mix_int (L x d int32), output (L x d f64),
    and the four scales.
    """
    v = 8
    qq, sq = quantize(q, qkv_bits)
    kq, sk = quantize(k, qkv_bits)
    vq, sv = quantize(vmat, qkv_bits)
    scores_int = sddmm(qq, kq.T, offsets, col_idx, v, qkv_bits, qkv_bits)
    alpha = sq * sk / np.sqrt(head_dim)
    scores = fp16_round(scores_int.astype(np.float64) * alpha)
    probs = _row_softmax(scores, offsets, v)
    smax = (1 << (softmax_bits - 1)) - 1
    sm_scale = 1.0 / smax
    probs_int = np.clip(np.rint(probs / sm_scale), -smax, smax).astype(np.int64)
    tile_k = plan(softmax_bits, qkv_bits, "spmm")["tile_k"]
    begin, end, sidx, svals = srbcrs_from_bcrs(offsets, col_idx, probs_int, v, tile_k)
    shuffled = qkv_bits == 4
    if shuffled:
        sidx = shuffle_idx(sidx)
    mix_int = spmm(begin, end, sidx, svals, v, tile_k, shuffled, softmax_bits,
                   vq, qkv_bits, seq_len)
    output = fp16_round(mix_int.astype(np.float64) * (sm_scale * sv))
    return {"scores_int": scores_int, "scores": scores, "probs": probs,
            "probs_int": probs_int, "mix_int": mix_int, "output": output,
            "scales": np.array([sq, sk, sv, sm_scale])}


# --------------------------------------------------------------------------
# problem builders mirroring bench._build_* (bench.py:93-136)
# --------------------------------------------------------------------------

def build_spmm_case(m: int, n: int, k: int, v: int, sparsity: float,
                    lhs_bits: int, rhs_bits: int, seed: int, stride_mult: int = 1):
    """bench._build_spmm (bench.py:93-110): SR-BCRS LHS + dense RHS, same RNG."""
    p = plan(lhs_bits, rhs_bits, "spmm")
    mag_l, mag_r = safe_magnitudes(lhs_bits, rhs_bits, k, "spmm")
    offs, cidx, vals = synthetic_bcrs(m, k, v, sparsity, seed, lhs_bits, mag_l)
    stride = p["tile_k"] * stride_mult
    begin, end, sidx, svals = srbcrs_from_bcrs(offs, cidx, vals, v, stride)
    shuffled = rhs_bits == 4
    if shuffled:
        sidx = shuffle_idx(sidx)
    rng = np.random.default_rng(seed + 1)
    rhs = rng.integers(-mag_r, mag_r + 1, (k, n))
    return {"m": m, "n": n, "k": k, "v": v, "stride": stride, "shuffled": shuffled,
            "lhs_bits": lhs_bits, "rhs_bits": rhs_bits,
            "bcrs_offsets": offs, "bcrs_cols": cidx, "bcrs_values": vals,
            "row_begin": begin, "row_end": end, "col_indices": sidx,
            "values": svals, "rhs": rhs.astype(np.int64)}


def build_sddmm_case(m: int, n: int, k: int, v: int, sparsity: float,
                     lhs_bits: int, rhs_bits: int, seed: int):
    """bench._build_sddmm (bench.py:113-126)."""
    mag_l, mag_r = safe_magnitudes(lhs_bits, rhs_bits, k, "sddmm")
    offs, cidx, _ = synthetic_bcrs(m, n, v, sparsity, seed, 8)
    rng = np.random.default_rng(seed + 1)
    a = rng.integers(-mag_l, mag_l + 1, (m, k))
    b = rng.integers(-mag_r, mag_r + 1, (k, n))
    return {"m": m, "n": n, "k": k, "v": v, "lhs_bits": lhs_bits, "rhs_bits": rhs_bits,
            "offsets": offs, "col_indices": cidx, "a": a.astype(np.int64),
            "b": b.astype(np.int64)}


def build_attention_case(seq_len: int, head_dim: int, sparsity: float, seed: int):
    """bench._build_attention (bench.py:129-136): mask + N(0,1) q, k, v."""
    offs, cidx, _ = synthetic_bcrs(seq_len, seq_len, 8, sparsity, seed, 8)
    rng = np.random.default_rng(seed + 1)
    q, k, vmat = (rng.normal(size=(seq_len, head_dim)) for _ in range(3))
    return {"offsets": offs, "col_indices": cidx, "q": q, "k": k, "v": vmat}
