"""Multi-GPU work partitioning for the hot path (no collective in the data path).

One process per GPU (torch.distributed, NCCL over NVLink on the B200 box, gloo in
CPU tests). SpMM / SDDMM are split into contiguous vector-row panels balanced by
stored vectors; attention is split over batch x head. Each rank computes a
disjoint slice of the output; `allgather_rows` (NCCL all-gather) is used only to
assemble outputs for validation, outside any timed region.

A rebased row panel of an SR-BCRS matrix reproduces exactly the corresponding
rows of the full product: row offsets are shifted by the panel's
first stored vector, and indices/values are sliced at stride boundaries, which
are word aligned for every supported (bits, V, stride) combination.
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .qint import PackedArray
from .sparse_format import BcrsMatrix, SrBcrsMatrix, _np


def _balanced_cuts(weights: np.ndarray, parts: int) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) ranges with near-equal total weight (prefix-sum split)."""
    n = int(weights.size)
    if parts <= 0:
        raise ValueError("parts must be positive")
    csum = np.concatenate([[0], np.cumsum(weights, dtype=np.int64)])
    total = int(csum[-1])
    cuts = [0]
    for i in range(1, parts):
        target = total * i / parts
        cuts.append(int(np.searchsorted(csum, target, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def row_panels(m: SrBcrsMatrix, parts: int) -> List[Tuple[int, int]]:
    """Vector-row panels of an SR-BCRS matrix balanced by stored vectors (+1 per row)."""
    begin, end = _np(m.row_begin, np.int64), _np(m.row_end, np.int64)
    stored = -(-(end - begin) // m.stride) * m.stride
    return _balanced_cuts(stored + 1, parts)


def srbcrs_panel(m: SrBcrsMatrix, lo: int, hi: int) -> SrBcrsMatrix:
    """Rebased sub-matrix of vector rows [lo, hi) (host arrays)."""
    v, s = m.vector_length, m.stride
    begin, end = _np(m.row_begin, np.int64), _np(m.row_end, np.int64)
    idx = _np(m.col_indices).view(np.uint32) if _np(m.col_indices).dtype != np.uint32 \
        else _np(m.col_indices)
    nrows = m.vector_rows
    p0 = int(begin[lo]) if lo < nrows else int(idx.size)
    p1 = int(begin[hi]) if hi < nrows else int(idx.size)
    vals = m.values
    if isinstance(vals, PackedArray):
        bits = vals.bit_width
        if (p0 * v * bits) % 32 or (p1 * v * bits) % 32:
            raise ValueError("panel boundary is not word aligned")
        words = _np(vals.words).view(np.uint32)
        sub_vals = PackedArray((p1 - p0) * v, bits, vals.signed,
                               words[p0 * v * bits // 32:p1 * v * bits // 32].copy())
    else:
        sub_vals = _np(vals)[p0 * v:p1 * v].copy()
    return SrBcrsMatrix((hi - lo) * v, m.scalar_cols, v, s, begin[lo:hi] - p0, end[lo:hi] - p0,
                        idx[p0:p1].copy(), sub_vals, shuffled=m.shuffled)


def bcrs_panel(b: BcrsMatrix, lo: int, hi: int) -> BcrsMatrix:
    """Rebased BCRS pattern/values of vector rows [lo, hi) (SDDMM output rows)."""
    offs = _np(b.row_offsets, np.int64)
    p0, p1 = int(offs[lo]), int(offs[hi])
    v = b.vector_length
    vals = b.values
    if isinstance(vals, PackedArray):
        flat = vals.to_values()[p0 * v:p1 * v]
        sub_vals = PackedArray.from_values(flat, vals.bit_width, vals.signed)
    else:
        sub_vals = _np(vals)[p0 * v:p1 * v].copy()
    return BcrsMatrix((hi - lo) * v, b.scalar_cols, v, offs[lo:hi + 1] - p0,
                      _np(b.col_indices).astype(np.uint32)[p0:p1].copy(), sub_vals)


def pattern_panels(b: BcrsMatrix, parts: int) -> List[Tuple[int, int]]:
    offs = _np(b.row_offsets, np.int64)
    return _balanced_cuts(np.diff(offs) + 1, parts)


def head_ranges(n_heads: int, parts: int) -> List[Tuple[int, int]]:
    """Batch x head split for attention: contiguous, sizes differ by at most one."""
    return [(n_heads * i // parts, n_heads * (i + 1) // parts) for i in range(parts)]


def allgather_rows(local, parts: Sequence[Tuple[int, int]], rows_per_unit: int, group=None):
    """All-gather per-rank row slices (torch tensors) into the full row-stacked tensor.

    Validation-only collective (NCCL on GPU, gloo on CPU): slices are padded to the
    largest one, gathered, then trimmed and concatenated in rank order.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [(hi - lo) * rows_per_unit for lo, hi in parts]
    width = max(sizes) if sizes else 0
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[r][:sizes[r]] for r in range(world)], dim=0)
