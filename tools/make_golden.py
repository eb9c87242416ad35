"""Generate golden vectors by importing the reference `qsparse` package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Writes tests/golden/*.npz. Every output array is produced by the reference's
own public API (kernels.spmm / kernels.sddmm / attention.sparse_attention /
sparse_format / qint), so the fixtures pin both the oracle restatement and the
CUDA path to the reference's behaviour.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("QSPARSE_SRC", "/root/reference/pkg/src"))

from qsparse import attention as at  # noqa: E402
from qsparse import bench as rb  # noqa: E402
from qsparse import emulation as em  # noqa: E402
from qsparse import kernels as kn  # noqa: E402
from qsparse import qint  # noqa: E402
from qsparse import sparse_format as sf  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

SPMM_PAIRS = [(8, 8), (4, 4), (16, 16), (16, 8), (16, 4), (12, 4), (8, 4)]
SDDMM_PAIRS = [(8, 8), (4, 4), (16, 16)]


def srbcrs_arrays(prefix, s: sf.SrBcrsMatrix, d: dict):
    d[prefix + "meta"] = np.array([s.scalar_rows, s.scalar_cols, s.vector_length, s.stride,
                                   s.values.bit_width, int(s.shuffled)], dtype=np.int64)
    d[prefix + "row_begin"] = s.row_begin
    d[prefix + "row_end"] = s.row_end
    d[prefix + "col_indices"] = s.col_indices
    d[prefix + "words"] = s.values.words


def spmm_case(d, name, seed, m=32, n=64, k=128, v=8, sparsity=0.7, lb=8, rbits=8,
              bs_n=64, stride_mult=1):
    scheme = em.plan(lb, rbits, em.SPMM)
    mag_l, mag_r = rb.safe_magnitudes(lb, rbits, k, em.SPMM)
    b = sf.generate_synthetic(m, k, v, sparsity, seed, bit_width=lb, max_magnitude=mag_l)
    lhs = sf.bcrs_to_srbcrs(b, scheme.tile.k * stride_mult)
    if rbits == 4:
        lhs = sf.shuffle_indices(lhs)
    rng = np.random.default_rng(seed + 1)
    rhs_dense = rng.integers(-mag_r, mag_r + 1, (k, n))
    rhs = qint.pack_dense(rhs_dense, rbits)
    out = kn.spmm(kn.SpmmProblem(lhs, rhs, kn.TilingConfig(bs_n=bs_n)))
    assert (out == sf.bcrs_to_dense(b) @ rhs_dense).all()
    p = name + "/"
    srbcrs_arrays(p + "lhs_", lhs, d)
    d[p + "bcrs_offsets"] = b.row_offsets
    d[p + "bcrs_cols"] = b.col_indices
    d[p + "bcrs_words"] = b.values.words
    d[p + "args"] = np.array([m, n, k, v, sparsity * 1000, lb, rbits, seed, stride_mult],
                             dtype=np.int64)
    d[p + "rhs_words"] = rhs.words
    d[p + "out"] = out


def sddmm_case(d, name, seed, m=32, n=48, k=64, v=8, sparsity=0.8, lb=8, rbits=8,
               out_format="bcrs"):
    mag_l, mag_r = rb.safe_magnitudes(lb, rbits, k, em.SDDMM)
    pattern = sf.generate_synthetic(m, n, v, sparsity, seed, bit_width=8)
    rng = np.random.default_rng(seed + 1)
    a_dense = rng.integers(-mag_l, mag_l + 1, (m, k))
    b_dense = rng.integers(-mag_r, mag_r + 1, (k, n))
    a = qint.pack_dense(a_dense, lb, qint.ROW_MAJOR)
    bm = qint.pack_dense(b_dense, rbits, qint.COL_MAJOR)
    out = kn.sddmm(kn.SddmmProblem(a, bm, pattern, out_format=out_format))
    p = name + "/"
    d[p + "args"] = np.array([m, n, k, v, sparsity * 1000, lb, rbits, seed,
                              int(out_format == "sr-bcrs")], dtype=np.int64)
    d[p + "a_words"] = a.words
    d[p + "b_words"] = bm.words
    d[p + "pattern_offsets"] = pattern.row_offsets
    d[p + "pattern_cols"] = pattern.col_indices
    if out_format == "bcrs":
        d[p + "out_values"] = np.asarray(out.values)
    else:
        d[p + "out_row_begin"] = out.row_begin
        d[p + "out_row_end"] = out.row_end
        d[p + "out_col_indices"] = out.col_indices
        d[p + "out_values"] = np.asarray(out.values)
        d[p + "out_stride"] = np.array([out.stride])


def attention_case(d, name, seq_len, sb, qb, sparsity, seed, head_dim=64, dense_mask=None):
    if dense_mask is None:
        mask = sf.generate_synthetic(seq_len, seq_len, 8, sparsity, seed)
    else:
        mask = sf.dense_to_bcrs(dense_mask, 8)
    cfg = at.AttentionConfig(seq_len, sb, qb, mask, head_dim=head_dim)
    rng = np.random.default_rng(seed + 1000)
    # fp16-representable inputs so device and reference see identical values
    q, k, v = (rng.normal(size=(seq_len, head_dim)).astype(np.float16).astype(np.float64)
               for _ in range(3))
    res = at.sparse_attention(q, k, v, cfg)
    p = name + "/"
    d[p + "args"] = np.array([seq_len, sb, qb, head_dim, seed], dtype=np.int64)
    d[p + "mask_offsets"] = mask.row_offsets
    d[p + "mask_cols"] = mask.col_indices
    d[p + "q"], d[p + "k"], d[p + "v"] = (x.astype(np.float16) for x in (q, k, v))
    d[p + "scores_int"] = res.scores_int
    d[p + "scores"] = np.asarray(res.scores._flat_values).astype(np.float16)
    d[p + "probs"] = np.asarray(res.probs._flat_values).astype(np.float16)
    d[p + "probs_int"] = res.probs_int.values.to_values()
    d[p + "mix_int"] = res.mix_int
    d[p + "output"] = res.output.astype(np.float16)
    d[p + "scales"] = np.array([res.params["q"].scale, res.params["k"].scale,
                                res.params["v"].scale, res.params["softmax"].scale])


def irregular_csr(rows, cols, seed):
    """An irregular DLMC-like pattern: per-row lengths 0..cols/3, sorted distinct columns."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, cols // 3 + 1, rows)
    lens[::7] = 0  # empty rows
    lens[3] = cols  # one full row
    idx = [np.sort(rng.choice(cols, size=int(n), replace=False)) for n in lens]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    return sf.CsrMatrix(rows, cols, int(offs[-1]), offs, np.concatenate(idx).astype(np.uint32))


def extra_goldens():
    """Round-2 fixtures: DLMC ingestion through the reference bench builders
    (bench.py:93-126, sparse_format.py:388-450) and the reference's per-nibble group
    check of 4-bit-width plans (tile_engine.py:246-247 via kernels.py:265-275)."""
    import io
    d = {}
    tiny = "3, 5, 2\n0 1 1 2\n4 0\n"  # test_sparse_format.py:10
    csr = sf.read_dlmc(tiny)
    d["dlmc_tiny/text"] = np.frombuffer(tiny.encode(), dtype=np.uint8)
    d["dlmc_tiny/offsets"] = csr.row_offsets
    d["dlmc_tiny/cols"] = csr.col_indices
    csr = irregular_csr(48, 256, seed=21)
    buf = io.StringIO()
    sf.write_dlmc(csr, buf)
    text = buf.getvalue()
    d["dlmc_irr/text"] = np.frombuffer(text.encode(), dtype=np.uint8)
    for (lb, rbits, v) in [(8, 8, 8), (8, 4, 8), (16, 8, 4), (4, 4, 2), (16, 16, 8)]:
        spec = rb.SweepSpec("spmm", [(0, 64, 256)], dlmc=sf.read_dlmc(text))
        seed = 1000 + lb * 10 + rbits + v
        prob, (m, n, k), _, _ = rb._build_spmm(spec, (0, 64, 256), v, 0.0, lb, rbits, seed)
        out = kn.spmm(prob)
        p = f"dlmc_spmm_{lb}_{rbits}_v{v}/"
        d[p + "args"] = np.array([m, n, k, v, lb, rbits, seed], dtype=np.int64)
        srbcrs_arrays(p + "lhs_", prob.lhs, d)
        d[p + "rhs_words"] = prob.rhs.words
        d[p + "out"] = out
    for (lb, rbits, v) in [(8, 8, 8), (16, 16, 4), (4, 4, 8)]:
        spec = rb.SweepSpec("sddmm", [(0, 0, 96)], dlmc=sf.read_dlmc(text))
        seed = 2000 + lb * 10 + rbits + v
        prob, (m, n, k), _, _ = rb._build_sddmm(spec, (0, 0, 96), v, 0.0, lb, rbits, seed)
        out = kn.sddmm(prob)
        p = f"dlmc_sddmm_{lb}_{rbits}_v{v}/"
        d[p + "args"] = np.array([m, n, k, v, lb, rbits, seed], dtype=np.int64)
        d[p + "offsets"] = prob.out_pattern.row_offsets
        d[p + "cols"] = prob.out_pattern.col_indices
        d[p + "a_words"] = prob.a.words
        d[p + "b_words"] = prob.b.words
        d[p + "out"] = np.asarray(out.values)
    # per-nibble group check (L16-R4, V = 8): the top-nibble group sum 4096 * sum(c3 * b)
    # leaves int32 while the final result still fits -> the reference raises
    for name, aval, k in [("nib_raise", -28673, 9216), ("nib_ok", 100, 9216)]:
        dense = np.full((8, k), aval, dtype=np.int64)
        lhs = sf.shuffle_indices(sf.bcrs_to_srbcrs(sf.dense_to_bcrs(dense, 8, bit_width=16), 32))
        rhs = qint.pack_dense(np.full((k, 64), -8, dtype=np.int64), 4)
        p = name + "/"
        d[p + "args"] = np.array([aval, k], dtype=np.int64)
        try:
            d[p + "out"] = kn.spmm(kn.SpmmProblem(lhs, rhs))
            d[p + "raises"] = np.array([0])
        except Exception as e:  # OverflowRiskError
            d[p + "raises"] = np.array([1])
            d[p + "error"] = np.frombuffer(type(e).__name__.encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "extra.npz"), **d)


def main():
    os.makedirs(OUT, exist_ok=True)
    if os.environ.get("GOLDEN_ONLY") == "extra":
        extra_goldens()
        return
    extra_goldens()

    # ---- qint / sparse_format KATs ----
    d = {}
    rng = np.random.default_rng(123)
    for bits in (4, 8, 12, 16):
        lo, hi = qint.signed_range(bits)
        vals = rng.integers(lo, hi + 1, 257)
        d[f"pack{bits}/values"] = vals
        d[f"pack{bits}/words"] = qint.pack_values(vals, bits)
    d["kat/neg19_int8"] = qint.pack_values([-19], 8)
    d["kat/split_signed_m19_4_2"] = np.array(qint.split_signed(-19, 4, 2).chunks)
    d["kat/split_unsigned_237_4_2"] = np.array(qint.split_unsigned(237, 4, 2).chunks)
    # hand SR-BCRS layout (test_sparse_format.py:46-56)
    dm = np.zeros((2, 8), dtype=np.int64)
    dm[:, 1] = (1, 2)
    dm[:, 5] = (3, 4)
    dm[:, 7] = (5, 6)
    s = sf.bcrs_to_srbcrs(sf.dense_to_bcrs(dm, 2), 4)
    srbcrs_arrays("hand_", s, d)
    d["hand_dense"] = dm
    # generator + packer + shuffle reproduction
    for i, (rows, cols, v, sp, seed, bw, stride) in enumerate(
            [(64, 128, 8, 0.7, 5, 8, 16), (32, 96, 4, 0.9, 6, 16, 16),
             (48, 64, 2, 0.5, 7, 4, 32), (64, 256, 8, 0.95, 8, 8, 32)]):
        b = sf.generate_synthetic(rows, cols, v, sp, seed, bit_width=bw)
        s = sf.bcrs_to_srbcrs(b, stride)
        p = f"gen{i}/"
        d[p + "args"] = np.array([rows, cols, v, int(sp * 1000), seed, bw, stride])
        d[p + "offsets"] = b.row_offsets
        d[p + "cols"] = b.col_indices
        d[p + "words"] = b.values.words
        srbcrs_arrays(p + "sr_", s, d)
        if stride % 8 == 0:
            d[p + "shuffled_cols"] = sf.shuffle_indices(s).col_indices
    # cell seed + safe magnitude KATs
    spec = rb.SweepSpec("spmm", [(512, 256, 512)])
    d["seed/c1"] = np.array([rb._cell_seed(spec, ((512, 256, 512), 8, 0.9, "L8-R8"))])
    mags = []
    for (lb, rbits) in SPMM_PAIRS:
        for k in (64, 128, 4096, 32768):
            mags.append((lb, rbits, k, *rb.safe_magnitudes(lb, rbits, k, em.SPMM)))
    d["safe_magnitudes"] = np.array(mags, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "formats.npz"), **d)

    # ---- SpMM ----
    d = {}
    for (lb, rbits) in SPMM_PAIRS:
        for v in (2, 4, 8):
            spmm_case(d, f"pair_{lb}_{rbits}_v{v}", seed=lb * 7 + rbits + v, v=v, lb=lb, rbits=rbits)
    for n in (40, 96, 200):
        spmm_case(d, f"ragged_n{n}", seed=n, n=n)
    for mult in (2, 4):
        spmm_case(d, f"stride_x{mult}", seed=11, sparsity=0.85, stride_mult=mult)
    spmm_case(d, "l8r4_stride64", seed=12, lb=8, rbits=4, stride_mult=2)
    spmm_case(d, "ablation_256x128x2304", seed=61, m=256, n=128, k=2304, v=8, sparsity=0.7)
    # config C1 (BASELINE configs[0]) with the bench cell seed
    c1_seed = rb._cell_seed(rb.SweepSpec("spmm", [(512, 256, 512)]),
                            ((512, 256, 512), 8, 0.9, "L8-R8"))
    spmm_case(d, "c1", seed=c1_seed, m=512, n=256, k=512, v=8, sparsity=0.9)
    np.savez_compressed(os.path.join(OUT, "spmm.npz"), **d)

    # ---- SDDMM ----
    d = {}
    for (lb, rbits) in SDDMM_PAIRS:
        for v in (2, 4, 8):
            sddmm_case(d, f"pair_{lb}_{rbits}_v{v}", seed=lb + v, v=v, lb=lb, rbits=rbits)
    sddmm_case(d, "random_64", seed=7, m=64, n=64, k=64, v=8, sparsity=0.9)
    sddmm_case(d, "ragged_k50", seed=8, k=50)
    sddmm_case(d, "srbcrs_out", seed=9, out_format="sr-bcrs")
    sddmm_case(d, "srbcrs_out_l4", seed=10, lb=4, rbits=4, out_format="sr-bcrs")
    sddmm_case(d, "k256", seed=13, m=64, n=128, k=256, v=8, sparsity=0.5)
    np.savez_compressed(os.path.join(OUT, "sddmm.npz"), **d)

    # ---- attention ----
    d = {}
    for sb, qb in ((16, 8), (8, 8), (8, 4)):
        for sp in (0.9, 0.95):
            attention_case(d, f"att_{sb}_{qb}_{int(sp * 100)}", 64, sb, qb, sp, seed=sb * 10 + qb)
    attention_case(d, "att_8_8_L128", 128, 8, 8, 0.9, seed=3)
    attention_case(d, "att_8_8_L256", 256, 8, 8, 0.9, seed=4)
    dmask = np.ones((32, 32), dtype=np.int64)
    dmask[8:16] = 0
    attention_case(d, "att_masked_rows", 32, 8, 8, 0.0, seed=5, head_dim=16, dense_mask=dmask)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **d)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
