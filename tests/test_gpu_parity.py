"""Device parity: CUDA path (through the C ABI) vs the reference's golden vectors and the oracle.

Integer results must be bit-exact; attention parity mode must reproduce the
reference's integer stages and fp16 output exactly; fast mode is checked
against the stated tolerance (max-abs 1e-3 on the fp16 output).
"""

import numpy as np
import pytest

import oracle as O
from conftest import cuda_available, golden_cases, load_golden

pytestmark = pytest.mark.gpu

if cuda_available():
    import torch
    import paper_2209_06979_b200 as mc
    from paper_2209_06979_b200.qint import COL_MAJOR, ROW_MAJOR

SPMM = load_golden("spmm")
SDDMM = load_golden("sddmm")
ATT = load_golden("attention")
FMT = load_golden("formats")


def _srbcrs_from_golden(g, prefix, device=False):
    rows, cols, v, stride, bits, shuffled = [int(x) for x in g[prefix + "meta"]]
    begin, end = g[prefix + "row_begin"], g[prefix + "row_end"]
    idx, words = g[prefix + "col_indices"], g[prefix + "words"]
    count = idx.size * v
    if device:
        begin, end = torch.from_numpy(begin).cuda(), torch.from_numpy(end).cuda()
        idx = torch.from_numpy(idx.view(np.int32)).cuda()
        words = torch.from_numpy(words.view(np.int32)).cuda()
    return mc.SrBcrsMatrix(rows, cols, v, stride, begin, end, idx,
                           mc.PackedArray(count, bits, True, words), shuffled=bool(shuffled))


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("name", golden_cases(SPMM))
def test_spmm_golden(name, device):
    m, n, k, v, sp, lb, rb, seed, mult = [int(x) for x in SPMM[name + "/args"]]
    lhs = _srbcrs_from_golden(SPMM, name + "/lhs_", device)
    words = SPMM[name + "/rhs_words"]
    if device:
        words = torch.from_numpy(words.view(np.int32)).cuda()
    rhs = mc.PackedMatrix(k, n, rb, ROW_MAJOR, True, words)
    out = mc.spmm(mc.SpmmProblem(lhs, rhs))
    if device:
        assert out.is_cuda and out.dtype == torch.int32
        out = out.cpu().numpy()
    assert out.dtype == np.int32
    assert (out == SPMM[name + "/out"]).all()


@pytest.mark.parametrize("name", ["pair_8_8_v8", "pair_16_4_v4"])
def test_spmm_pipelined_trace(name):
    lhs = _srbcrs_from_golden(SPMM, name + "/lhs_")
    m, n, k, v, sp, lb, rb, seed, mult = [int(x) for x in SPMM[name + "/args"]]
    rhs = mc.PackedMatrix(k, n, rb, ROW_MAJOR, True, SPMM[name + "/rhs_words"])
    out, traces = mc.spmm_pipelined(mc.SpmmProblem(lhs, rhs, mc.TilingConfig(pipeline=True)))
    assert (out == SPMM[name + "/out"]).all()
    steps = lhs.stored_count(0) // mc.plan(lb, rb).tile.k
    assert traces[0][1] == mc.alg1_trace(steps)


def test_spmm_epilogue_hook():
    name = "pair_8_8_v8"
    lhs = _srbcrs_from_golden(SPMM, name + "/lhs_")
    rhs = mc.PackedMatrix(128, 64, 8, ROW_MAJOR, True, SPMM[name + "/rhs_words"])
    out = mc.spmm(mc.SpmmProblem(lhs, rhs, epilogue=lambda acc: acc.astype(np.float64) * 0.5))
    assert out.dtype == np.float64
    assert (out == SPMM[name + "/out"] * 0.5).all()


@pytest.mark.parametrize("name", golden_cases(SDDMM))
def test_sddmm_golden(name):
    m, n, k, v, sp, lb, rb, seed, fmt = [int(x) for x in SDDMM[name + "/args"]]
    offs, cols = SDDMM[name + "/pattern_offsets"], SDDMM[name + "/pattern_cols"]
    pattern = mc.BcrsMatrix(m, n, v, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * v), 8))
    a = mc.PackedMatrix(m, k, lb, ROW_MAJOR, True, SDDMM[name + "/a_words"])
    b = mc.PackedMatrix(k, n, rb, COL_MAJOR, True, SDDMM[name + "/b_words"])
    out = mc.sddmm(mc.SddmmProblem(a, b, pattern, out_format="sr-bcrs" if fmt else "bcrs"))
    if fmt:
        assert isinstance(out, mc.SrBcrsMatrix) and out.stride == int(SDDMM[name + "/out_stride"][0])
        assert (out.col_indices == SDDMM[name + "/out_col_indices"]).all()
        assert (out.row_begin == SDDMM[name + "/out_row_begin"]).all()
    assert (np.asarray(out.values) == SDDMM[name + "/out_values"]).all()


@pytest.mark.parametrize("case", range(4))
def test_device_packer_and_shuffle(case):
    p = f"gen{case}/"
    rows, cols, v, sp, seed, bw, stride = [int(x) for x in FMT[p + "args"]]
    b = mc.BcrsMatrix(rows, cols, v, FMT[p + "offsets"], FMT[p + "cols"],
                      mc.PackedArray(FMT[p + "cols"].size * v, bw, True, FMT[p + "words"]))
    s = mc.bcrs_to_srbcrs(b, stride)
    assert (s.row_begin == FMT[p + "sr_row_begin"]).all()
    assert (s.row_end == FMT[p + "sr_row_end"]).all()
    assert (s.col_indices == FMT[p + "sr_col_indices"]).all()
    assert (s.values.words == FMT[p + "sr_words"]).all()
    if p + "shuffled_cols" in FMT.files:
        sh = mc.shuffle_indices(s)
        assert sh.shuffled and (sh.col_indices == FMT[p + "shuffled_cols"]).all()
        with pytest.raises(mc.ShuffleStateError):
            mc.shuffle_indices(sh)


@pytest.mark.parametrize("dtype", ["float64", "int64", "float32", "int32", "float16", "int16"])
@pytest.mark.parametrize("where", ["host", "device"])
def test_device_packer_keeps_raw_value_dtype(dtype, where):
    """Raw (unpacked) block values keep their dtype through the device packer, like the
    reference's values.astype(b.values.dtype) (sparse_format.py:303-304)."""
    offs, cols, _ = O.synthetic_bcrs(64, 96, 4, 0.8, 11, 8)
    rng = np.random.default_rng(5)
    vals = (rng.normal(size=cols.size * 4) * 1000).astype(dtype)
    b_host = mc.BcrsMatrix(64, 96, 4, offs, cols, vals)
    want_b, want_e, want_i, want_v = O.srbcrs_from_bcrs(offs, cols, vals, 4, 16)
    if where == "device":
        b = mc.BcrsMatrix(64, 96, 4, torch.from_numpy(offs).cuda(),
                          torch.from_numpy(cols.view(np.int32)).cuda(), torch.from_numpy(vals).cuda())
        s = mc.bcrs_to_srbcrs(b, 16)
        got = s.values.cpu().numpy()
    else:
        s = mc.bcrs_to_srbcrs(b_host, 16)
        got = np.asarray(s.values)
    assert got.dtype == np.dtype(dtype)
    assert (got.view(np.uint8) == want_v.astype(dtype).view(np.uint8)).all()


def test_packer_hand_layout_and_generator():
    d = FMT["hand_dense"]
    s = mc.bcrs_to_srbcrs(mc.dense_to_bcrs(d, 2), 4)
    assert list(s._flat_values) == [1, 3, 5, 0, 2, 4, 6, 0]
    assert (s.col_indices == FMT["hand_col_indices"]).all()
    assert (mc.srbcrs_to_dense(s) == d).all()


@pytest.mark.parametrize("name", golden_cases(ATT))
def test_attention_parity_golden(name):
    L, sb, qb, d, seed = [int(x) for x in ATT[name + "/args"]]
    offs, cols = ATT[name + "/mask_offsets"], ATT[name + "/mask_cols"]
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, sb, qb, mask, head_dim=d)
    q, k, v = (ATT[name + "/" + x].astype(np.float64) for x in "qkv")
    res = mc.sparse_attention(q, k, v, cfg, mode="parity")
    assert (res.scores_int == ATT[name + "/scores_int"]).all()
    assert (res.probs_int._flat_values == ATT[name + "/probs_int"]).all()
    assert (res.mix_int == ATT[name + "/mix_int"]).all()
    assert (res.output.astype(np.float16) == ATT[name + "/output"]).all()
    sc = ATT[name + "/scales"]
    assert [res.params[x].scale for x in ("q", "k", "v", "softmax")] == list(sc)


@pytest.mark.parametrize("name", ["att_8_8_90", "att_16_8_95", "att_8_4_90", "att_8_8_L256"])
def test_attention_fast_mode_tolerance(name):
    L, sb, qb, d, seed = [int(x) for x in ATT[name + "/args"]]
    offs, cols = ATT[name + "/mask_offsets"], ATT[name + "/mask_cols"]
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, sb, qb, mask, head_dim=d)
    q, k, v = (torch.from_numpy(ATT[name + "/" + x]).cuda() for x in "qkv")
    out = mc.batched_sparse_attention(q[None], k[None], v[None], cfg, mode="fast")[0]
    ref = ATT[name + "/output"].astype(np.float64)
    err = np.abs(out.double().cpu().numpy() - ref).max()
    assert err <= mc.attention.FAST_MODE_TOLERANCE, err


def test_multi_head_equals_single_head():
    a = O.build_attention_case(64, 16, 0.9, seed=11)
    mask = mc.BcrsMatrix(64, 64, 8, a["offsets"], a["col_indices"],
                         mc.PackedArray.from_values(np.ones(a["col_indices"].size * 8), 8))
    cfg = mc.AttentionConfig(64, 8, 8, mask, head_dim=16, num_heads=3)
    rng = np.random.default_rng(12)
    q, k, v = (rng.normal(size=(3, 64, 16)) for _ in range(3))
    out = mc.multi_head_attention(q, k, v, cfg)
    single = mc.sparse_attention(q[1], k[1], v[1], cfg)
    assert out.shape == (3, 64, 16)
    assert (out[1] == single.output).all()


# ---------------- randomized oracle sweeps (beyond the golden grid) ----------------

PAIRS = [(16, 16), (16, 8), (16, 4), (12, 4), (8, 4), (8, 8), (4, 4)]


@pytest.mark.parametrize("pair", PAIRS)
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("sparsity", [0.5, 0.9, 0.98])
def test_spmm_random_vs_oracle(pair, v, sparsity):
    lb, rb = pair
    c = O.build_spmm_case(128, 192, 512, v, sparsity, lb, rb, seed=lb * 100 + rb * 10 + v)
    lhs = mc.SrBcrsMatrix(128, 512, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], rb)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"],
                  c["shuffled"], lb, c["rhs"], rb, 512)
    assert (out == want).all()


@pytest.mark.parametrize("n", [1, 7, 33, 100, 130])
def test_spmm_unaligned_n_generic_path(n):
    c = O.build_spmm_case(32, n, 96, 8, 0.7, 8, 4, seed=n)
    lhs = mc.SrBcrsMatrix(32, 96, 8, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], 8), shuffled=True)
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], 4)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"], True,
                  8, c["rhs"], 4, 96)
    assert (out == want).all()


@pytest.mark.parametrize("pair", [(16, 16), (8, 8), (4, 4)])
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("k", [64, 100, 256])
def test_sddmm_random_vs_oracle(pair, v, k):
    lb, rb = pair
    s = O.build_sddmm_case(128, 256, k, v, 0.7, lb, rb, seed=k + v)
    pat = mc.BcrsMatrix(128, 256, v, s["offsets"], s["col_indices"],
                        mc.PackedArray.from_values(np.ones(s["col_indices"].size * v), 8))
    out = mc.sddmm(mc.SddmmProblem(mc.pack_dense(s["a"], lb, ROW_MAJOR),
                                   mc.pack_dense(s["b"], rb, COL_MAJOR), pat))
    want = O.sddmm(s["a"], s["b"], s["offsets"], s["col_indices"], v, lb, rb)
    assert (np.asarray(out.values) == want).all()


def test_spmm_overflow_raises_like_reference():
    # L16-R16, K=64, all values 32767: result 64*32767^2 > 2^31 -> OverflowRiskError
    d = np.full((8, 64), 32767, dtype=np.int64)
    lhs = mc.bcrs_to_srbcrs(mc.dense_to_bcrs(d, 8, bit_width=16), 16)
    rhs = mc.pack_dense(np.full((64, 64), 32767), 16)
    with pytest.raises(mc.OverflowRiskError):
        mc.spmm(mc.SpmmProblem(lhs, rhs))
    # the status word is reset: a good problem afterwards succeeds
    small = mc.pack_dense(np.ones((64, 64), dtype=np.int64), 16)
    lhs1 = mc.bcrs_to_srbcrs(mc.dense_to_bcrs(np.ones((8, 64), dtype=np.int64), 8, bit_width=16), 16)
    assert (mc.spmm(mc.SpmmProblem(lhs1, small)) == 64).all()


def test_sddmm_overflow_raises():
    pattern = mc.dense_to_bcrs(np.ones((8, 8), dtype=np.int64), 8)
    a = mc.pack_dense(np.full((8, 64), -32768), 16, ROW_MAJOR)
    b = mc.pack_dense(np.full((64, 8), -32768), 16, COL_MAJOR)
    with pytest.raises(mc.OverflowRiskError):
        mc.sddmm(mc.SddmmProblem(a, b, pattern))


def test_c3_full_size_rows_subset():
    """Config C3 shape (M=K=4096, N=512, 90%) L8-R8 V=8: check 24 rows against the oracle."""
    c = O.build_spmm_case(4096, 512, 4096, 8, 0.9, 8, 8, seed=3)
    lhs = mc.SrBcrsMatrix(4096, 4096, 8, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], 8))
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], 8)))
    rows = list(range(0, 512, 23))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"], False,
                  8, c["rhs"], 8, 4096, rows=rows)
    got = np.concatenate([out[r * 8:(r + 1) * 8] for r in rows])
    assert (got == want).all()


# ---------------- dense tcgen05 SDDMM path vs gather path ----------------

@pytest.mark.parametrize("path", ["dense", "gather"])
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("shape", [(512, 512, 256, 0.5), (1024, 640, 128, 0.9), (264, 300, 256, 0.7),
                                   (256, 128, 256, 0.98), (768, 512, 64, 0.8)])
def test_sddmm_paths_vs_oracle(path, v, shape, monkeypatch):
    m, n, k, sp = shape
    monkeypatch.setenv("MCUBE_SDDMM_PATH", path)
    s = O.build_sddmm_case(m, n, k, v, sp, 8, 8, seed=m + n + v)
    pat = mc.BcrsMatrix(m, n, v, s["offsets"], s["col_indices"],
                        mc.PackedArray.from_values(np.ones(s["col_indices"].size * v), 8))
    out = mc.sddmm(mc.SddmmProblem(mc.pack_dense(s["a"], 8, ROW_MAJOR), mc.pack_dense(s["b"], 8, COL_MAJOR), pat))
    want = O.sddmm(s["a"], s["b"], s["offsets"], s["col_indices"], v, 8, 8)
    assert (np.asarray(out.values) == want).all()


def test_sddmm_dense_c2_full_size(monkeypatch):
    """C2 at 50% through the tcgen05 path, checked on sampled rows against the oracle."""
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "dense")
    s = O.build_sddmm_case(4096, 4096, 256, 8, 0.5, 8, 8, seed=5)
    pat = mc.BcrsMatrix(4096, 4096, 8, s["offsets"], s["col_indices"],
                        mc.PackedArray.from_values(np.ones(s["col_indices"].size * 8), 8))
    out = np.asarray(mc.sddmm(mc.SddmmProblem(mc.pack_dense(s["a"], 8, ROW_MAJOR),
                                              mc.pack_dense(s["b"], 8, COL_MAJOR), pat)).values)
    offs = s["offsets"]
    for r in list(range(0, 512, 37)) + [511]:
        lo, hi = int(offs[r]), int(offs[r + 1])
        want = O.sddmm(s["a"][r * 8:(r + 1) * 8], s["b"], np.array([0, hi - lo]), s["col_indices"][lo:hi],
                       8, 8, 8)
        assert (out[lo * 8:hi * 8] == want).all(), r


def _irregular_pattern(m, n, v, seed):
    """Rows with skewed column distributions: empty rows, full rows, clustered rows
    (defeats the interpolation probe of the dense path and exercises its fallback)."""
    rng = np.random.default_rng(seed)
    offs, cols = [0], []
    for r in range(m // v):
        kind = r % 5
        if kind == 0:
            c = np.array([], dtype=np.int64)
        elif kind == 1:
            c = np.arange(n)
        elif kind == 2:  # clustered at the start
            c = np.arange(min(n, 3 + r % 97))
        elif kind == 3:  # clustered at the end
            c = np.arange(max(0, n - 5 - r % 211), n)
        else:
            c = np.sort(rng.choice(n, size=int(rng.integers(0, n)), replace=False))
        cols.append(c.astype(np.uint32))
        offs.append(offs[-1] + c.size)
    return np.array(offs, dtype=np.int64), np.concatenate(cols) if cols else np.zeros(0, np.uint32)


@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("shape", [(1024, 2048, 256), (768, 1000, 128), (2048, 384, 256)])
def test_sddmm_dense_irregular_rows(v, shape, monkeypatch):
    m, n, k = shape
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "dense")
    rng = np.random.default_rng(m + n + k + v)
    offs, cols = _irregular_pattern(m, n, v, m + v)
    a = rng.integers(-128, 128, size=(m, k))
    b = rng.integers(-128, 128, size=(k, n))
    pat = mc.BcrsMatrix(m, n, v, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * v), 8))
    out = mc.sddmm(mc.SddmmProblem(mc.pack_dense(a, 8, ROW_MAJOR), mc.pack_dense(b, 8, COL_MAJOR), pat))
    want = O.sddmm(a, b, offs, cols, v, 8, 8)
    assert (np.asarray(out.values) == want).all()


@pytest.mark.parametrize("sparsity", [0.5, 0.7, 0.9, 0.95, 0.98])
def test_sddmm_dense_c2_all_rows(sparsity, monkeypatch):
    """Every C2 sparsity through the tcgen05 path, all rows against the oracle."""
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "dense")
    s = O.build_sddmm_case(4096, 4096, 256, 8, sparsity, 8, 8, seed=11)
    pat = mc.BcrsMatrix(4096, 4096, 8, s["offsets"], s["col_indices"],
                        mc.PackedArray.from_values(np.ones(s["col_indices"].size * 8), 8))
    out = np.asarray(mc.sddmm(mc.SddmmProblem(mc.pack_dense(s["a"], 8, ROW_MAJOR),
                                              mc.pack_dense(s["b"], 8, COL_MAJOR), pat)).values)
    want = O.sddmm(s["a"], s["b"], s["offsets"], s["col_indices"], 8, 8, 8)
    assert (out == want).all()


@pytest.mark.parametrize("v", [4, 8])
def test_sddmm_dense_batched_with_f16_epilogue(v, monkeypatch):
    """mc_sddmm_batched on the tcgen05 path: 3 items sharing one pattern, int32 + fp16 outputs."""
    import torch
    from paper_2209_06979_b200 import _native as Nn
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "dense")
    m, n, k, batch = 640, 896, 128, 3
    s = O.build_sddmm_case(m, n, k, v, 0.8, 8, 8, seed=21)
    offs, cols = s["offsets"], s["col_indices"]
    rng = np.random.default_rng(3)
    a = rng.integers(-128, 128, size=(batch, m, k)).astype(np.int8)
    bt = rng.integers(-128, 128, size=(batch, n, k)).astype(np.int8)  # B^T row-major = B col-major
    dev = torch.device("cuda", 0)
    a_d = torch.from_numpy(a.reshape(-1).view(np.int32).copy()).to(dev)
    b_d = torch.from_numpy(bt.reshape(-1).view(np.int32).copy()).to(dev)
    o_d = torch.from_numpy(offs.astype(np.int64)).to(dev)
    c_d = torch.from_numpy(cols.astype(np.uint32).view(np.int32)).to(dev)
    nblk = cols.size
    out = torch.empty(batch * nblk * v, dtype=torch.int32, device=dev)
    out16 = torch.empty(batch * nblk * v, dtype=torch.float16, device=dev)
    alpha = torch.tensor([0.25, 1.0 / 3.0, 1e-3], dtype=torch.float64, device=dev)
    ad = Nn.McDense(m, k, 8, Nn.MC_ROW_MAJOR, Nn.ptr(a_d))
    bd = Nn.McDense(k, n, 8, Nn.MC_COL_MAJOR, Nn.ptr(b_d))
    pd = Nn.McBcrs(m, n, v, 0, nblk, Nn.ptr(o_d), Nn.ptr(c_d))
    epi = Nn.McEpilogue(Nn.ptr(alpha), 0.0, Nn.ptr(out16), nblk * v)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = Nn.lib()
    Nn.check(lib.mc_sddmm_batched(ad, m * k // 4, bd, n * k // 4, pd, batch, epi, Nn.ptr(out), nblk * v,
                                  Nn.ptr(status), Nn.stream_ptr()))
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    got = out.view(batch, -1).cpu().numpy()
    got16 = out16.view(batch, -1).cpu().numpy()
    for i in range(batch):
        want = O.sddmm(a[i].astype(np.int64), bt[i].T.astype(np.int64), offs, cols, v, 8, 8)
        assert (got[i] == want).all(), i
        w16 = (want.astype(np.float64) * float(alpha[i])).astype(np.float16)
        assert (got16[i].view(np.uint16) == w16.view(np.uint16)).all(), i


# ---------------- tcgen05 SpMM path (gather4 + MN-major UMMA) vs the oracle ----------------

def _spmm_irregular(m, k, v, seed, stride):
    """SR-BCRS with empty, full, clustered and random rows (8-bit values)."""
    rng = np.random.default_rng(seed)
    offs, cols = _irregular_pattern(m, k, v, seed)
    vals = rng.integers(-127, 128, size=cols.size * v)
    vals[vals == 0] = 1
    begin, end, sidx, svals = O.srbcrs_from_bcrs(offs, cols, vals, v, stride)
    return begin, end, sidx, svals


@pytest.mark.parametrize("path", ["tc", "mma"])
@pytest.mark.parametrize("shape", [(512, 256, 512, 0.9, 1), (1024, 384, 2048, 0.7, 1), (256, 512, 4096, 0.98, 2),
                                   (768, 144, 1024, 0.5, 4)])
def test_spmm_l8r8_paths_vs_oracle(path, shape, monkeypatch):
    m, n, k, sp, smult = shape
    monkeypatch.setenv("MCUBE_SPMM_PATH", path)
    c = O.build_spmm_case(m, n, k, 8, sp, 8, 8, seed=m + n + smult, stride_mult=smult)
    lhs = mc.SrBcrsMatrix(m, k, 8, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], 8))
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], 8)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"], False,
                  8, c["rhs"], 8, n)
    assert (np.asarray(out) == want).all()


@pytest.mark.parametrize("gather", ["cpasync", "tma"])
@pytest.mark.parametrize("stride", [16, 32])
def test_spmm_tc_irregular_rows(stride, gather, monkeypatch):
    monkeypatch.setenv("MCUBE_SPMM_PATH", "tc")
    monkeypatch.setenv("MCUBE_SPMM_GATHER", "tma" if gather == "tma" else "cp")
    m, n, k = 640, 256, 1536
    begin, end, sidx, svals = _spmm_irregular(m, k, 8, 5 + stride, stride)
    rng = np.random.default_rng(9)
    rhs = rng.integers(-127, 128, size=(k, n))
    lhs = mc.SrBcrsMatrix(m, k, 8, stride, begin, end, sidx, mc.PackedArray.from_values(svals, 8))
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(rhs, 8)))
    want = O.spmm(begin, end, sidx, svals, 8, stride, False, 8, rhs, 8, n)
    assert (np.asarray(out) == want).all()


# ---------------- dense-tile SpMM (densify + exact tcgen05 GEMM) vs the oracle ----------------

@pytest.mark.parametrize("pair", PAIRS)
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("sparsity", [0.5, 0.9, 0.98])
def test_spmm_dense_path_vs_oracle(pair, v, sparsity, monkeypatch):
    lb, rb = pair
    monkeypatch.setenv("MCUBE_SPMM_PATH", "dense")
    m, n, k = 256, 256, 512
    c = O.build_spmm_case(m, n, k, v, sparsity, lb, rb, seed=lb * 100 + rb + v + int(sparsity * 100))
    lhs = mc.SrBcrsMatrix(m, k, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], rb)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"],
                  c["shuffled"], lb, c["rhs"], rb, n)
    assert (np.asarray(out) == want).all()


@pytest.mark.parametrize("cluster", ["0", "1"])
def test_spmm_dense_path_irregular_and_c3_rows(cluster, monkeypatch):
    """Irregular rows (empty / full / clustered) and a C3-size L8-R8 problem on the dense path
    (persistent GEMM and the 4-CTA multicast-cluster variant)."""
    monkeypatch.setenv("MCUBE_SPMM_PATH", "dense")
    monkeypatch.setenv("MCUBE_GEMM_CLUSTER", cluster)
    m, n, k = 640, 256, 1536
    begin, end, sidx, svals = _spmm_irregular(m, k, 8, 77, 16)
    rhs = np.random.default_rng(4).integers(-127, 128, size=(k, n))
    lhs = mc.SrBcrsMatrix(m, k, 8, 16, begin, end, sidx, mc.PackedArray.from_values(svals, 8))
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(rhs, 8)))
    assert (np.asarray(out) == O.spmm(begin, end, sidx, svals, 8, 16, False, 8, rhs, 8, n)).all()
    c = O.build_spmm_case(4096, 512, 4096, 8, 0.9, 8, 8, seed=3)
    lhs = mc.SrBcrsMatrix(4096, 4096, 8, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], 8))
    out = np.asarray(mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], 8))))
    rows = list(range(0, 512, 41)) + [511]
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"], False,
                  8, c["rhs"], 8, 4096, rows=rows)
    got = np.concatenate([out[r * 8:(r + 1) * 8] for r in rows])
    assert (got == want).all()


# ---------------- fused score + softmax kernel (8-bit, d = 64) ----------------

@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("L,sparsity", [(512, 0.9), (1024, 0.5), (768, 0.98)])
def test_attention_fused_matches_unfused_and_oracle(mode, L, sparsity, monkeypatch):
    """The fused kernel (no stage outputs requested; P x V folded in) equals the score/softmax-only
    fused kernel + SpMM and the unfused pipeline bit for bit
    and the oracle (parity: exact; fast: within FAST_MODE_TOLERANCE). L=1024 at 50 % has rows
    longer than the kernel's 512-block cache (recompute path)."""
    import torch
    d, heads = 64, 3
    a = O.build_attention_case(L, d, sparsity, seed=L + int(sparsity * 100))
    offs, cols = a["offsets"], a["col_indices"]
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, 8, 8, mask, head_dim=d, num_heads=heads)
    g = torch.Generator(device="cuda").manual_seed(L)
    q, k, v = (torch.randn((heads, L, d), device="cuda", generator=g).half() for _ in range(3))
    fused = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    monkeypatch.setenv("MCUBE_ATTN_NOMIX", "1")  # fused scores/softmax + separate SpMM
    nomix = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    assert torch.equal(fused, nomix)
    monkeypatch.setenv("MCUBE_ATTN_UNFUSED", "1")
    unfused = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    assert torch.equal(fused, unfused)
    for h in range(heads):
        qh, kh, vh = (x[h].double().cpu().numpy() for x in (q, k, v))
        ref = O.attention(qh, kh, vh, offs, cols, L, d, 8, 8)
        err = float(np.abs(fused[h].double().cpu().numpy() - ref["output"]).max())
        assert err <= (0.0 if mode == "parity" else mc.attention.FAST_MODE_TOLERANCE), (h, err)


@pytest.mark.parametrize("pair", [(8, 8), (16, 8), (8, 4)])
def test_spmm_dense_path_k_beyond_one_densify_chunk(pair, monkeypatch):
    """K = 8448 > 4096: the densify kernel covers each vector row in several column chunks."""
    lb, rb = pair
    monkeypatch.setenv("MCUBE_SPMM_PATH", "dense")
    m, n, k = 256, 128, 8448
    c = O.build_spmm_case(m, n, k, 8, 0.8, lb, rb, seed=k + lb + rb)
    lhs = mc.SrBcrsMatrix(m, k, 8, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], rb)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"],
                  c["shuffled"], lb, c["rhs"], rb, n)
    assert (np.asarray(out) == want).all()


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_attention_long_sequence_streams_quant_slices(mode):
    """L = 8192: each quantisation CTA's slice (8 per tensor) exceeds its register tile, so the
    streaming second pass of absquant_f16_kernel runs; the fused kernel's rows (1638 blocks at
    80 %) exceed its shared-memory cache (recompute path)."""
    import torch
    L, d, heads, sp = 8192, 64, 1, 0.8
    a = O.build_attention_case(L, d, sp, seed=8192)
    offs, cols = a["offsets"], a["col_indices"]
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, 8, 8, mask, head_dim=d, num_heads=heads)
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn((heads, L, d), device="cuda", generator=g).half() for _ in range(3))
    out = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    qh, kh, vh = (x[0].double().cpu().numpy() for x in (q, k, v))
    ref = O.attention(qh, kh, vh, offs, cols, L, d, 8, 8)
    err = float(np.abs(out[0].double().cpu().numpy() - ref["output"]).max())
    assert err <= (0.0 if mode == "parity" else mc.attention.FAST_MODE_TOLERANCE), err


@pytest.mark.parametrize("v", [4, 8])
@pytest.mark.parametrize("shape", [(1024, 2048, 256), (768, 1000, 128)])
def test_sddmm_dense_16_row_tiles(v, shape, monkeypatch):
    """The tcgen05 SDDMM with 16-vector-row tiles (MCUBE_SDDMM_VR=16): UMMA N = 16 V, half
    the builder warps active, irregular rows."""
    m, n, k = shape
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "dense")
    monkeypatch.setenv("MCUBE_SDDMM_VR", "16")
    rng = np.random.default_rng(m + n + k + v + 16)
    offs, cols = _irregular_pattern(m, n, v, m + v + 16)
    a = rng.integers(-128, 128, size=(m, k))
    b = rng.integers(-128, 128, size=(k, n))
    pat = mc.BcrsMatrix(m, n, v, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * v), 8))
    out = mc.sddmm(mc.SddmmProblem(mc.pack_dense(a, 8, ROW_MAJOR), mc.pack_dense(b, 8, COL_MAJOR), pat))
    want = O.sddmm(a, b, offs, cols, v, 8, 8)
    assert (np.asarray(out.values) == want).all()


@pytest.mark.parametrize("gpw", ["2", "3"])
@pytest.mark.parametrize("pair", [(8, 8), (16, 16), (4, 4)])
def test_sddmm_gather_several_groups_per_warp(gpw, pair, monkeypatch):
    """Gather SDDMM with 2-3 groups of 16 blocks per warp (MCUBE_SDDMM_GPW), irregular rows."""
    lb, rb = pair
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "gather")
    monkeypatch.setenv("MCUBE_SDDMM_GPW", gpw)
    m, n, k, v = 512, 1536, 128, 8
    rng = np.random.default_rng(lb * 100 + rb + int(gpw))
    offs, cols = _irregular_pattern(m, n, v, 77 + int(gpw))
    lim = min((1 << (lb - 1)) - 1, 1000), min((1 << (rb - 1)) - 1, 1000)  # no int32 overflow at K=128
    a = rng.integers(-lim[0], lim[0] + 1, size=(m, k))
    b = rng.integers(-lim[1], lim[1] + 1, size=(k, n))
    pat = mc.BcrsMatrix(m, n, v, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * v), 8))
    out = mc.sddmm(mc.SddmmProblem(mc.pack_dense(a, lb, ROW_MAJOR), mc.pack_dense(b, rb, COL_MAJOR), pat))
    want = O.sddmm(a, b, offs, cols, v, lb, rb)
    assert (np.asarray(out.values) == want).all()


@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("bits", [(16, 8), (8, 4)])
def test_attention_runner_other_precisions(mode, bits, monkeypatch):
    """AttentionRunner on fp16 device inputs for (sb, qb) = (16, 8) (fused scores/softmax with
    16-bit SR-BCRS probabilities + L16-R8 SpMM) and (8, 4) (unfused 4-bit pipeline), vs oracle."""
    import torch
    sb, qb = bits
    L, d, heads, sp = 512, 64, 2, 0.9
    a = O.build_attention_case(L, d, sp, seed=sb * 10 + qb)
    offs, cols = a["offsets"], a["col_indices"]
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, sb, qb, mask, head_dim=d, num_heads=heads)
    g = torch.Generator(device="cuda").manual_seed(sb + qb)
    q, k, v = (torch.randn((heads, L, d), device="cuda", generator=g).half() for _ in range(3))
    out = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    for h in range(heads):
        qh, kh, vh = (x[h].double().cpu().numpy() for x in (q, k, v))
        ref = O.attention(qh, kh, vh, offs, cols, L, d, sb, qb)
        err = float(np.abs(out[h].double().cpu().numpy() - ref["output"]).max())
        assert err <= (0.0 if mode == "parity" else mc.attention.FAST_MODE_TOLERANCE), (h, err)


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_attention_fused_irregular_mask_rows(mode):
    """The two-kernel C4 path on a mask whose vector rows hold 0, 1, ..., 480 (the fused
    kernel's cache), 481 and up to all 2048 blocks: empty rows give 0, long rows recompute."""
    import torch
    L, d, heads = 2048, 64, 2
    rng = np.random.default_rng(2048)
    lens = [0, 1, 5, 31, 32, 33, 100, 479, 480, 481, 1000, 2048]
    offs, cols = [0], []
    for r in range(L // 8):
        n = lens[r % len(lens)]
        c = np.sort(rng.choice(L, size=n, replace=False)).astype(np.uint32)
        cols.append(c)
        offs.append(offs[-1] + n)
    offs = np.array(offs, dtype=np.int64)
    cols = np.concatenate(cols)
    mask = mc.BcrsMatrix(L, L, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(L, 8, 8, mask, head_dim=d, num_heads=heads)
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((heads, L, d), device="cuda", generator=g).half() for _ in range(3))
    out = mc.AttentionRunner(cfg, heads, mode=mode)(q, k, v, check=True).clone()
    for h in range(heads):
        qh, kh, vh = (x[h].double().cpu().numpy() for x in (q, k, v))
        ref = O.attention(qh, kh, vh, offs, cols, L, d, 8, 8)
        got = out[h].double().cpu().numpy()
        assert (got[:8] == 0).all()  # vector row 0 is empty
        err = float(np.abs(got - ref["output"]).max())
        assert err <= (0.0 if mode == "parity" else mc.attention.FAST_MODE_TOLERANCE), (h, err)


# ---------------- pipelined 8-bit gather SDDMM (sddmm_g8_kernel) ----------------

def _sddmm_path_id(a, b, pat):
    from paper_2209_06979_b200 import _device as D
    from paper_2209_06979_b200 import _native as Nn
    ad, _k1 = D.dense_struct(a)
    bd, _k2 = D.dense_struct(b)
    pd, _k3 = D.bcrs_struct(pat)
    pid = Nn.ctypes.c_int32(-1)
    Nn.check(Nn.lib().mc_sddmm_path(ad, bd, pd, Nn.ctypes.byref(pid)))
    return pid.value


@pytest.mark.gpu
@pytest.mark.parametrize("splits", ["1", "2", "3", "5"])
@pytest.mark.parametrize("v", [4, 8])
@pytest.mark.parametrize("k", [64, 128, 192, 256])
def test_sddmm_g8_irregular_rows_vs_oracle(splits, v, k, monkeypatch):
    """Pipelined 8-bit gather kernel on irregular rows (empty, full, clustered, random), with
    1-5 warps per vector row (odd / even group counts per warp, pairs and single tails)."""
    monkeypatch.setenv("MCUBE_SDDMM_PATH", "gather")
    monkeypatch.setenv("MCUBE_SDDMM_SPLITS", splits)
    m, n = 384, 1100
    rng = np.random.default_rng(k + v + int(splits))
    offs, cols = _irregular_pattern(m, n, v, 5 + k + v)
    a = rng.integers(-128, 128, size=(m, k))
    b = rng.integers(-128, 128, size=(k, n))
    pat = mc.BcrsMatrix(m, n, v, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * v), 8))
    pa, pb = mc.pack_dense(a, 8, ROW_MAJOR), mc.pack_dense(b, 8, COL_MAJOR)
    assert _sddmm_path_id(pa, pb, pat) == 2
    out = mc.sddmm(mc.SddmmProblem(pa, pb, pat))
    assert (np.asarray(out.values) == O.sddmm(a, b, offs, cols, v, 8, 8)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("sparsity", [0.9, 0.95, 0.98])
def test_sddmm_c2_sparse_cells_default_path_all_rows(sparsity):
    """C2 cells at 90/95/98 % on the default dispatch (the pipelined gather kernel), all rows."""
    s = O.build_sddmm_case(4096, 4096, 256, 8, sparsity, 8, 8, seed=13)
    pat = mc.BcrsMatrix(4096, 4096, 8, s["offsets"], s["col_indices"],
                        mc.PackedArray.from_values(np.ones(s["col_indices"].size * 8), 8))
    pa, pb = mc.pack_dense(s["a"], 8, ROW_MAJOR), mc.pack_dense(s["b"], 8, COL_MAJOR)
    assert _sddmm_path_id(pa, pb, pat) == 2
    out = np.asarray(mc.sddmm(mc.SddmmProblem(pa, pb, pat)).values)
    assert (out == O.sddmm(s["a"], s["b"], s["offsets"], s["col_indices"], 8, 8, 8)).all()


@pytest.mark.gpu
def test_sddmm_g8_batched_and_bad_index():
    """mc_sddmm_batched through the pipelined gather kernel (3 items sharing one pattern),
    then an out-of-range column index: flagged, reported as FormatError by mc_status_fetch."""
    import torch
    from paper_2209_06979_b200 import _native as Nn
    m, n, k, v, batch = 256, 512, 128, 8, 3
    s = O.build_sddmm_case(m, n, k, v, 0.95, 8, 8, seed=31)
    offs, cols = s["offsets"], s["col_indices"].astype(np.uint32)
    rng = np.random.default_rng(9)
    a = rng.integers(-128, 128, size=(batch, m, k)).astype(np.int8)
    bt = rng.integers(-128, 128, size=(batch, n, k)).astype(np.int8)
    dev = torch.device("cuda", 0)
    a_d = torch.from_numpy(a.reshape(-1).view(np.int32).copy()).to(dev)
    b_d = torch.from_numpy(bt.reshape(-1).view(np.int32).copy()).to(dev)
    o_d = torch.from_numpy(offs.astype(np.int64)).to(dev)
    c_d = torch.from_numpy(cols.view(np.int32).copy()).to(dev)
    nblk = cols.size
    out = torch.zeros(batch * nblk * v, dtype=torch.int32, device=dev)
    ad = Nn.McDense(m, k, 8, Nn.MC_ROW_MAJOR, Nn.ptr(a_d))
    bd = Nn.McDense(k, n, 8, Nn.MC_COL_MAJOR, Nn.ptr(b_d))
    pd = Nn.McBcrs(m, n, v, 0, nblk, Nn.ptr(o_d), Nn.ptr(c_d))
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = Nn.lib()
    pid = Nn.ctypes.c_int32(-1)
    Nn.check(lib.mc_sddmm_path(ad, bd, pd, Nn.ctypes.byref(pid)))
    assert pid.value == 2
    Nn.check(lib.mc_sddmm_batched(ad, m * k // 4, bd, n * k // 4, pd, batch, None, Nn.ptr(out), nblk * v,
                                  Nn.ptr(status), Nn.stream_ptr()))
    Nn.check(lib.mc_status_fetch(Nn.ptr(status), Nn.stream_ptr()))
    got = out.view(batch, -1).cpu().numpy()
    for i in range(batch):
        assert (got[i] == O.sddmm(a[i].astype(np.int64), bt[i].T.astype(np.int64), offs, cols, v, 8, 8)).all(), i
    c_d[nblk // 2] = n + 7  # out of range
    Nn.check(lib.mc_sddmm(ad, bd, pd, Nn.ptr(out), Nn.ptr(status), Nn.stream_ptr()))
    with pytest.raises(mc.FormatError):
        Nn.check(lib.mc_status_fetch(Nn.ptr(status), Nn.stream_ptr()))
