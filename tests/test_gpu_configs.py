"""Device parity at the BASELINE.json configurations (C3, C4, C5) and for row-panel shards.

Every case builds its inputs with the reference generators (oracle.build_*_case =
bench._build_* semantics, bench.py:93-136), runs the default device dispatch through
the C ABI, and compares sampled vector rows / heads with the CPU oracle:

* C5  -- SpMM L8-R4, V=8, S=32, shuffled, M=K=32768, N=2048, 95 %: 64 sampled rows;
* C3  -- SpMM {L16-R16, L16-R8, L8-R8, L8-R4, L4-R4} x V in {2,4,8} x {70, 90, 98} % at
         M=K=4096, N=512: 16 sampled rows per cell;
* C4  -- 8-bit fused attention, L=4096, d=64, 90 % mask, 16 heads (B=2 x H=8): 3 sampled
         heads, parity mode bit-exact, fast mode within FAST_MODE_TOLERANCE;
* shards -- the north-star multi-GPU split (vector-row panels, batch x head) run
         sequentially on one GPU: the concatenated shard outputs equal the unsharded run
         bit-for-bit (the NCCL all-gather in bench.py only assembles these shards).
"""

import numpy as np
import pytest

import oracle as O
from conftest import cuda_available

pytestmark = pytest.mark.gpu

if cuda_available():
    import torch
    import paper_2209_06979_b200 as mc
    from paper_2209_06979_b200 import shard

C3_PAIRS = [(16, 16), (16, 8), (8, 8), (8, 4), (4, 4)]


def _device_problem(c, m, k, lb, rb):
    t = torch
    lhs = mc.SrBcrsMatrix(m, k, c["v"], c["stride"], t.from_numpy(c["row_begin"]).cuda(),
                          t.from_numpy(c["row_end"]).cuda(),
                          t.from_numpy(c["col_indices"].view(np.int32)).cuda(),
                          mc.PackedArray(c["values"].size, lb, True,
                                         t.from_numpy(mc.pack_values(c["values"], lb).view(np.int32)).cuda()),
                          shuffled=c["shuffled"])
    rhs = mc.PackedMatrix(k, c["n"], rb, mc.qint.ROW_MAJOR, True,
                          t.from_numpy(mc.pack_values(c["rhs"], rb).view(np.int32)).cuda())
    return mc.SpmmProblem(lhs, rhs)


def _check_rows(c, out, rows, lb, rb, k):
    v = c["v"]
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"],
                  c["shuffled"], lb, c["rhs"], rb, k, rows=rows)
    got = torch.cat([out[r * v:(r + 1) * v] for r in rows]).cpu().numpy()
    assert (got == want).all()


def test_c5_sampled_rows():
    m = k = 32768
    n = 2048
    seed = O.cell_seed(0, ((m, n, k), 8, 0.95, "L8-R4"))
    c = O.build_spmm_case(m, n, k, 8, 0.95, 8, 4, seed)
    assert c["stride"] == 32 and c["shuffled"]
    p = _device_problem(c, m, k, 8, 4)
    out = mc.spmm(p)
    rows = list(range(0, m // 8, 64))  # 64 vector rows spread over the 4096
    _check_rows(c, out, rows, 8, 4, k)


@pytest.mark.parametrize("sparsity", [0.7, 0.9, 0.98])
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("pair", C3_PAIRS)
def test_c3_grid_sampled_rows(pair, v, sparsity):
    lb, rb = pair
    m = k = 4096
    n = 512
    seed = O.cell_seed(0, ((m, n, k), v, sparsity, f"L{lb}-R{rb}"))
    c = O.build_spmm_case(m, n, k, v, sparsity, lb, rb, seed)
    out = mc.spmm(_device_problem(c, m, k, lb, rb))
    vr = m // v
    rows = sorted(set(list(range(0, vr, vr // 14)) + [vr - 1]))
    _check_rows(c, out, rows, lb, rb, k)


@pytest.mark.parametrize("mode", ["fast", "parity"])
def test_c4_attention_sampled_heads(mode):
    seq, d, heads, batch = 4096, 64, 8, 2
    seed = O.cell_seed(0, ((seq, d, heads), 8, 0.9, "L8-R8"))
    offs, cols, _ = O.synthetic_bcrs(seq, seq, 8, 0.9, seed, 8)
    mask = mc.BcrsMatrix(seq, seq, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(seq, 8, 8, mask, head_dim=d, num_heads=heads)
    nh = batch * heads
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, vv = (torch.randn((nh, seq, d), device="cuda", generator=g).half() for _ in range(3))
    run = mc.AttentionRunner(cfg, nh, mode=mode)
    out = run(q, k, vv, check=True)
    tol = mc.attention.FAST_MODE_TOLERANCE if mode == "fast" else 0.0
    for h in (0, 7, nh - 1):
        ref = O.attention(q[h].double().cpu().numpy(), k[h].double().cpu().numpy(),
                          vv[h].double().cpu().numpy(), offs, cols, seq, d, 8, 8)
        err = float(np.abs(out[h].double().cpu().numpy() - ref["output"]).max())
        assert err <= tol, (h, err)


@pytest.mark.parametrize("pair,v", [((8, 4), 8), ((16, 8), 4), ((8, 8), 2)])
def test_spmm_row_panel_shards_equal_unsharded(pair, v):
    lb, rb = pair
    m = k = 4096
    c = O.build_spmm_case(m, 512, k, v, 0.9, lb, rb, seed=77 + v)
    lhs = mc.SrBcrsMatrix(m, k, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
    rhs = mc.pack_dense(c["rhs"], rb)
    full = mc.spmm(mc.SpmmProblem(lhs, rhs))
    parts = shard.row_panels(lhs, 8)
    outs = [mc.spmm(mc.SpmmProblem(shard.srbcrs_panel(lhs, lo, hi), rhs)) for lo, hi in parts]
    assert (np.concatenate(outs) == full).all()


def test_sddmm_row_panel_shards_equal_unsharded():
    m = n = 4096
    c = O.build_sddmm_case(m, n, 256, 8, 0.9, 8, 8, seed=5)
    pat = mc.BcrsMatrix(m, n, 8, c["offsets"], c["col_indices"],
                        mc.PackedArray.from_values(np.ones(c["col_indices"].size * 8), 8))
    b = mc.pack_dense(c["b"], 8, mc.qint.COL_MAJOR)
    full = np.asarray(mc.sddmm(mc.SddmmProblem(mc.pack_dense(c["a"], 8, mc.qint.ROW_MAJOR), b, pat)).values)
    outs = []
    for lo, hi in shard.pattern_panels(pat, 8):
        sub = shard.bcrs_panel(pat, lo, hi)
        a = mc.pack_dense(c["a"][lo * 8:hi * 8], 8, mc.qint.ROW_MAJOR)
        outs.append(np.asarray(mc.sddmm(mc.SddmmProblem(a, b, sub)).values))
    assert (np.concatenate(outs) == full).all()


def test_attention_head_shards_equal_unsharded():
    seq, d, nh = 1024, 64, 12
    offs, cols, _ = O.synthetic_bcrs(seq, seq, 8, 0.9, 3, 8)
    mask = mc.BcrsMatrix(seq, seq, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(seq, 8, 8, mask, head_dim=d)
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, vv = (torch.randn((nh, seq, d), device="cuda", generator=g).half() for _ in range(3))
    full = mc.AttentionRunner(cfg, nh, mode="parity")(q, k, vv, check=True).clone()
    parts = []
    for lo, hi in shard.head_ranges(nh, 5):
        r = mc.AttentionRunner(cfg, hi - lo, mode="parity")
        parts.append(r(q[lo:hi].contiguous(), k[lo:hi].contiguous(), vv[lo:hi].contiguous(), check=True).clone())
    assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("prexor", ["1", "0"])
@pytest.mark.parametrize("sparsity", [0.5, 0.95])
@pytest.mark.parametrize("v", [2, 4, 8])
@pytest.mark.parametrize("pair,n", [((8, 4), 512), ((8, 4), 96), ((4, 4), 256), ((8, 8), 384), ((8, 8), 48),
                                    ((16, 8), 256)])
def test_spmm_segment_path_vs_oracle(pair, n, v, sparsity, prexor, monkeypatch):
    """The row-segment SpMM kernel (spmm_seg.cu, the C5 kernel) forced on small problems:
    every V, ragged N (zero-filled segment tails), empty / irregular rows; 4-bit right-hand
    sides with the pre-XORed workspace copy (mc_spmm_ws) and without it."""
    if prexor == "0" and pair[1] != 4:
        pytest.skip("the workspace variant exists for 4-bit right-hand sides only")
    monkeypatch.setenv("MCUBE_SPMM_PATH", "seg")
    monkeypatch.setenv("MCUBE_SEG_PREXOR", prexor)
    lb, rb = pair
    m, k = 256, 640
    c = O.build_spmm_case(m, n, k, v, sparsity, lb, rb, seed=lb + rb + v + n)
    lhs = mc.SrBcrsMatrix(m, k, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], rb)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"], c["shuffled"], lb,
                  c["rhs"], rb, k)
    assert (out == want).all()
    # irregular rows: empty, full, clustered (the device packer builds the SR-BCRS)
    rng = np.random.default_rng(v + n)
    lens = rng.integers(0, k // 3, m // v)
    lens[::5] = 0
    lens[1] = k
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, size=int(x), replace=False)) for x in lens]).astype(np.uint32)
    mag = min(c["values"].max(), 127)
    vals = rng.integers(-mag, mag + 1, cols.size * v)
    b = mc.BcrsMatrix(m, k, v, offs, cols, mc.PackedArray.from_values(vals, lb))
    sr = mc.bcrs_to_srbcrs(b, c["stride"])
    if rb == 4:
        sr = mc.shuffle_indices(sr)
    out = mc.spmm(mc.SpmmProblem(sr, mc.pack_dense(c["rhs"], rb)))
    want = O.spmm(sr.row_begin, sr.row_end, sr.col_indices, sr.values.to_values(), v, sr.stride, sr.shuffled, lb,
                  c["rhs"], rb, k)
    assert (out == want).all()


def _segment_case_extreme(m, k, n, lb, stride, seed, vmax):
    """Dense-ish rows with the extreme operand values the y' / h nibble decomposition has to
    keep exact: LHS at +-(2^(lb-1)-1) or -2^(lb-1), RHS nibbles over the whole range
    including -8 (sign bit of the low nibble set) and 7."""
    rng = np.random.default_rng(seed)
    v = 8
    vr = m // v
    lens = rng.integers(k // 2, k + 1, vr)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, size=int(x), replace=False)) for x in lens]).astype(np.uint32)
    lo, hi = -(1 << (lb - 1)), (1 << (lb - 1)) - 1
    vals = rng.choice(np.array([lo, hi, lo + 1, -1, 1, 0], dtype=np.int64), size=cols.size * v,
                      p=[0.35, 0.35, 0.1, 0.08, 0.07, 0.05]) if vmax else rng.integers(lo, hi + 1, cols.size * v)
    rhs = rng.choice(np.array([-8, 7, -7, -1, 0, 1], dtype=np.int64), size=(k, n), p=[0.3, 0.3, 0.1, 0.1, 0.1, 0.1])
    b = mc.BcrsMatrix(m, k, v, offs, cols, mc.PackedArray.from_values(vals, lb))
    sr = mc.shuffle_indices(mc.bcrs_to_srbcrs(b, stride))
    return sr, rhs


@pytest.mark.parametrize("prexor", ["1", "0"])
@pytest.mark.parametrize("lb,stride", [(8, 32), (4, 32)])
def test_spmm_segment_nibble_decomposition_extremes(lb, stride, prexor, monkeypatch):
    """The row-segment kernel feeds a 4-bit RHS byte y to two MMAs (y ^ 0x08 and y & 0xF0)
    and recovers the even column as acc(y') - acc(h) - 8 sum(a): exact at the extreme
    operand values and with long rows (|sums| up to ~K * 128 * 8), with and without the
    pre-XORed workspace copy."""
    monkeypatch.setenv("MCUBE_SPMM_PATH", "seg")
    monkeypatch.setenv("MCUBE_SEG_PREXOR", prexor)
    m, k, n = 128, 8192, 512
    sr, rhs = _segment_case_extreme(m, k, n, lb, stride, seed=lb + stride, vmax=True)
    out = np.asarray(mc.spmm(mc.SpmmProblem(sr, mc.pack_dense(rhs, 4))))
    want = O.spmm(sr.row_begin, sr.row_end, sr.col_indices, sr.values.to_values(), 8, stride, True, lb,
                  rhs, 4, k)
    assert (out == want).all()


def test_spmm_segment_path_declines_beyond_its_int32_bound():
    """|16 * sum| < 2^31 bounds the segment kernel's 4-bit forms: at K = 131104 (> 2^31 /
    (16 * 1024)) an L8-R4 problem must not take it, and still matches the oracle."""
    from paper_2209_06979_b200 import _device as Dv
    from paper_2209_06979_b200 import _native as Nn
    m, k, n = 64, 131104, 256
    rng = np.random.default_rng(11)
    vr = m // 8
    lens = rng.integers(1, 64, vr)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(k, size=int(x), replace=False)) for x in lens]).astype(np.uint32)
    vals = rng.integers(-127, 128, cols.size * 8)
    rhs = rng.integers(-8, 8, size=(k, n))
    b = mc.BcrsMatrix(m, k, 8, offs, cols, mc.PackedArray.from_values(vals, 8))
    sr = mc.shuffle_indices(mc.bcrs_to_srbcrs(b, 32))
    p = mc.SpmmProblem(sr, mc.pack_dense(rhs, 4))
    lhs_s, _k1 = Dv.srbcrs_struct(p.lhs)
    rhs_s, _k2 = Dv.dense_struct(p.rhs)
    pid = Nn.ctypes.c_int32(-1)
    Nn.check(Nn.lib().mc_spmm_path(lhs_s, rhs_s, Nn.ctypes.byref(pid)))
    assert pid.value != 1  # MC_SPMM_PATH_SEGMENT (include/mcube.h)
    out = np.asarray(mc.spmm(p))
    want = O.spmm(sr.row_begin, sr.row_end, sr.col_indices, sr.values.to_values(), 8, 32, True, 8, rhs, 4, k)
    assert (out == want).all()
