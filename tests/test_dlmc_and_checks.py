"""DLMC ingestion and the 4-bit-width per-nibble group check, pinned to the reference.

Fixtures (`tests/golden/extra.npz`, `tools/make_golden.py::extra_goldens`) come from the
reference's own bench builders (`bench.py:93-126`: `dilate` -> `bcrs_to_srbcrs` ->
`shuffle_indices` -> `kernels.spmm` / `kernels.sddmm`) on an irregular DLMC text, and
from the reference raising `OverflowRiskError` in its stacked-group check
(`tile_engine.py:246-247` via `kernels.py:265-275`) for an L16-R4 V=8 problem whose
final result fits int32.

CPU tests pin the host DLMC reader/dilation and the oracle; `-m gpu` tests run the
device packer + kernels through the C ABI.
"""

import io

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

X = load_golden("extra")
SPMM_CASES = sorted({k.split("/")[0] for k in X.files if k.startswith("dlmc_spmm_")})
SDDMM_CASES = sorted({k.split("/")[0] for k in X.files if k.startswith("dlmc_sddmm_")})


def _text(name):
    return X[name + "/text"].tobytes().decode()


def _mc():
    import paper_2209_06979_b200 as mc
    return mc


# ---------------- CPU: host DLMC reader, dilation and the oracle ----------------

def test_read_dlmc_tiny_matches_reference():
    mc = _mc()
    csr = mc.read_dlmc(_text("dlmc_tiny"))
    assert (csr.row_offsets == X["dlmc_tiny/offsets"]).all()
    assert (csr.col_indices == X["dlmc_tiny/cols"]).all()
    buf = io.StringIO()
    mc.write_dlmc(csr, buf)
    assert buf.getvalue() == _text("dlmc_tiny")


@pytest.mark.parametrize("name", SPMM_CASES)
def test_dlmc_dilate_pack_and_oracle_spmm(name):
    """read_dlmc -> dilate (seeded values, bench caps) -> SR-BCRS (+shuffle) equals the
    reference's arrays, and the oracle reproduces the reference's SpMM output."""
    mc = _mc()
    m, n, k, v, lb, rb, seed = [int(x) for x in X[name + "/args"]]
    csr = mc.read_dlmc(_text("dlmc_irr"))
    mag_l, mag_r = O.safe_magnitudes(lb, rb, 256, "spmm")
    b = mc.dilate(csr, v, value_seed=seed, bit_width=lb, max_magnitude=mag_l)
    assert (b.scalar_rows, b.scalar_cols) == (m, k)
    vals = b.values.to_values()
    stride = 16 if (lb % 8 == 0 and rb % 8 == 0) else 32
    beg, end, idx, sv = O.srbcrs_from_bcrs(b.row_offsets, b.col_indices, vals, v, stride)
    if rb == 4:
        idx = O.shuffle_idx(idx)
    p = name + "/lhs_"
    assert (beg == X[p + "row_begin"]).all() and (end == X[p + "row_end"]).all()
    assert (idx == X[p + "col_indices"]).all()
    assert (O.pack_bits(sv, lb) == X[p + "words"]).all()
    rhs = O.unpack_bits(X[name + "/rhs_words"], k * n, rb).reshape(k, n)
    out = O.spmm(beg, end, idx, sv, v, stride, rb == 4, lb, rhs, rb, k)
    assert (out == X[name + "/out"]).all()


@pytest.mark.parametrize("name", SDDMM_CASES)
def test_dlmc_pattern_and_oracle_sddmm(name):
    mc = _mc()
    m, n, k, v, lb, rb, seed = [int(x) for x in X[name + "/args"]]
    pat = mc.dilate(mc.read_dlmc(_text("dlmc_irr")), v, value_seed=seed, bit_width=8)
    assert (pat.row_offsets == X[name + "/offsets"]).all()
    assert (pat.col_indices == X[name + "/cols"]).all()
    a = O.unpack_bits(X[name + "/a_words"], m * k, lb).reshape(m, k)
    bt = O.unpack_bits(X[name + "/b_words"], k * n, rb).reshape(n, k)
    out = O.sddmm(a, bt.T, pat.row_offsets, pat.col_indices, v, lb, rb)
    assert (out == X[name + "/out"]).all()


def _nib_problem(name):
    aval, k = [int(x) for x in X[name + "/args"]]
    dense = np.full((8, k), aval, dtype=np.int64)
    rhs = np.full((k, 64), -8, dtype=np.int64)
    return dense, rhs, k


@pytest.mark.parametrize("name", ["nib_raise", "nib_ok"])
def test_oracle_nibble_group_check(name):
    dense, rhs, k = _nib_problem(name)
    offs = np.array([0, k])
    cols = np.arange(k, dtype=np.uint32)
    beg, end, idx, sv = O.srbcrs_from_bcrs(offs, cols, dense.T.reshape(-1), 8, 32)
    args = (beg, end, O.shuffle_idx(idx), sv, 8, 32, True, 16, rhs, 4, k)
    if int(X[name + "/raises"][0]):
        with pytest.raises(O.OracleOverflow):
            O.spmm(*args)
    else:
        assert (O.spmm(*args) == X[name + "/out"]).all()


# ---------------- GPU: the same cases through the device packer and kernels ----------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", SPMM_CASES)
def test_gpu_dlmc_spmm_matches_reference(name):
    mc = _mc()
    m, n, k, v, lb, rb, seed = [int(x) for x in X[name + "/args"]]
    mag_l, _ = O.safe_magnitudes(lb, rb, 256, "spmm")
    b = mc.dilate(mc.read_dlmc(_text("dlmc_irr")), v, value_seed=seed, bit_width=lb, max_magnitude=mag_l)
    stride = 16 if (lb % 8 == 0 and rb % 8 == 0) else 32
    lhs = mc.bcrs_to_srbcrs(b, stride)  # device packer
    if rb == 4:
        lhs = mc.shuffle_indices(lhs)  # device shuffle
    p = name + "/lhs_"
    assert (np.asarray(lhs.col_indices) == X[p + "col_indices"]).all()
    assert (np.asarray(lhs.values.words) == X[p + "words"]).all()
    rhs = mc.PackedMatrix(k, n, rb, mc.qint.ROW_MAJOR, True, X[name + "/rhs_words"])
    out = mc.spmm(mc.SpmmProblem(lhs, rhs))
    assert (out == X[name + "/out"]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", SDDMM_CASES)
def test_gpu_dlmc_sddmm_matches_reference(name):
    mc = _mc()
    m, n, k, v, lb, rb, seed = [int(x) for x in X[name + "/args"]]
    pat = mc.dilate(mc.read_dlmc(_text("dlmc_irr")), v, value_seed=seed, bit_width=8)
    a = mc.PackedMatrix(m, k, lb, mc.qint.ROW_MAJOR, True, X[name + "/a_words"])
    bm = mc.PackedMatrix(k, n, rb, mc.qint.COL_MAJOR, True, X[name + "/b_words"])
    out = mc.sddmm(mc.SddmmProblem(a, bm, pat))
    assert (np.asarray(out.values) == X[name + "/out"]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["nib_raise", "nib_ok"])
def test_gpu_nibble_group_check_like_reference(name):
    """L16-R4 V=8, K=9216: the device keeps per-nibble chunk accumulators and raises
    exactly when the reference's top-nibble group sum leaves int32."""
    mc = _mc()
    dense, rhs, k = _nib_problem(name)
    lhs = mc.shuffle_indices(mc.bcrs_to_srbcrs(mc.dense_to_bcrs(dense, 8, bit_width=16), 32))
    prob = mc.SpmmProblem(lhs, mc.pack_dense(rhs, 4))
    if int(X[name + "/raises"][0]):
        with pytest.raises(mc.OverflowRiskError):
            mc.spmm(prob)
    else:
        assert (mc.spmm(prob) == X[name + "/out"]).all()


@pytest.mark.gpu
@pytest.mark.parametrize("lb,k,v", [(16, 9216, 8), (16, 9216, 4), (12, 131104, 8), (8, 4096, 8)])
def test_gpu_nibble_chunk_path_exact(lb, k, v):
    """Random problems on both sides of the nibble-chunk threshold stay bit-exact."""
    mc = _mc()
    c = O.build_spmm_case(32, 64, k, v, 0.9 if k < 100000 else 0.999, lb, 4, seed=lb + v)
    lhs = mc.SrBcrsMatrix(32, k, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                          mc.PackedArray.from_values(c["values"], lb), shuffled=True)
    out = mc.spmm(mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], 4)))
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"], True,
                  lb, c["rhs"], 4, k)
    assert (out == want).all()

