"""CPU tests: the drop-in host API (validation, errors, formats, plans) and the C-ABI library.

No kernel is launched here (no GPU in the build container); the library is
only loaded and its exported symbols checked against include/mcube.h.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2209_06979_b200 as mc
from paper_2209_06979_b200 import _native
from paper_2209_06979_b200.qint import COL_MAJOR, ROW_MAJOR
from conftest import ROOT, load_golden

FMT = load_golden("formats")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "mcube.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t)\s+(mc_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native._SIGNATURES), "ctypes signatures out of sync with mcube.h"
    assert lib.mc_version() == 1


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("bits", [4, 8, 12, 16])
def test_pack_matches_reference(bits):
    vals = FMT[f"pack{bits}/values"]
    assert (mc.pack_values(vals, bits) == FMT[f"pack{bits}/words"]).all()
    assert (mc.unpack_values(FMT[f"pack{bits}/words"], vals.size, bits) == vals).all()


def test_pack_kats_and_ranges():
    assert mc.pack_values([-19], 8)[0] == 0xED
    assert mc.split_signed(-19, 4, 2).chunks == (13, -2)
    assert mc.split_unsigned(237, 4, 2).chunks == (13, 14)
    with pytest.raises(ValueError):
        mc.pack_values([8], 4)
    with pytest.raises(ValueError):
        mc.pack_values([1], 5)
    for v in range(-128, 128):
        d = mc.split_signed(v, 4, 2)
        assert d.recombine() == v


@pytest.mark.parametrize("case", range(4))
def test_generator_reproduces_reference(case):
    p = f"gen{case}/"
    rows, cols, v, sp, seed, bw, stride = [int(x) for x in FMT[p + "args"]]
    b = mc.generate_synthetic(rows, cols, v, sp / 1000, seed, bit_width=bw)
    assert (b.row_offsets == FMT[p + "offsets"]).all()
    assert (b.col_indices == FMT[p + "cols"]).all()
    assert (b.values.words == FMT[p + "words"]).all()


def test_plan_table():
    assert mc.plan(16, 16).weights == (1, 256, 256, 65536)
    assert mc.plan(8, 4).native_width == 4 and mc.plan(8, 4).lhs_chunks == 2
    assert mc.plan(16, 8).device_chunk_products == 2
    assert mc.plan(8, 4).device_chunk_products == 1
    with pytest.raises(mc.UnsupportedPrecisionError):
        mc.plan(16, 8, "sddmm")
    with pytest.raises(mc.OverflowRiskError):
        mc.check_accumulation_bound(40000, 8)
    assert mc.parse_precision("l8-r4") == (8, 4)


def _lhs(v=8, bits=8, shuffled=False):
    c = O.build_spmm_case(16, 32, 64, v, 0.5, bits, 4 if bits == 4 else 8, seed=1)
    return mc.SrBcrsMatrix(16, 64, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                           mc.PackedArray.from_values(c["values"], bits), shuffled=shuffled)


def test_spmm_problem_validation_mirrors_reference():
    lhs = _lhs()
    rhs = mc.pack_dense(np.zeros((64, 32), dtype=np.int64), 8)
    mc.SpmmProblem(lhs, rhs)
    with pytest.raises(ValueError, match="row-major"):
        mc.SpmmProblem(lhs, mc.pack_dense(np.zeros((64, 32), dtype=np.int64), 8, COL_MAJOR))
    with pytest.raises(ValueError, match="K mismatch"):
        mc.SpmmProblem(lhs, mc.pack_dense(np.zeros((32, 32), dtype=np.int64), 8))
    with pytest.raises(mc.ShuffleStateError):
        mc.SpmmProblem(lhs, mc.pack_dense(np.zeros((64, 32), dtype=np.int64), 4))
    with pytest.raises(mc.UnsupportedPrecisionError):
        mc.SpmmProblem(_lhs(bits=4), rhs)
    with pytest.raises(ValueError):
        mc.TilingConfig(bs_n=96)
    with pytest.raises(ValueError, match="BS_m"):
        mc.SpmmProblem(lhs, rhs, mc.TilingConfig(bs_m=4))


def test_sddmm_problem_validation():
    pattern = mc.dense_to_bcrs(np.ones((8, 8), dtype=np.int64), 8)
    a = mc.pack_dense(np.ones((8, 16), dtype=np.int64), 8, ROW_MAJOR)
    b = mc.pack_dense(np.ones((16, 8), dtype=np.int64), 8, COL_MAJOR)
    mc.SddmmProblem(a, b, pattern)
    with pytest.raises(ValueError):
        mc.SddmmProblem(mc.pack_dense(np.ones((8, 16), dtype=np.int64), 8, COL_MAJOR), b, pattern)
    with pytest.raises(ValueError):
        mc.SddmmProblem(a, b, pattern, out_format="csr")
    with pytest.raises(mc.UnsupportedPrecisionError):
        mc.SddmmProblem(mc.pack_dense(np.ones((8, 16), dtype=np.int64), 16, ROW_MAJOR), b, pattern)


def test_formats_validation():
    with pytest.raises(mc.StructureError, match="column 1 of vector row 0"):
        d = np.zeros((2, 4), dtype=np.int64)
        d[0, 1] = 7
        mc.dense_to_bcrs(d, 2)
    with pytest.raises(mc.FormatError, match="strictly increasing"):
        mc.BcrsMatrix(2, 8, 2, np.array([0, 2]), np.array([3, 3], dtype=np.uint32),
                      mc.PackedArray.from_values([1, 2, 3, 4], 8))
    with pytest.raises(mc.FormatError):
        mc.SrBcrsMatrix(4, 8, 2, 4, np.array([0, 3]), np.array([2, 4]),
                        np.zeros(8, dtype=np.uint32), mc.PackedArray.from_values(np.zeros(16), 8))
    b = mc.dense_to_bcrs(FMT["hand_dense"], 2)
    assert (mc.bcrs_to_dense(b) == FMT["hand_dense"]).all()


def test_srbcrs_host_helpers_match_reference_layout():
    begin, end = FMT["hand_row_begin"], FMT["hand_row_end"]
    s = mc.SrBcrsMatrix(2, 8, 2, 4, begin, end, FMT["hand_col_indices"],
                        mc.PackedArray(8, int(FMT["hand_meta"][4]), True, FMT["hand_words"]))
    assert list(s._flat_values) == [1, 3, 5, 0, 2, 4, 6, 0]
    assert (mc.srbcrs_to_dense(s) == FMT["hand_dense"]).all()
    assert (mc.bcrs_to_dense(mc.srbcrs_to_bcrs(s)) == FMT["hand_dense"]).all()
    assert s.padded_fraction == 0.25


def test_dlmc_roundtrip_and_errors():
    import io
    b = mc.generate_synthetic(16, 32, 8, 0.75, seed=3)
    buf = io.StringIO()
    mc.write_dlmc(mc.bcrs_to_csr(b), buf)
    csr = mc.read_dlmc(buf.getvalue())
    assert (csr.col_indices == b.col_indices).all()
    with pytest.raises(mc.DlmcParseError) as e:
        mc.read_dlmc("2, 4\n0 1 2\n0 1\n")
    assert e.value.line == 1


def test_alg1_trace_shape():
    t = mc.alg1_trace(2)
    assert t == [("load_lhs", 0), ("sync",), ("prefetch_rhs", 0), ("store_rhs", 0), ("load_lhs", 1),
                 ("sync",), ("prefetch_rhs", 1), ("mma", 0), ("sync",), ("store_rhs", 1), ("sync",),
                 ("mma", 1)]


def test_attention_config_validation():
    mask = mc.generate_synthetic(64, 64, 8, 0.9, seed=0)
    with pytest.raises(ValueError):
        mc.AttentionConfig(60, 8, 8, mask)
    with pytest.raises(mc.UnsupportedPrecisionError):
        mc.AttentionConfig(64, 4, 4, mask)
    cfg = mc.AttentionConfig(64, 16, 8, mask)
    assert cfg.softmax_scale == 1.0 / 32767


def test_compute_requires_cuda_no_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lhs = _lhs()
    rhs = mc.pack_dense(np.zeros((64, 32), dtype=np.int64), 8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mc.spmm(mc.SpmmProblem(lhs, rhs))
