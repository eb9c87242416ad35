"""The `qsparse-bench` front door (paper_2209_06979_b200.bench_cli; reference cli.py / bench.py).

CPU tests pin the seeds, caps and report formats to the reference (golden KATs from the
imported reference); `-m gpu` tests mirror the reference's TestRunSweep / TestCli
(tests/test_bench.py) on the device kernels, including the fault-injection negative control.
"""

import csv
import dataclasses

import numpy as np
import pytest

from conftest import load_golden

FMT = load_golden("formats")


def _cli():
    from paper_2209_06979_b200 import bench_cli
    return bench_cli


def tiny_spec(**kw):
    b = _cli()
    defaults = dict(op="spmm", shapes=[(16, 32, 32)], sparsities=[0.5], vector_lengths=[8],
                    precisions=["L8-R8"], repetitions=2, seed=0)
    defaults.update(kw)
    return b.SweepSpec(**defaults)


def test_cell_seed_and_magnitudes_match_reference():
    b = _cli()
    spec = b.SweepSpec("spmm", [(512, 256, 512)])
    assert b.cell_seed(spec, ((512, 256, 512), 8, 0.9, "L8-R8")) == int(FMT["seed/c1"][0])
    for lb, rb, k, ml, mr in FMT["safe_magnitudes"]:
        assert b.safe_magnitudes(int(lb), int(rb), int(k), "spmm") == (ml, mr)


def test_report_roundtrip_and_columns(tmp_path):
    b = _cli()
    recs = [b.BenchRecord("spmm", 16, 32, 32, 8, 0.5, "L8-R8", 64, False, 2, 0, verified=True,
                          median_s=1e-3, p95_s=2e-3, bytes_lhs=10, bytes_rhs=20, device_median_s=1e-5,
                          tops=1.5, kernel="k")]
    path = tmp_path / "r.json"
    b.report(recs, "json", str(path))
    assert b.load_records(str(path)) == recs
    cpath = tmp_path / "r.csv"
    b.report(recs, "csv", str(cpath))
    header = next(csv.reader(open(cpath)))
    # the reference's columns first, in its order (bench.py:45-67), GPU columns appended
    assert header[:18] == ["op", "m", "n", "k", "vector_length", "sparsity", "precision", "bs_n", "pipeline",
                           "repetitions", "seed", "status", "reason", "verified", "median_s", "p95_s",
                           "bytes_lhs", "bytes_rhs"]
    with pytest.raises(ValueError):
        b.report([], "xml", str(tmp_path / "x"))


@pytest.mark.gpu
class TestSweepGpu:
    def test_single_verified_cell(self):
        recs = _cli().run_sweep(tiny_spec())
        assert len(recs) == 1 and recs[0].status == "ok" and recs[0].verified is True
        assert recs[0].median_s > 0 and recs[0].p95_s >= recs[0].median_s and recs[0].device_median_s > 0

    def test_infeasible_cell_skipped_run_continues(self):
        recs = _cli().run_sweep(tiny_spec(precisions=["L8-R16", "L8-R8"]))
        assert [r.status for r in recs] == ["skipped", "ok"]
        assert "not supported" in recs[0].reason

    def test_determinism_across_runs(self):
        strip = lambda r: dataclasses.replace(r, median_s=0.0, p95_s=0.0, device_median_s=0.0, tops=0.0)
        a = _cli().run_sweep(tiny_spec(sparsities=[0.5, 0.9]))
        b = _cli().run_sweep(tiny_spec(sparsities=[0.5, 0.9]))
        assert [strip(x) for x in a] == [strip(x) for x in b]

    @pytest.mark.parametrize("op,prec", [("spmm", "L8-R4"), ("spmm", "L16-R8"), ("sddmm", "L16-R16"),
                                         ("sddmm", "L4-R4"), ("attention", "L8-R8"), ("attention", "L16-R8")])
    def test_verify_and_negative_control(self, op, prec):
        b = _cli()
        shape = (64, 64, 1) if op == "attention" else (64, 96, 128)
        assert b.verify(op, shape, 8, 0.7, prec).passed
        out = b.verify(op, shape, 8, 0.7, prec, inject_fault=True)
        assert not out.passed and "mismatch" in out.message


@pytest.mark.gpu
class TestCliGpu:
    ARGS = ["--m", "16", "--n", "32", "--k", "32", "--sparsity", "0.5", "--reps", "1", "--seed", "3"]

    def test_spmm_exit_zero(self, capsys):
        assert _cli().main(["spmm"] + self.ARGS) == 0
        assert "verify=ok" in capsys.readouterr().out

    def test_report_written(self, tmp_path):
        out = tmp_path / "report.csv"
        assert _cli().main(["spmm"] + self.ARGS + ["--out", str(out), "--format", "csv"]) == 0 and out.exists()

    def test_skipped_pairs_do_not_fail(self, capsys):
        assert _cli().main(["spmm"] + self.ARGS + ["--lhs-bits", "8,4", "--rhs-bits", "8"]) == 0
        assert "skipped" in capsys.readouterr().out

    def test_no_verify_flag(self, capsys):
        assert _cli().main(["spmm"] + self.ARGS + ["--no-verify"]) == 0
        assert "verify=-" in capsys.readouterr().out

    def test_verify_subcommand(self, capsys):
        assert _cli().main(["verify", "spmm"] + self.ARGS) == 0
        assert "pass" in capsys.readouterr().out

    def test_sddmm_and_attention_subcommands(self):
        assert _cli().main(["sddmm"] + self.ARGS) == 0
        assert _cli().main(["attention", "--m", "64", "--k", "64", "--n", "1", "--sparsity", "0.9",
                            "--lhs-bits", "8", "--rhs-bits", "8", "--reps", "1"]) == 0

    def test_dlmc_flag(self, tmp_path):
        dlmc = tmp_path / "m.dlmc"
        dlmc.write_text("4, 32, 8\n0 2 4 6 8\n0 5 3 9 1 2 7 8\n")
        assert _cli().main(["spmm"] + self.ARGS + ["--dlmc", str(dlmc)]) == 0
