"""Benchmark / verification front door (reference: qsparse.bench + qsparse.cli).

Same sweep grid, cell seeds, builders, report formats and exit codes as the reference's
`qsparse-bench` (cli.py:27-133, bench.py:25-286), running the B200 kernels:

* `SweepSpec`, `BenchRecord`, `run_sweep`, `verify`, `report`, `load_records` mirror
  bench.py:28-67, :140-286 -- records carry the reference's columns (CSV order kept) plus
  three GPU columns appended at the end: `device_median_s` (CUDA-event median of the
  device-resident launch), `tops` (logical ops / device time) and `kernel` (the kernel the
  library chose, mc_spmm_path / the SDDMM density dispatch);
* matrices come from the reference generators (`generate_synthetic` / `dilate`, seeded by
  the reference's `_cell_seed`, capped by `safe_magnitudes`, bench.py:70-136);
* `verify` compares the kernel output with a dense wide-integer product computed on the
  GPU in float64 (cuBLAS DGEMM through torch; exact below 2^53) -- the role of the
  reference's `reference.spmm_reference` / `sddmm_reference` / `attention_reference`
  (reference.py:19-56); `inject_fault` flips one output bit first (negative control);
* `main` is the `qsparse-bench` CLI: `spmm | sddmm | attention | verify`, same flags;
  exit code 0 only if every executed cell verified (or --no-verify).

    python -m paper_2209_06979_b200.bench_cli spmm --m 512 --n 256 --k 512 --sparsity 0.9
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import json
import math
import sys
import time
from dataclasses import asdict, dataclass, fields
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _device as D
from . import _native as N
from . import attention, emulation, kernels
from .errors import UnsupportedPrecisionError
from .qint import COL_MAJOR, ROW_MAJOR, pack_dense, signed_range
from .sparse_format import (CsrMatrix, bcrs_to_dense, bcrs_to_srbcrs, dilate, generate_synthetic,
                            read_dlmc, shuffle_indices, srbcrs_to_dense)

JSON_SCHEMA = "qsparse-bench-v1"
DEFAULT_SPARSITIES = (0.5, 0.7, 0.8, 0.9, 0.95, 0.98)
DEFAULT_REPETITIONS = 32


@dataclass(frozen=True)
class SweepSpec:
    """bench.SweepSpec (bench.py:28-42)."""
    op: str
    shapes: Sequence[Tuple[int, int, int]]
    sparsities: Sequence[float] = DEFAULT_SPARSITIES
    vector_lengths: Sequence[int] = (8,)
    precisions: Sequence[str] = ("L8-R8",)
    bs_n: int = 64
    pipeline: bool = False
    repetitions: int = DEFAULT_REPETITIONS
    seed: int = 0
    dlmc: Optional[CsrMatrix] = None


@dataclass
class BenchRecord:
    """bench.BenchRecord (bench.py:45-64) + GPU columns (appended)."""
    op: str
    m: int
    n: int
    k: int
    vector_length: int
    sparsity: float
    precision: str
    bs_n: int
    pipeline: bool
    repetitions: int
    seed: int
    status: str = "ok"
    reason: str = ""
    verified: Optional[bool] = None
    median_s: float = 0.0
    p95_s: float = 0.0
    bytes_lhs: int = 0
    bytes_rhs: int = 0
    device_median_s: float = 0.0
    tops: float = 0.0
    kernel: str = ""


CSV_COLUMNS = [f.name for f in fields(BenchRecord)]


@dataclass
class VerifyOutcome:
    passed: bool
    message: str = ""


def safe_magnitudes(lhs_bits: int, rhs_bits: int, k: int, op: str) -> Tuple[int, int]:
    """bench.safe_magnitudes (bench.py:70-83): caps keeping every int32 accumulator in range."""
    scheme = emulation.plan(lhs_bits, rhs_bits, op)
    limit = (1 << 31) - 1
    root = int(math.isqrt(limit // max(k, 1)))
    chunk_max = (1 << scheme.native_width) - 1
    mag_l = min(signed_range(lhs_bits)[1], root, limit // (max(k, 1) * chunk_max))
    mag_r = min(signed_range(rhs_bits)[1], root)
    return max(mag_l, 1), max(mag_r, 1)


def cell_seed(spec: SweepSpec, coords: tuple) -> int:
    """bench._cell_seed (bench.py:86-90): process-independent sha256 of the cell."""
    key = repr((spec.seed,) + coords).encode()
    return int.from_bytes(hashlib.sha256(key).digest()[:4], "little")


def _build_spmm(spec, shape, v, sparsity, lb, rb, seed):
    """bench._build_spmm (bench.py:93-110); the SR-BCRS packer and shuffle run on the GPU."""
    m, n, k = shape
    scheme = emulation.plan(lb, rb, emulation.SPMM)
    mag_l, mag_r = safe_magnitudes(lb, rb, k, emulation.SPMM)
    if spec.dlmc is not None:
        b = dilate(spec.dlmc, v, value_seed=seed, bit_width=lb, max_magnitude=mag_l)
        m, k = b.scalar_rows, b.scalar_cols
    else:
        b = generate_synthetic(m, k, v, sparsity, seed, bit_width=lb, max_magnitude=mag_l)
    lhs = bcrs_to_srbcrs(b, scheme.tile.k)
    if rb == 4:
        lhs = shuffle_indices(lhs)
    rng = np.random.default_rng(seed + 1)
    rhs = pack_dense(rng.integers(-mag_r, mag_r + 1, (k, n)), rb, ROW_MAJOR)
    cfg = kernels.TilingConfig(bs_n=spec.bs_n, pipeline=spec.pipeline)
    return kernels.SpmmProblem(lhs, rhs, cfg), (m, n, k), lhs.nbytes, rhs.nbytes


def _build_sddmm(spec, shape, v, sparsity, lb, rb, seed):
    """bench._build_sddmm (bench.py:113-126)."""
    m, n, k = shape
    mag_l, mag_r = safe_magnitudes(lb, rb, k, emulation.SDDMM)
    if spec.dlmc is not None:
        pattern = dilate(spec.dlmc, v, value_seed=seed, bit_width=8)
        m, n = pattern.scalar_rows, pattern.scalar_cols
    else:
        pattern = generate_synthetic(m, n, v, sparsity, seed, bit_width=8)
    rng = np.random.default_rng(seed + 1)
    a = pack_dense(rng.integers(-mag_l, mag_l + 1, (m, k)), lb, ROW_MAJOR)
    bmat = pack_dense(rng.integers(-mag_r, mag_r + 1, (k, n)), rb, COL_MAJOR)
    cfg = kernels.TilingConfig(bs_n=spec.bs_n, pipeline=False)
    return kernels.SddmmProblem(a, bmat, pattern, config=cfg), (m, n, k), a.nbytes, bmat.nbytes


def _build_attention(spec, shape, v, sparsity, sb, qb, seed):
    """bench._build_attention (bench.py:129-136)."""
    seq_len, head_dim, heads = shape
    mask = generate_synthetic(seq_len, seq_len, 8, sparsity, seed, bit_width=8)
    cfg = attention.AttentionConfig(seq_len, sb, qb, mask, head_dim=head_dim, num_heads=heads)
    rng = np.random.default_rng(seed + 1)
    q, k, vmat = (rng.normal(size=(seq_len, head_dim)) for _ in range(3))
    return cfg, (q, k, vmat)


# ---------------------------------------------------------------------------------------
# verification: dense products on the GPU in float64 (exact for these magnitudes)
# ---------------------------------------------------------------------------------------

def _f64(x):
    t = D.torch()
    return t.as_tensor(np.asarray(x, dtype=np.float64), device="cuda")


def _spmm_dense_reference(p) -> np.ndarray:
    t = D.torch()
    return t.matmul(_f64(srbcrs_to_dense(p.lhs)), _f64(p.rhs.to_dense())).round().to(t.int64).cpu().numpy()


def _sddmm_dense_reference(p) -> np.ndarray:
    t = D.torch()
    mask = _f64(bcrs_to_dense(p.out_pattern) != 0) != 0
    full = t.matmul(_f64(p.a.to_dense()), _f64(p.b.to_dense())).round().to(t.int64)
    return t.where(mask, full, t.zeros_like(full)).cpu().numpy()


def _attention_dense_reference(q, k, v, cfg):
    """reference.attention_reference (reference.py:29-56): the dense quantised pipeline with
    the same rounding steps (float64 on the GPU; fp16 rounding via half casts)."""
    t = D.torch()
    qmax = (1 << (cfg.qkv_bits - 1)) - 1

    def quant(x):
        x = _f64(x)
        am = float(x.abs().max()) if x.numel() else 0.0
        s = am / qmax if am > 0 else 1.0
        return t.clamp(t.round(x / s), -qmax, qmax), s

    qi, sq = quant(q)
    ki, sk = quant(k)
    vi, sv = quant(v)
    mask = _f64(bcrs_to_dense(cfg.mask) != 0) != 0
    scores_int = t.where(mask, qi @ ki.T, t.zeros((), dtype=t.float64, device="cuda"))
    alpha = sq * sk / math.sqrt(cfg.head_dim)
    scores = (scores_int * alpha).half().double()
    neg = t.full_like(scores, -math.inf)
    x = t.where(mask, scores, neg)
    mx = x.max(dim=1, keepdim=True).values
    e = t.where(mask, t.exp(x - t.where(t.isfinite(mx), mx, t.zeros_like(mx))), t.zeros_like(scores))
    s = e.sum(dim=1, keepdim=True)
    probs = t.where(s > 0, e / t.where(s > 0, s, t.ones_like(s)), t.zeros_like(e)).half().double()
    smax = (1 << (cfg.softmax_bits - 1)) - 1
    probs_int = t.clamp(t.round(probs / (1.0 / smax)), -smax, smax)
    mix = probs_int @ vi
    return {"probs_int": probs_int.to(t.int64).cpu().numpy(), "mix_int": mix.to(t.int64).cpu().numpy()}


def _first_mismatch(got: np.ndarray, want: np.ndarray) -> str:
    diff = np.nonzero(got != want)
    idx = tuple(int(d[0]) for d in diff)
    return f"first mismatch at {idx}: kernel={got[idx]} oracle={want[idx]}"


def verify(op: str, shape, vector_length: int, sparsity: float, precision: str, bs_n: int = 64,
           pipeline: bool = False, seed: int = 0, dlmc: Optional[CsrMatrix] = None,
           inject_fault: bool = False) -> VerifyOutcome:
    """bench.verify (bench.py:151-190): one cell against the dense wide-integer product."""
    lb, rb = emulation.parse_precision(precision)
    spec = SweepSpec(op, [tuple(shape)], [sparsity], [vector_length], [precision], bs_n=bs_n,
                     pipeline=pipeline, seed=seed, dlmc=dlmc)
    cs = cell_seed(spec, (tuple(shape), vector_length, sparsity, precision))
    if op == "spmm":
        problem, _, _, _ = _build_spmm(spec, shape, vector_length, sparsity, lb, rb, cs)
        got = kernels.spmm(problem)
        want = _spmm_dense_reference(problem)
    elif op == "sddmm":
        problem, _, _, _ = _build_sddmm(spec, shape, vector_length, sparsity, lb, rb, cs)
        got = bcrs_to_dense(kernels.sddmm(problem))
        want = _sddmm_dense_reference(problem)
    elif op == "attention":
        cfg, (q, k, v) = _build_attention(spec, shape, vector_length, sparsity, lb, rb, cs)
        res = attention.sparse_attention(q, k, v, cfg)
        ref = _attention_dense_reference(q, k, v, cfg)
        got = np.asarray(res.mix_int, dtype=np.int64)
        want = ref["mix_int"]
        if not (bcrs_to_dense(res.probs_int) == ref["probs_int"]).all():
            return VerifyOutcome(False, "quantized softmax stage mismatch")
    else:
        raise ValueError(f"unknown op {op!r}")
    got = np.asarray(got, dtype=np.int64).copy()
    if inject_fault:
        got.flat[got.size // 2] ^= 1
    if (got == want).all():
        return VerifyOutcome(True, "bit-exact")
    return VerifyOutcome(False, _first_mismatch(got, want))


# ---------------------------------------------------------------------------------------
# sweeps
# ---------------------------------------------------------------------------------------

def _device_time(launch, reps: int) -> float:
    """Median CUDA-event time (s) of a device-resident launch."""
    t = D.torch()
    launch()
    ev = [(t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        launch()
        b.record()
    t.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev])) * 1e-3


def _spmm_kernel_name(p) -> str:
    lhs, _k1 = D.srbcrs_struct(p.lhs)
    rhs, _k2 = D.dense_struct(p.rhs)
    pid = N.ctypes.c_int32(-1)
    N.check(N.lib().mc_spmm_path(lhs, rhs, N.ctypes.byref(pid)))
    return N.SPMM_PATHS[pid.value]


def _sddmm_kernel_name(p) -> str:
    a, _k1 = D.dense_struct(p.a)
    b, _k2 = D.dense_struct(p.b)
    pat, _k3 = D.bcrs_struct(p.out_pattern)
    pid = N.ctypes.c_int32(-1)
    N.check(N.lib().mc_sddmm_path(a, b, pat, N.ctypes.byref(pid)))
    return N.SDDMM_PATHS[pid.value]


def run_sweep(spec: SweepSpec, verify_cells: bool = True) -> List[BenchRecord]:
    """bench.run_sweep (bench.py:193-207): every cell in stable order."""
    records: List[BenchRecord] = []
    for shape in spec.shapes:
        for v in spec.vector_lengths:
            for sparsity in spec.sparsities:
                for precision in spec.precisions:
                    records.append(_run_cell(spec, tuple(shape), v, sparsity, precision, verify_cells))
    return records


def _run_cell(spec: SweepSpec, shape, v, sparsity, precision, verify_cells) -> BenchRecord:
    rec = BenchRecord(spec.op, shape[0], shape[1], shape[2], v, sparsity, precision, spec.bs_n,
                      spec.pipeline, spec.repetitions, spec.seed)
    try:
        lb, rb = emulation.parse_precision(precision)
        op_kind = emulation.SDDMM if spec.op == "sddmm" else emulation.SPMM
        if spec.op in ("spmm", "sddmm"):
            emulation.plan(lb, rb, op_kind)
    except (UnsupportedPrecisionError, ValueError) as e:
        rec.status, rec.reason = "skipped", str(e)
        return rec
    seed = cell_seed(spec, (shape, v, sparsity, precision))
    t = D.torch()
    try:
        if spec.op == "spmm":
            problem, dims, rec.bytes_lhs, rec.bytes_rhs = _build_spmm(spec, shape, v, sparsity, lb, rb, seed)
            rec.m, rec.n, rec.k = dims
            runner = lambda: kernels.spmm(problem)
            out = t.empty((problem.lhs.scalar_rows, problem.rhs.cols), dtype=t.int32, device="cuda")
            device = lambda: kernels.spmm_device(problem, out=out, check_status=False)
            nnz = int((np.asarray(problem.lhs.row_end) - np.asarray(problem.lhs.row_begin)).sum())
            ops = 2 * v * rec.n * nnz
            rec.kernel = _spmm_kernel_name(problem)
        elif spec.op == "sddmm":
            problem, dims, rec.bytes_lhs, rec.bytes_rhs = _build_sddmm(spec, shape, v, sparsity, lb, rb, seed)
            rec.m, rec.n, rec.k = dims
            runner = lambda: kernels.sddmm(problem)
            out = t.empty(problem.out_pattern.n_blocks * v, dtype=t.int32, device="cuda")
            device = lambda: kernels.sddmm_device(problem, out=out, check_status=False)
            ops = 2 * v * rec.k * problem.out_pattern.n_blocks
            rec.kernel = _sddmm_kernel_name(problem)
        elif spec.op == "attention":
            cfg, (q, k, vmat) = _build_attention(spec, shape, v, sparsity, lb, rb, seed)
            runner = lambda: attention.sparse_attention(q, k, vmat, cfg)
            run = attention.AttentionRunner(cfg, 1, mode="parity")
            qd, kd, vd = (t.as_tensor(x, device="cuda").half()[None] for x in (q, k, vmat))
            device = lambda: run(qd, kd, vd)
            ops = 4 * 8 * cfg.head_dim * cfg.mask.n_blocks
            rec.kernel = "absquant_f16_kernel + score_softmax_kernel (fused SDDMM/softmax/SpMM)"
        else:
            raise ValueError(f"unknown op {spec.op!r}")
    except (UnsupportedPrecisionError, ValueError) as e:
        rec.status, rec.reason = "skipped", str(e)
        return rec
    times = []
    res = None
    for _ in range(spec.repetitions):
        t0 = time.perf_counter()
        res = runner()
        times.append(time.perf_counter() - t0)
    rec.median_s = float(np.median(times))
    rec.p95_s = float(np.percentile(times, 95))
    rec.device_median_s = _device_time(device, max(3, min(spec.repetitions, 20)))
    rec.tops = ops / rec.device_median_s / 1e12 if rec.device_median_s > 0 else 0.0
    if spec.op == "attention":
        rec.bytes_lhs = int(np.asarray(res.probs_int.values.words if hasattr(res.probs_int.values, "words")
                                       else res.probs_int.values).nbytes)
        rec.bytes_rhs = (cfg.seq_len * cfg.head_dim * cfg.qkv_bits + 31) // 32 * 4
    if verify_cells:
        rec.verified = verify(spec.op, shape, v, sparsity, precision, spec.bs_n, spec.pipeline, spec.seed,
                              spec.dlmc).passed
    return rec


def report(records: Sequence[BenchRecord], fmt: str, out_path: str) -> None:
    """bench.report (bench.py:264-277): stable CSV column order or the versioned JSON schema."""
    if fmt == "csv":
        with open(out_path, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=CSV_COLUMNS)
            w.writeheader()
            for r in records:
                w.writerow(asdict(r))
    elif fmt == "json":
        with open(out_path, "w") as f:
            json.dump({"schema": JSON_SCHEMA, "records": [asdict(r) for r in records]}, f, indent=2)
    else:
        raise ValueError(f"format must be csv or json, got {fmt!r}")


def load_records(path: str) -> List[BenchRecord]:
    """bench.load_records (bench.py:280-286)."""
    with open(path) as f:
        doc = json.load(f)
    if doc.get("schema") != JSON_SCHEMA:
        raise ValueError(f"unknown schema {doc.get('schema')!r}")
    return [BenchRecord(**r) for r in doc["records"]]


# ---------------------------------------------------------------------------------------
# CLI (cli.py:27-133)
# ---------------------------------------------------------------------------------------

def _int_list(text: str) -> List[int]:
    return [int(t) for t in text.split(",") if t]


def _float_list(text: str) -> List[float]:
    return [float(t) for t in text.split(",") if t]


def _add_common(p: argparse.ArgumentParser, op: str):
    p.add_argument("--m", type=int, default=64, help="rows (spmm/sddmm) or sequence length (attention)")
    p.add_argument("--n", type=int, default=64, help="output columns (spmm/sddmm) or head count (attention)")
    p.add_argument("--k", type=int, default=128, help="reduction size (spmm/sddmm) or head dimension (attention)")
    p.add_argument("--vlen", type=_int_list, default=[8], help="comma-separated vector lengths from {2,4,8}")
    p.add_argument("--sparsity", type=_float_list, default=list(DEFAULT_SPARSITIES), help="comma-separated sparsities")
    p.add_argument("--lhs-bits", type=_int_list, default=[8], help="LHS precisions (softmax bits for attention)")
    p.add_argument("--rhs-bits", type=_int_list, default=[8], help="RHS precisions (Q/K/V bits for attention)")
    p.add_argument("--bsn", type=int, choices=(64, 128), default=64)
    p.add_argument("--pipeline", choices=("on", "off"), default="off")
    p.add_argument("--reps", type=int, default=DEFAULT_REPETITIONS)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--dlmc", type=str, default=None, help="path to a DLMC text file; synthetic matrices otherwise")
    p.add_argument("--format", choices=("csv", "json"), default="csv")
    p.add_argument("--out", type=str, default=None, help="report output path")
    p.add_argument("--no-verify", action="store_true", help="skip oracle comparison for executed cells")
    p.set_defaults(op=op)


def _build_spec(args) -> SweepSpec:
    precisions = [emulation.precision_name(l, r) for l in args.lhs_bits for r in args.rhs_bits]
    dlmc = None
    if args.dlmc:
        with open(args.dlmc) as f:
            dlmc = read_dlmc(f)
    op = getattr(args, "target_op", args.op)
    shape = (args.m, args.k, args.n) if op == "attention" else (args.m, args.n, args.k)
    return SweepSpec(op=args.op, shapes=[shape], sparsities=args.sparsity, vector_lengths=args.vlen,
                     precisions=precisions, bs_n=args.bsn, pipeline=args.pipeline == "on",
                     repetitions=args.reps, seed=args.seed, dlmc=dlmc)


def _cmd_sweep(args) -> int:
    spec = _build_spec(args)
    records = run_sweep(spec, verify_cells=not args.no_verify)
    for r in records:
        if r.status == "skipped":
            print(f"{r.op} {r.precision} V={r.vector_length} sp={r.sparsity}: skipped ({r.reason})")
            continue
        flag = "-" if r.verified is None else ("ok" if r.verified else "FAIL")
        dims = f"L={r.m} d_k={r.n} heads={r.k}" if r.op == "attention" else f"M={r.m} N={r.n} K={r.k}"
        print(f"{r.op} {dims} V={r.vector_length} sp={r.sparsity} {r.precision} bsn={r.bs_n} "
              f"pipe={'on' if r.pipeline else 'off'}: median {r.median_s * 1e3:.3f} ms  "
              f"p95 {r.p95_s * 1e3:.3f} ms  device {r.device_median_s * 1e6:.1f} us  "
              f"{r.tops:.2f} TOPS [{r.kernel}]  verify={flag}")
    if args.out:
        report(records, args.format, args.out)
        print(f"wrote {len(records)} records to {args.out}")
    executed = [r for r in records if r.status == "ok"]
    if args.no_verify:
        return 0
    return 0 if all(r.verified for r in executed) else 1


def _cmd_verify(args) -> int:
    spec = _build_spec(args)
    code = 0
    for v in spec.vector_lengths:
        for sp in spec.sparsities:
            for prec in spec.precisions:
                outcome = verify(args.target_op, spec.shapes[0], v, sp, prec, bs_n=spec.bs_n,
                                 pipeline=spec.pipeline, seed=spec.seed, dlmc=spec.dlmc)
                status = "pass" if outcome.passed else f"FAIL: {outcome.message}"
                print(f"{args.target_op} {prec} V={v} sp={sp}: {status}")
                code |= 0 if outcome.passed else 1
    return code


def main(argv=None) -> int:
    parser = argparse.ArgumentParser(prog="qsparse-bench", description=__doc__.splitlines()[0])
    sub = parser.add_subparsers(dest="command", required=True)
    for op in ("spmm", "sddmm", "attention"):
        _add_common(sub.add_parser(op, help=f"sweep the {op} kernel"), op)
    pv = sub.add_parser("verify", help="verify one cell against the dense reference")
    pv.add_argument("target_op", choices=("spmm", "sddmm", "attention"))
    _add_common(pv, "verify")
    args = parser.parse_args(argv)
    if args.command == "verify":
        return _cmd_verify(args)
    return _cmd_sweep(args)


if __name__ == "__main__":
    sys.exit(main())
