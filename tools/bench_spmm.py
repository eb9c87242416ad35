"""SpMM throughput on B200 for BASELINE configs C1, C3 (grid) and C5 (CUDA-graph timing, cold L2).

usage: python tools/bench_spmm.py [c1] [c3l8] [c3] [c3full] [c5] [--out file.json]

Per cell: inputs from the reference generators (oracle.build_spmm_case semantics:
generate_synthetic + bcrs_to_srbcrs + shuffle for R4, bench.py:93-110), resident on
the device; each timed launch is preceded by an L2 flush; the roofline uses the
compulsory HBM bytes of SURVEY.md §8(d) and MEASURED_PEAKS.json.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (input generation + sampled correctness check)
import paper_2209_06979_b200 as mc  # noqa: E402
from paper_2209_06979_b200 import _device as D  # noqa: E402
from paper_2209_06979_b200 import _native as N  # noqa: E402

PAIRS = [(16, 16), (16, 8), (8, 8), (8, 4), (4, 4)]


def peaks():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        d = json.load(f)
    return float(d["hbm_gbs"]), 2.0 * float(d["bf16_tflops"])  # int8 dense ~ 2x bf16 (not measured)


def build(m, n, k, v, sp, lb, rb, seed):
    c = O.build_spmm_case(m, n, k, v, sp, lb, rb, seed)
    t = torch
    lhs = mc.SrBcrsMatrix(m, k, v, c["stride"], t.from_numpy(c["row_begin"]).cuda(),
                          t.from_numpy(c["row_end"]).cuda(),
                          t.from_numpy(c["col_indices"].view(np.int32)).cuda(),
                          mc.PackedArray(c["values"].size, lb, True,
                                         t.from_numpy(mc.pack_values(c["values"], lb).view(np.int32)).cuda()),
                          shuffled=c["shuffled"])
    rhs = mc.PackedMatrix(k, n, rb, mc.qint.ROW_MAJOR, True,
                          t.from_numpy(mc.pack_values(c["rhs"], rb).view(np.int32)).cuda())
    return c, mc.SpmmProblem(lhs, rhs)


def measure(p, reps=20, flush=None):
    lib = N.lib()
    stream = torch.cuda.current_stream()
    out = torch.empty((p.lhs.scalar_rows, p.rhs.cols), dtype=torch.int32, device="cuda")
    mc.kernels.spmm_device(p, out=out)  # warm + status check
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            mc.kernels.spmm_device(p, out=out, stream=cap, check_status=False)
    stream.wait_stream(cap)
    torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for i in range(reps + 2):
        lib.mc_l2_flush(N.ptr(flush), flush.numel(), N.stream_ptr(stream))
        if i >= 2:
            e0[i - 2].record(stream)
        g.replay()
        if i >= 2:
            e1[i - 2].record(stream)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in zip(e0, e1)])), out


def cell(m, n, k, v, sp, lb, rb, seed, flush, check_rows=8):
    hbm, p8 = peaks()
    c, p = build(m, n, k, v, sp, lb, rb, seed)
    ms, out = measure(p, flush=flush)
    nnz = int((c["row_end"] - c["row_begin"]).sum())
    stored = int(c["col_indices"].size)
    ops = 2 * v * n * nnz
    byts = stored * v * lb // 8 + 4 * stored + 16 * (m // v) + k * n * rb // 8 + 4 * m * n
    chunk = {(16, 16): 4, (16, 8): 2}.get((lb, rb), 1)
    t_roof = max(ops * chunk / (p8 * 1e12), byts / (hbm * 1e9))
    rows = list(range(0, m // v, max(1, (m // v) // check_rows)))[:check_rows]
    want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], v, c["stride"],
                  c["shuffled"], lb, c["rhs"], rb, k, rows=rows)
    got = torch.cat([out[r * v:(r + 1) * v] for r in rows]).cpu().numpy()
    return {"M": m, "N": n, "K": k, "V": v, "sparsity": sp, "pair": f"L{lb}-R{rb}", "us": ms * 1e3,
            "tops": ops / (ms * 1e-3) / 1e12, "hbm_gbs": byts / (ms * 1e-3) / 1e9,
            "roofline_frac": t_roof / (ms * 1e-3), "bound": "hbm" if byts / (hbm * 1e9) >= ops * chunk / (p8 * 1e12) else "tensor",
            "bytes": byts, "ops": ops, "exact_sampled_rows": bool((got == want).all())}


def main():
    args = sys.argv[1:]
    outp = None
    if "--out" in args:
        outp = args[args.index("--out") + 1]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = []
    if "c1" in args:
        seed = O.cell_seed(0, ((512, 256, 512), 8, 0.9, "L8-R8"))
        res.append(dict(cfg="C1", **cell(512, 256, 512, 8, 0.9, 8, 8, seed, flush)))
    if "c3l8" in args:  # the tcgen05 path's cells: L8-R8, V=8
        for sp in (0.7, 0.9, 0.95, 0.98):
            seed = O.cell_seed(0, ((4096, 512, 4096), 8, sp, "L8-R8"))
            r = dict(cfg="C3", **cell(4096, 512, 4096, 8, sp, 8, 8, seed, flush))
            res.append(r)
            print(json.dumps(r), flush=True)
    if "c3" in args or "c3full" in args:
        sps = (0.7, 0.8, 0.9, 0.95, 0.98) if "c3full" in args else (0.7, 0.9, 0.98)
        for lb, rb in PAIRS:
            for v in (8, 4, 2):
                for sp in sps:
                    seed = O.cell_seed(0, ((4096, 512, 4096), v, sp, f"L{lb}-R{rb}"))
                    r = dict(cfg="C3", **cell(4096, 512, 4096, v, sp, lb, rb, seed, flush))
                    res.append(r)
                    print(json.dumps(r), flush=True)
    if "c5" in args:
        t0 = time.time()
        seed = O.cell_seed(0, ((32768, 2048, 32768), 8, 0.95, "L8-R4"))
        r = dict(cfg="C5", **cell(32768, 2048, 32768, 8, 0.95, 8, 4, seed, flush, check_rows=4))
        r["build_s"] = time.time() - t0
        res.append(r)
    for r in res:
        if r["cfg"] != "C3":
            print(json.dumps(r), flush=True)
    if outp:
        with open(outp, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
