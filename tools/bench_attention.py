"""Quantized sparse attention throughput (BASELINE config C4) on B200.

usage: python tools/bench_attention.py [--batch B] [--heads H] [--seq L] [--mode fast|parity] [--out f.json]

C4: 8-bit (softmax 8b, qkv 8b), seq 4096, 8 heads, d=64, batch 64, 90% mask (V=8,
shared by all heads). One step = one layer: quantize Q/K/V -> SDDMM + dequant ->
softmax + requant -> SpMM + dequant for all B*H heads (mc_sparse_attention).
seq/s = B / t_layer. Inputs fp16 N(0,1), resident on the device; L2 flushed per step.
Correctness: a sampled head is compared with the oracle (parity mode exact,
fast mode within FAST_MODE_TOLERANCE).
"""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2209_06979_b200 as mc  # noqa: E402
from paper_2209_06979_b200 import _native as N  # noqa: E402


def run(batch=64, heads=8, seq=4096, d=64, sparsity=0.9, mode="fast", sb=8, qb=8, steps=10):
    seed = O.cell_seed(0, ((seq, d, heads), 8, sparsity, f"L{sb}-R{qb}"))
    offs, cols, _ = O.synthetic_bcrs(seq, seq, 8, sparsity, seed, 8)
    mask = mc.BcrsMatrix(seq, seq, 8, offs, cols, mc.PackedArray.from_values(np.ones(cols.size * 8), 8))
    cfg = mc.AttentionConfig(seq, sb, qb, mask, head_dim=d, num_heads=heads)
    nh = batch * heads
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn((nh, seq, d), device="cuda", generator=g).half() for _ in range(3))
    run_ = mc.AttentionRunner(cfg, nh, mode=mode)
    lib = N.lib()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    run_(q, k, v, check=True)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    lib.mc_launch_count(1)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph, stream=cap):
            run_(q, k, v, stream=cap)
    launches = int(lib.mc_launch_count(0))
    stream.wait_stream(cap)
    torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps + 2):
        lib.mc_l2_flush(N.ptr(flush), flush.numel(), N.stream_ptr(stream))
        if i >= 2:
            e0[i - 2].record(stream)
        graph.replay()
        if i >= 2:
            e1[i - 2].record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in zip(e0, e1)]))
    # sampled correctness vs the oracle (head 0 and the last head)
    errs = []
    for h in (0, nh - 1):
        qh, kh, vh = (x[h].double().cpu().numpy() for x in (q, k, v))
        ref = O.attention(qh, kh, vh, offs, cols, seq, d, sb, qb)
        errs.append(float(np.abs(run_.out[h].double().cpu().numpy() - ref["output"]).max()))
    nblk = int(offs[-1])
    ops = nh * 4 * 8 * d * nblk
    in_bytes = 3 * nh * seq * d * 2
    out_bytes = nh * seq * d * 2
    byts = in_bytes + out_bytes + 8 * (seq // 8 + 1) + 4 * nblk
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    return {"cfg": "C4", "batch": batch, "heads": heads, "seq": seq, "d": d, "sparsity": sparsity,
            "precision": f"{sb}b-{qb}b", "mode": mode, "ms_per_layer": ms, "seq_per_s": batch / (ms * 1e-3),
            "tops": ops / (ms * 1e-3) / 1e12, "hbm_roofline_ms": byts / (hbm * 1e9) * 1e3,
            "roofline_frac": (byts / (hbm * 1e9)) / (ms * 1e-3), "launches_per_layer": launches,
            "max_abs_err_vs_oracle": max(errs),
            "tolerance": mc.attention.FAST_MODE_TOLERANCE if mode == "fast" else 0.0}


def main():
    a = sys.argv[1:]

    def opt(name, default, cast):
        return cast(a[a.index(name) + 1]) if name in a else default
    r = run(batch=opt("--batch", 64, int), heads=opt("--heads", 8, int), seq=opt("--seq", 4096, int),
            mode=opt("--mode", "fast", str))
    print(json.dumps(r), flush=True)
    if "--out" in a:
        with open(a[a.index("--out") + 1], "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
