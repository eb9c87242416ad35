"""C2 step composition probe: device time of 200-step CUDA graphs with different launch orders
of the five sweep problems (same cold-L2 copy rotation as bench.py), to see what the
transitions between dense-tile and gather SDDMM launches cost."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
import paper_2209_06979_b200 as mc  # noqa: E402

ctx = B.Ctx()
lib, Nn, dev = ctx.lib, ctx.Nn, ctx.dev
status = torch.zeros(1, dtype=torch.int32, device=dev)
probs = []
for s, c in B.c2_rank_cases(0, 1):
    pat = mc.BcrsMatrix(B.M, B.N, B.V, c["offsets"], c["col_indices"],
                        mc.PackedArray.from_values(np.ones(c["col_indices"].size * B.V), 8))
    p = mc.SddmmProblem(mc.pack_dense(c["a"], 8, mc.qint.ROW_MAJOR), mc.pack_dense(c["b"], 8, mc.qint.COL_MAJOR), pat)
    nblk = pat.n_blocks
    base = [torch.from_numpy(np.asarray(p.a.words).view(np.int32).copy()).to(dev),
            torch.from_numpy(np.asarray(p.b.words).view(np.int32).copy()).to(dev),
            torch.from_numpy(np.asarray(c["offsets"], dtype=np.int64)).to(dev),
            torch.from_numpy(np.asarray(c["col_indices"], dtype=np.uint32).view(np.int32)).to(dev),
            torch.empty(nblk * B.V, dtype=torch.int32, device=dev)]
    foot = sum(t.numel() * t.element_size() for t in base)
    ncopy = max(2, -(-B.COLD_BYTES // foot))
    copies, keep = [], []
    for i in range(ncopy):
        ts = base if i == 0 else [t.clone() for t in base[:4]] + [torch.empty_like(base[4])]
        st, tens = B._sddmm_structs(ts, nblk, Nn)
        copies.append(st)
        keep.append(tens)
    probs.append(dict(s=s, copies=copies, keep=keep, ncopy=ncopy, ops=2 * B.V * B.K * nblk))
sp = lambda st: Nn.stream_ptr(st)


def graph(seq):
    def body(cap):
        for j, ci in seq:
            a, b, pat, out = probs[j]["copies"][ci]
            Nn.check(lib.mc_sddmm(a, b, pat, Nn.ptr(out), Nn.ptr(status), sp(cap)))
    return ctx.capture(body)


def timed(g, pre=True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pre:
        g.replay()
    torch.cuda.synchronize()
    e0.record(ctx.stream); g.replay(); e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000


steps = 200
seq0 = [(j, st % probs[j]["ncopy"]) for st in range(steps) for j in range(5)]
print("first replay (no pre-replay) us/step", round(timed(graph(seq0), pre=False) / steps, 2), flush=True)
g0 = graph(seq0)
try:
    from cuda.bindings import runtime as cudart
    err = cudart.cudaGraphUpload(cudart.cudaGraphExec_t(g0.raw_cuda_graph_exec()), cudart.cudaStream_t(ctx.stream.cuda_stream))
    torch.cuda.synchronize()
    print("upload", err, "then first replay us/step", round(timed(g0, pre=False) / steps, 2), flush=True)
except Exception as ex:
    print("upload failed", repr(ex))
orders = {"50,70,90,95,98": [0, 1, 2, 3, 4], "98,95,90,70,50": [4, 3, 2, 1, 0], "50,90,70,95,98": [0, 2, 1, 3, 4]}
for name, order in orders.items():
    seq = [(j, st % probs[j]["ncopy"]) for st in range(steps) for j in order]
    print(name, "us/step", round(timed(graph(seq)) / steps, 2), flush=True)
for j in range(5):
    seq = [(j, st % probs[j]["ncopy"]) for st in range(steps)]
    print("single", probs[j]["s"], "us", round(timed(graph(seq)) / steps, 2), flush=True)
for a, b in [(0, 4), (0, 2), (1, 2)]:
    seq = [(j, st % probs[j]["ncopy"]) for st in range(steps) for j in (a, b)]
    print("pair", probs[a]["s"], probs[b]["s"], "us/pair", round(timed(graph(seq)) / steps, 2), flush=True)
