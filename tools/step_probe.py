"""Probe: per-kernel vs mixed-sequence device time of the C2 sweep launches (warm L2)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench as B  # noqa: E402
from paper_2209_06979_b200 import _native as Nn  # noqa: E402

lib = Nn.lib()
dev = torch.device("cuda", 0)
cases = B.build_c2(0)
probs = []
for s, c in cases:
    import paper_2209_06979_b200 as mc
    pat = mc.BcrsMatrix(B.M, B.N, B.V, c["offsets"], c["col_indices"], mc.PackedArray.from_values(np.ones(c["col_indices"].size * B.V), 8))
    a = mc.pack_dense(c["a"], 8, mc.qint.ROW_MAJOR)
    b = mc.pack_dense(c["b"], 8, mc.qint.COL_MAJOR)
    nblk = pat.n_blocks
    t = [torch.from_numpy(np.asarray(a.words).view(np.int32).copy()).to(dev),
         torch.from_numpy(np.asarray(b.words).view(np.int32).copy()).to(dev),
         torch.from_numpy(np.asarray(c["offsets"], dtype=np.int64)).to(dev),
         torch.from_numpy(np.asarray(c["col_indices"], dtype=np.uint32).view(np.int32)).to(dev),
         torch.empty(nblk * 8, dtype=torch.int32, device=dev)]
    probs.append(B._structs(t, nblk, Nn))
status = torch.zeros(1, dtype=torch.int32, device=dev)

def graph(seq, reps):
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        sp = Nn.stream_ptr(cap)
        with torch.cuda.graph(g, stream=cap):
            for _ in range(reps):
                for i in seq:
                    a, b, pat, out = probs[i]
                    Nn.check(lib.mc_sddmm(a, b, pat, Nn.ptr(out), Nn.ptr(status), sp))
    torch.cuda.synchronize()
    return g

def timeit(g):
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3

R = 20
single = [timeit(graph([i], R)) / R for i in range(5)]
print("single us:", [round(x, 2) for x in single], "sum", round(sum(single), 2))
for seq in ([0, 1, 2, 3, 4], [3, 4, 0, 1, 2], [0, 1, 2], [3, 4], [0, 3], [2, 3]):
    t = timeit(graph(seq, R)) / R
    print("seq", seq, round(t, 2), "sum singles", round(sum(single[i] for i in seq), 2))
