"""Print the per-CTA globaltimer timeline of the dense SDDMM kernel (debug aid)."""

import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["MCUBE_DEBUG_TIMELINE"] = "1"
os.environ.setdefault("MCUBE_LIB_PATH", os.path.join(ROOT, "paper_2209_06979_b200", "libmcube_timeline.so"))
os.environ["MCUBE_SDDMM_PATH"] = "dense"

import oracle as O  # noqa: E402
import paper_2209_06979_b200 as mc  # noqa: E402
from paper_2209_06979_b200 import _native  # noqa: E402
from paper_2209_06979_b200.qint import COL_MAJOR, ROW_MAJOR  # noqa: E402

sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
s = O.build_sddmm_case(4096, 4096, 256, 8, sp, 8, 8, seed=1)
pat = mc.BcrsMatrix(4096, 4096, 8, s["offsets"], s["col_indices"],
                    mc.PackedArray.from_values(np.ones(s["col_indices"].size * 8), 8))
p = mc.SddmmProblem(mc.pack_dense(s["a"], 8, ROW_MAJOR), mc.pack_dense(s["b"], 8, COL_MAJOR), pat)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
b2b = len(sys.argv) > 2 and sys.argv[2] == "b2b"  # stamps of the last of 6 back-to-back launches
for rep in range(3):
    _native.load().mc_l2_flush(flush.data_ptr(), flush.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if b2b:
        if rep == 0:
            mc.kernels.sddmm_device(p, check_status=False)  # device copies + tensor maps cached
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            with torch.cuda.graph(graph, stream=cap):
                for _ in range(6):
                    mc.kernels.sddmm_device(p, stream=cap, check_status=False)
        graph.replay()
    else:
        mc.kernels.sddmm_device(p, check_status=False)
    e1.record()
    torch.cuda.synchronize()
    print("kernel ms", e0.elapsed_time(e1))
lib = _native.load()
buf = (ctypes.c_ulonglong * (148 * 128))()
lib.mc_debug_timeline(buf, 148 * 128)
t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 128).astype(np.int64)
base = t[:, 0].min()
names = {0: "start", 1: "setup", 40: "search", 63: "end", 100: "binit", 101: "talloc", 102: "pdlw", 103: "prebar0", 104: "prebarB"}
for i in range(6):
    names[2 + i] = f"tma{i}"
    names[10 + i] = f"mma_go{i}"
    names[16 + i] = f"mma_done{i}"
    names[22 + 3 * i] = f"ep_built{i}"
    names[23 + 3 * i] = f"ep_full{i}"
    names[24 + 3 * i] = f"ep_done{i}"
for i in range(5):
    names[41 + 4 * i] = f"p1start{i}"
    names[42 + 4 * i] = f"p1done{i}"
    names[43 + 4 * i] = f"pempty_ok{i}"
for i in range(5):
    names[64 + 5 * i] = f"b_go{i}"
    names[65 + 5 * i] = f"b_loop{i}"
    names[66 + 5 * i] = f"b_red{i}"
    names[67 + 5 * i] = f"b_pempty{i}"
for i in range(5):
    names[90 + i] = f"b_land{i}"
for i in range(3):
    names[110 + i] = f"c_ld0_{i}"
    names[113 + i] = f"c_loop_{i}"
    names[116 + i] = f"c7_done{i}"
for cta in (0, 1, 77, 147):
    row = t[cta]
    ev = sorted((int(v - base), names.get(k, str(k))) for k, v in enumerate(row) if v >= base and v != 0)
    print(f"CTA {cta}: " + " ".join(f"{n}@{x / 1000:.1f}" for x, n in ev))
