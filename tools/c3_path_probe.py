"""C3 cells on a forced SpMM path (MCUBE_SPMM_PATH from the environment), for dispatch tuning.
usage: MCUBE_SPMM_PATH=dense|mma python tools/c3_path_probe.py <V> <sparsity> [...]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench_spmm as B  # noqa: E402
import oracle as O  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
vs = [int(x) for x in sys.argv[1].split(",")]
sps = [float(x) for x in sys.argv[2].split(",")]
for lb, rb in B.PAIRS:
    for v in vs:
        for sp in sps:
            seed = O.cell_seed(0, ((4096, 512, 4096), v, sp, f"L{lb}-R{rb}"))
            r = B.cell(4096, 512, 4096, v, sp, lb, rb, seed, flush)
            print(os.environ.get("MCUBE_SPMM_PATH"), f"L{lb}-R{rb}", v, sp, round(r["us"], 1), r["exact_sampled_rows"], flush=True)
