"""Launch one hot-path kernel configuration a few times (for ncu captures).

usage: python tools/prof_case.py sddmm <sparsity> [dense|gather] [reps]
       python tools/prof_case.py spmm <M> <N> <K> <V> <sparsity> <L> <R> [reps]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (input generation only)
import paper_2209_06979_b200 as mc  # noqa: E402
from paper_2209_06979_b200.qint import COL_MAJOR, ROW_MAJOR  # noqa: E402


def main():
    op = sys.argv[1]
    if op == "sddmm":
        sp = float(sys.argv[2])
        if len(sys.argv) > 3:
            os.environ["MCUBE_SDDMM_PATH"] = sys.argv[3]
        reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
        s = O.build_sddmm_case(4096, 4096, 256, 8, sp, 8, 8, seed=1)
        pat = mc.BcrsMatrix(4096, 4096, 8, s["offsets"], s["col_indices"],
                            mc.PackedArray.from_values(np.ones(s["col_indices"].size * 8), 8))
        p = mc.SddmmProblem(mc.pack_dense(s["a"], 8, ROW_MAJOR), mc.pack_dense(s["b"], 8, COL_MAJOR), pat)
        for _ in range(reps):
            mc.kernels.sddmm_device(p)
    else:
        m, n, k, v = (int(x) for x in sys.argv[2:6])
        sp = float(sys.argv[6])
        lb, rb = int(sys.argv[7]), int(sys.argv[8])
        reps = int(sys.argv[9]) if len(sys.argv) > 9 else 3
        c = O.build_spmm_case(m, n, k, v, sp, lb, rb, seed=1)
        lhs = mc.SrBcrsMatrix(m, k, v, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                              mc.PackedArray.from_values(c["values"], lb), shuffled=c["shuffled"])
        p = mc.SpmmProblem(lhs, mc.pack_dense(c["rhs"], rb))
        for _ in range(reps):
            mc.kernels.spmm_device(p)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
