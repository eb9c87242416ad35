"""World-size-2 gloo tests of the multi-GPU partitioning (CPU, no GPU needed).

Each rank takes its row panel (SpMM / SDDMM) or head range (attention), computes
its slice with the oracle (the device kernels compute the same slice on a B200),
and the slices are all-gathered (the validation-only collective) and compared on
every rank with the unpartitioned oracle result.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2209_06979_b200 as mc
from paper_2209_06979_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _srbcrs(c, lb):
    return mc.SrBcrsMatrix(c["m"], c["k"], c["v"], c["stride"], c["row_begin"], c["row_end"],
                           c["col_indices"], mc.PackedArray.from_values(c["values"], lb),
                           shuffled=c["shuffled"])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ---- SpMM row panels (L8-R4, shuffled, ragged row lengths via 2 patterns) ----
        c = O.build_spmm_case(96, 40, 256, 8, 0.7, 8, 4, seed=7)
        m = _srbcrs(c, 8)
        parts = shard.row_panels(m, world)
        lo, hi = parts[rank]
        sub = shard.srbcrs_panel(m, lo, hi)
        mine = O.spmm(sub.row_begin, sub.row_end, sub.col_indices, sub._flat_values, 8, sub.stride,
                      sub.shuffled, 8, c["rhs"], 4, 256)
        full = shard.allgather_rows(torch.from_numpy(mine), parts, 8).numpy()
        want = O.spmm(c["row_begin"], c["row_end"], c["col_indices"], c["values"], 8, c["stride"], True,
                      8, c["rhs"], 4, 256)
        ok_spmm = bool((full == want).all())

        # ---- SDDMM pattern panels ----
        s = O.build_sddmm_case(64, 48, 64, 4, 0.6, 8, 8, seed=3)
        pat = mc.BcrsMatrix(64, 48, 4, s["offsets"], s["col_indices"],
                            mc.PackedArray.from_values(np.ones(s["col_indices"].size * 4), 8))
        pparts = shard.pattern_panels(pat, world)
        lo, hi = pparts[rank]
        sub = shard.bcrs_panel(pat, lo, hi)
        vals = O.sddmm(s["a"][lo * 4:hi * 4], s["b"], sub.row_offsets, sub.col_indices, 4, 8, 8)
        blocks = [(int(s["offsets"][b]) - int(s["offsets"][a])) for a, b in pparts]
        mine_t = torch.from_numpy(vals.reshape(-1, 4))
        width = max(blocks)
        pad = torch.zeros((width, 4), dtype=torch.int32)
        pad[:mine_t.shape[0]] = mine_t
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        got = torch.cat([bufs[r][:blocks[r]] for r in range(world)]).numpy().reshape(-1)
        ok_sddmm = bool((got == O.sddmm(s["a"], s["b"], s["offsets"], s["col_indices"], 4, 8, 8)).all())

        # ---- attention batch x head ranges ----
        a = O.build_attention_case(32, 16, 0.75, seed=5)
        rng = np.random.default_rng(9)
        heads = 3
        qkv = [rng.normal(size=(heads, 32, 16)) for _ in range(3)]
        hparts = shard.head_ranges(heads, world)
        h0, h1 = hparts[rank]
        outs = [O.attention(qkv[0][h], qkv[1][h], qkv[2][h], a["offsets"], a["col_indices"], 32, 16, 8, 8)["output"]
                for h in range(h0, h1)]
        mine = torch.from_numpy(np.stack(outs) if outs else np.zeros((0, 32, 16)))
        full = shard.allgather_rows(mine, hparts, 1).numpy()
        want = np.stack([O.attention(qkv[0][h], qkv[1][h], qkv[2][h], a["offsets"], a["col_indices"], 32, 16,
                                     8, 8)["output"] for h in range(heads)])
        ok_att = bool((full == want).all())
        q.put((rank, ok_spmm, ok_sddmm, ok_att, parts, pparts, hparts))
    finally:
        dist.destroy_process_group()


def test_row_panel_partition_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_spmm, ok_sddmm, ok_att, parts, pparts, hparts in res:
        assert ok_spmm and ok_sddmm and ok_att, (rank, ok_spmm, ok_sddmm, ok_att)
        assert parts[0][0] == 0 and parts[-1][1] == 12 and parts[0][1] == parts[1][0]


def test_balanced_cuts_and_alignment():
    c = O.build_spmm_case(256, 16, 128, 2, 0.5, 4, 4, seed=1)
    m = _srbcrs(c, 4)
    for world in (1, 2, 3, 8):
        parts = shard.row_panels(m, world)
        assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == m.vector_rows
        for lo, hi in parts:
            sub = shard.srbcrs_panel(m, lo, hi)
            assert sub.vector_rows == hi - lo
            want = O.srbcrs_dense(256, 128, 2, c["stride"], c["row_begin"], c["row_end"], c["col_indices"],
                                  c["values"], shuffled=True)[lo * 2:hi * 2]
            assert (mc.srbcrs_to_dense(sub) == want).all()
    assert shard.head_ranges(512, 8)[3] == (192, 256)


def test_bench_c2_row_panels_partition_one_problem():
    """bench.py at N ranks: every rank's C2 panel is a slice of ONE global problem of
    M = 4096 * N rows (weak scaling), and the panels tile it exactly."""
    import bench
    world = 2
    panels = [bench.c2_rank_cases(r, world) for r in range(world)]
    for i, s in enumerate(bench.SPARSITIES):
        seed = O.cell_seed(0, ((bench.M * world, bench.N, bench.K), bench.V, s, "L8-R8"))
        g = O.build_sddmm_case(bench.M * world, bench.N, bench.K, bench.V, s, 8, 8, seed)
        offs = np.concatenate([[0]] + [p[i][1]["offsets"][1:] + sum(int(q[i][1]["offsets"][-1]) for q in panels[:r])
                                       for r, p in enumerate(panels)])
        assert (offs == g["offsets"]).all()
        assert (np.concatenate([p[i][1]["col_indices"] for p in panels]) == g["col_indices"]).all()
        assert (np.concatenate([p[i][1]["a"] for p in panels]) == g["a"]).all()
        assert all((p[i][1]["b"] == g["b"]).all() for p in panels)
    # world = 1 is exactly the C2 configuration (the reference cell seed of M = 4096)
    one = bench.c2_rank_cases(0, 1)
    seed = O.cell_seed(0, ((bench.M, bench.N, bench.K), bench.V, 0.9, "L8-R8"))
    g = O.build_sddmm_case(bench.M, bench.N, bench.K, bench.V, 0.9, 8, 8, seed)
    assert (one[2][1]["col_indices"] == g["col_indices"]).all()
