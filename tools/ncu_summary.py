"""Print the headline counters of an ncu report (first kernel) as JSON.
usage: python tools/ncu_summary.py REPORT.ncu-rep [extra_metric ...]"""
import csv, io, json, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'l1tex__m_xbar2l1tex_read_bytes.sum', 'l1tex__m_xbar2l1tex_read_bytes.sum.per_second',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'lts__t_sectors_srcunit_tex_op_write.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'launch__shared_mem_per_block_dynamic', 'launch__grid_size', 'launch__block_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
STALLS = ['long_scoreboard', 'short_scoreboard', 'wait', 'selected', 'not_selected', 'math_pipe_throttle',
          'mio_throttle', 'lg_throttle', 'barrier', 'membar', 'no_instructions', 'dispatch_stall',
          'branch_resolving', 'sleeping', 'tex_throttle', 'drain']

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units, v = r[0], r[1], r[2]
res = {"kernel": v[h.index("Kernel Name")][:160]}
for k in KEYS + sys.argv[2:]:
    if k in h:
        i = h.index(k)
        res[k] = [units[i], v[i]]
tot = 0
st = {}
for s in STALLS:
    k = f"smsp__pcsamp_warps_issue_stalled_{s}"
    if k in h:
        st[s] = float(v[h.index(k)] or 0)
tot = sum(st.values()) or 1
res["stall_samples_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x}
print(json.dumps(res, indent=1))
