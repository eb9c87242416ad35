#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench line, launch list, ncu of the top kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_c2_s050 python tools/prof_case.py sddmm 0.5 dense 3 > /dev/null 2>&1; echo ncu_rc=$?
