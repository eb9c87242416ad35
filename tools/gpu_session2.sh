#!/bin/bash
# Session-2 baseline measurement: GPU tests, bench, timeline, ncu full captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; cat gpurun_out/bench.json
timeout 120 python tools/timeline.py 0.5 > gpurun_out/timeline05.txt 2>&1
timeout 120 python tools/timeline.py 0.9 > gpurun_out/timeline09.txt 2>&1
cat gpurun_out/timeline09.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_sddmm_tc python tools/prof_case.py sddmm 0.9 dense 3 > gpurun_out/ncu_tc.log 2>&1; echo ncu_rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:spmm_kernel -s 2 -c 1 -o gpurun_out/prof_spmm python tools/prof_case.py spmm 4096 512 4096 8 0.9 8 8 3 > gpurun_out/ncu_spmm.log 2>&1; echo ncu_rc=$?
