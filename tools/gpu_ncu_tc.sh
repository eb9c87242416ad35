#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_tc_v4 python tools/prof_case.py sddmm ${1:-0.9} dense 3 > gpurun_out/ncu_tc_v3.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_tc_v3.log
