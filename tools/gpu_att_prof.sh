#!/bin/bash
# Fused attention kernel: launch list + one full ncu capture with source counters.
mkdir -p gpurun_out
bash tools/gpu_att_launches.sh 8
timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_softmax -s 2 -c 1 -o gpurun_out/prof_att python tools/bench_attention.py --batch 4 > gpurun_out/att_prof.log 2>&1; echo ncu_rc=$?
