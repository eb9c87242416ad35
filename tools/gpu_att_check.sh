#!/bin/bash
# Attention path: parity tests + C4 timing.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "attention or multi_head or sddmm" > gpurun_out/pytest_att.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_att.log
timeout 600 python tools/bench_attention.py --out gpurun_out/att_c4.json > gpurun_out/att_c4.log 2>&1; echo att_rc=$?; tail -2 gpurun_out/att_c4.log
