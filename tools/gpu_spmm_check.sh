#!/bin/bash
# SpMM paths: parity tests + C1/C3/C5 timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "spmm" > gpurun_out/pytest_spmm.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_spmm.log | grep -v "^  " | tail -8
