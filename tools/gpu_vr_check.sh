#!/bin/bash
# SDDMM tile height experiment: parity with VR=16 forced, then the bench sweep at VR=16 / 32.
mkdir -p gpurun_out
MCUBE_SDDMM_VR=16 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sddmm" > gpurun_out/pytest_vr16.log 2>&1; echo vr16_pytest_rc=$?; tail -1 gpurun_out/pytest_vr16.log
for vr in 16 32; do
  MCUBE_SDDMM_VR=$vr timeout 300 python bench.py > gpurun_out/bench_vr$vr.json 2> gpurun_out/bench_vr$vr.err
  python3 -c "
import json;d=json.load(open('gpurun_out/bench_vr$vr.json'))
print('VR=$vr', round(d['value'],1), d['ms_per_step'], {k:round(v['us'],2) for k,v in d['sweep'].items()})"
done
