#!/bin/bash
# Dense SDDMM path: parity tests, timeline, bench line.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sddmm" > gpurun_out/pytest_sddmm.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_sddmm.log
for s in 0.5 0.9; do timeout 120 python tools/timeline.py $s > gpurun_out/timeline_$s.txt 2>&1; cat gpurun_out/timeline_$s.txt | tail -5; done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step']); print({k:(round(v['us'],2),round(v['roofline_frac'],3)) for k,v in d['sweep'].items()})"
tail -3 gpurun_out/bench.err
