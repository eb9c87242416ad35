#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the gather, packer, tcgen05 and
# attention paths (small golden cases + smoke). Logs into gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='test_spmm_segment_path_vs_oracle or test_spmm_golden or test_sddmm_golden or test_device_packer or test_attention_parity_golden or test_sddmm_paths_vs_oracle or test_spmm_l8r8_paths_vs_oracle or test_spmm_dense_path_vs_oracle'
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "$SEL" -p no:cacheprovider \
     > gpurun_out/sanitizer_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_${tool}.log
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
     python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_${tool}_smoke.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_${tool}_smoke.log
done
for f in gpurun_out/sanitizer_*.log; do echo "== $f"; tail -4 $f; done
