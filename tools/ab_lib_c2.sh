#!/bin/bash
# same-box A/B of libmcube builds on the C2 sweep: tools/ab_lib_c2.sh libA.so libB.so ... (2 rounds)
mkdir -p gpurun_out
for round in 1 2; do
  for lib in "$@"; do
    MCUBE_LIB_PATH=$PWD/paper_2209_06979_b200/$lib python bench.py --only c2 --no-cpu-baseline --steps 20 --warmup 5 2>gpurun_out/ab_err.txt | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['value'],1), {k:round(c['us'],2) for k,c in d['sweep'].items()}, 'exact', d['validation']['sampled_rows_exact'])" || tail -3 gpurun_out/ab_err.txt
  done
done
