#!/bin/bash
# same-box A/B of libmcube variants on the C2 sweep: tools/ab_c2.sh libA.so libB.so [rounds]
mkdir -p gpurun_out
R=${3:-3}
for r in $(seq 1 $R); do
  for lib in "$1" "$2"; do
    MCUBE_LIB_PATH=$PWD/paper_2209_06979_b200/$lib python bench.py --only c2 --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['value'],1), {k:round(v['us'],2) for k,v in d['sweep'].items()})"
  done
done
