#!/bin/bash
# same-box A/B of run-time knobs on the C2 sweep: each argument is one env assignment list
# (quoted, space separated; "-" = defaults), e.g.
#   tools/ab_env_c2.sh - "MCUBE_SDDMM_G8_OFF=1" "MCUBE_SDDMM_GPW=2"
mkdir -p gpurun_out
for round in 1 2; do
  for v in "$@"; do
    envs=""
    [ "$v" != "-" ] && envs="$v"
    env $envs python bench.py --only c2 --no-cpu-baseline --steps 20 --warmup 5 2>gpurun_out/ab_err.txt | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', round(d['value'],1), {k:(round(c['us'],2), c['kernel'][:12]) for k,c in d['sweep'].items()}, 'exact', d['validation']['sampled_rows_exact'])" || tail -3 gpurun_out/ab_err.txt
  done
done
