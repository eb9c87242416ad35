#!/bin/bash
# GPU box: our bench line (+ optional reference arm), logs into gpurun_out/
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ -n "$WITH_REF" ]; then
  timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "ref rc=$?" >> gpurun_out/bench_ref.err
fi
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
