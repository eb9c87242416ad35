#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, bench lines (ours + reference arm), the bench's
# launch list, and ncu --set full captures of the C2 / C3 / C4 / C5 kernels (gpurun_out/).
mkdir -p gpurun_out
bash tools/gpu_tests.sh
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --only c2 --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_c2_s050 \
  python tools/prof_case.py sddmm 0.5 dense 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:sddmm_tc -s 2 -c 1 -o gpurun_out/prof_c2_s090 \
  python tools/prof_case.py sddmm 0.9 dense 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:score_softmax -s 1 -c 1 -o gpurun_out/prof_c4 \
  python tools/bench_attention.py --batch 4 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:spmm_seg -s 1 -c 1 -o gpurun_out/prof_c3_l8r4 \
  python tools/prof_case.py spmm 4096 512 4096 8 0.9 8 4 2 > /dev/null 2>&1
ls -la gpurun_out | tail -20
