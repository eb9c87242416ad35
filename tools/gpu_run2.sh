set -x
timeout 300 python -m pytest tests -q -m gpu -k "sddmm_paths or dense_c2" -x > gpurun_out/pytest_tc.log 2>&1; echo tc_rc=$?
tail -25 gpurun_out/pytest_tc.log
timeout 600 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 2500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
