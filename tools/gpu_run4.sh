timeout 300 python -m pytest tests -q -m gpu -k "spmm" -x > gpurun_out/pytest_spmm.log 2>&1; echo spmm_tests_rc=$?; tail -2 gpurun_out/pytest_spmm.log
timeout 900 python tools/bench_spmm.py c1 c3 c5 --out gpurun_out/spmm_bench.json > gpurun_out/spmm_bench.log 2>&1; echo rc=$?
python3 -c "
import json
for r in json.load(open('gpurun_out/spmm_bench.json')):
    print(r['cfg'], r['pair'], 'V',r['V'], r['sparsity'], round(r['us'],2),'us', round(r['tops'],1),'TOPS', 'frac',round(r['roofline_frac'],3), r['exact_sampled_rows'])
"
tail -3 gpurun_out/spmm_bench.log
