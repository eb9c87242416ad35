timeout 300 python -m pytest tests -q -m gpu -k "sddmm" -x > gpurun_out/pytest_tc.log 2>&1; echo tc_rc=$?
tail -3 gpurun_out/pytest_tc.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'frac', d['roofline']['frac'])
for k,v in d['sweep'].items(): print(k, round(v['us'],2), 'us', round(v['tops'],1), 'TOPS', round(v['roofline_frac'],3))
"
tail -3 gpurun_out/bench.err
