timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo ncu_rc=$?
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches.csv')))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; data=rows[hdr+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
seq=[(r[ki][:40], r[gi], float(r[vi].replace(',',''))) for r in data]
for s in seq[-12:]: print(s)
PY
