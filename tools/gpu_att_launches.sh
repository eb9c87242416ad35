#!/bin/bash
# Launch list of one C4 attention layer (reduced batch) with per-kernel device times.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/att_launches.csv python tools/bench_attention.py --batch ${1:-8} > gpurun_out/att_ncu.log 2>&1; echo rc=$?
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/att_launches.csv')) if len(r)>10]
h=rows[0]; rows=rows[1:]
ik=h.index("Kernel Name"); iv=h.index("Metric Value")
agg=collections.OrderedDict()
for r in rows:
    k=r[ik][:70]; agg.setdefault(k,[0,0]); agg[k][0]+=1; agg[k][1]+=float(r[iv].replace(',',''))
for k,(n,t) in agg.items(): print(f"{n:5d} {t/1000:10.1f} us  {k}")
PY
