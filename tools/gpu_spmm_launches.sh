#!/bin/bash
# Per-kernel device times of the C3 L8-R8 V=8 cells (launch list under ncu, cold caches).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/spmm_launches.csv python tools/bench_spmm.py ${1:-c3l8} > gpurun_out/spmm_ncu.log 2>&1; echo rc=$?
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/spmm_launches.csv')) if len(r)>10]
h=rows[0]; rows=rows[1:]
ik=h.index("Kernel Name"); iv=h.index("Metric Value")
agg=collections.OrderedDict()
for r in rows:
    k=r[ik][:90]; agg.setdefault(k,[0,0,[]]); agg[k][0]+=1; agg[k][1]+=float(r[iv].replace(',','')); agg[k][2].append(float(r[iv].replace(',','')))
for k,(n,t,l) in agg.items(): print(f"{n:5d} {t/n/1000:10.2f} us/launch  {k}  {[round(x/1000,1) for x in l[:12]]}")
PY
