"""Summarise an ncu report's SASS page: hottest basic blocks (by stall samples) with exec counts.
usage: python tools/sass_hot.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(int(x[iS]) for x in rows)
totE = sum(int(x[iE]) for x in rows)
print("samples", tot, "warp-instructions", totE)
seg, cur = [], None
for i, x in enumerate(rows):
    e, s = int(x[iE]), int(x[iS])
    if cur and cur[0] == e:
        cur[2] += s; cur[3] = i; cur[4] += 1
    else:
        cur = [e, i, s, i, 1]; seg.append(cur)
for e, a, s, b, n in sorted(sorted(seg, key=lambda c: -c[2])[:top], key=lambda c: c[1]):
    print(f"rows {a:5d}-{b:5d} n={n:4d} exec={e:10d} inst={e*n:11d} samples={s:6d} ({100*s/tot:4.1f}%) "
          f"{rows[a][1].strip()[:48]}")
