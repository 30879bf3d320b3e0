"""Stall-sample breakdown of one kernel from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv).
Development aid: python tools/ncu_stalls.py X.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
f = lambda r, c: float(r[ix[c]] or 0)
tot = sum(f(r, S) for r in data)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(f(r, c) for r in data) for c in cols}
print(f"samples {tot:.0f}:", ", ".join(f"{c[6:]} {v / tot * 100:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0))
# by phase: contiguous address ranges split at the instruction with the most DFMA density
for r in sorted(data, key=lambda r: -f(r, S))[:top_n]:
    st = sorted(((f(r, c), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{r[0][-5:]} {f(r, S):5.0f}  {r[1].strip()[:58]:58s} {st[0][1]} {st[0][0]:.0f} {st[1][1]} {st[1][0]:.0f}")
