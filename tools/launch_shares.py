"""Per-kernel share of a ncu launch list (gpu__time_duration.sum, CSV).

    python tools/launch_shares.py gpurun_out/launches_TAG.csv > profiles/TAG_launch_shares.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    t = float(r[iv]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[r[iu]]
    name = r[ik].split("(const")[0].split("(jf::")[0]
    agg[name][0] += 1
    agg[name][1] += t
tot = sum(v[1] for v in agg.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 --warmup 3 --no-graph (cold, serialised)")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:5d} launches {t:10.1f} us {100 * t / tot:5.1f}%  avg {t / n:8.1f} us  {name[:90]}")
