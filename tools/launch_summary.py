"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel and grid:
    python tools/launch_summary.py gpurun_out/launches_C3.csv
The list holds one V-cycle (replayed graph) followed by the isolated hot kernels (bench.py --profile);
ncu times are cold-cache and serialised: compare shares, not absolute times."""
import collections
import csv
import re
import sys

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, gi, vi, ui = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
total = 0.0
for r in rows[1:]:
    us = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1e-3)
    name = re.sub(r"\(Tables.*|\(long.*|\(const .*|\(int .*|\(Cg1Args.*", "", r[ki]).strip()
    key = (name, r[gi])
    n, t = agg.get(key, (0, 0.0))
    agg[key] = (n + 1, t + us)
    total += us
print(f"total {total:.1f} us over {sum(n for n, _ in agg.values())} launches")
for (name, grid), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.1f} us {100 * t / total:5.1f}%  {n:3d}x {name} {grid}")
