"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum --csv --log-file`):
  python scripts/launch_summary.py launches.csv [N]"""
import collections
import csv
import gzip
import sys

_open = gzip.open if sys.argv[1].endswith(".gz") else open
lines = [l for l in _open(sys.argv[1], "rt") if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
im = h.index("Metric Name")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
agg = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) == len(h) and r[iv] and r[im] == "gpu__time_duration.sum":
        agg[r[ik].split("(")[0]].append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-3))
tot = sum(sum(v) for v in agg.values())
print(f"total {tot / 1e3:.3f} ms over {sum(len(v) for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{k[:60]:60s} {len(v):6d} {sum(v) / len(v):9.2f} us  {100 * sum(v) / tot:5.1f}%")
