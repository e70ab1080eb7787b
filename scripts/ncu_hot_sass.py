"""Top SASS instructions of one kernel in an `ncu --set full` report by warp-stall
samples (source page), to locate stalls:  python scripts/ncu_hot_sass.py rep.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        data.append((int(r[iss] or 0), r[ia], r[isrc]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {a}  {src}")
