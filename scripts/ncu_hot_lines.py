"""Warp-stall samples of one kernel in an `ncu --set full --import-source on` report,
per CUDA source line (cuda,sass view):  python scripts/ncu_hot_lines.py rep.ncu-rep kernel_regex [N]"""
import csv
import io
import os
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
fpath, iss, hdr = "", None, None
lines = []
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fpath = os.path.basename(r[1])
    elif r and r[0] == "Line No":
        hdr = r
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        iex = hdr.index("Instructions Executed")
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        lines.append((int(r[iss] or 0), int(r[iex] or 0), f"{fpath}:{r[0]}", r[1].strip()[:120]))
tot = sum(l[0] for l in lines) or 1
print(f"total samples {tot}")
for s, ex, loc, src in sorted(lines, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  inst {ex:>12}  {loc:22} {src}")
