"""Summarise an ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list: per-kernel launches, total / mean
time, share of the GPU time, DRAM bytes per launch and achieved DRAM GB/s.
  python scripts/ncu_summary.py launches.csv [--json out.json]"""
import collections
import csv
import json
import sys

UNIT_T = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}
UNIT_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    d = collections.defaultdict(dict)
    for r in rows[1:]:
        if not r[ii].isdigit():
            continue
        v = float(r[vi].replace(",", "")) if r[vi] not in ("", "n/a") else 0.0
        d[int(r[ii])][r[mi]] = (v, r[ui])
        d[int(r[ii])]["name"] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    return d


def summarise(d):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for _, m in sorted(d.items()):
        t, tu = m["gpu__time_duration.sum"]
        rb, ru = m.get("dram__bytes_read.sum", (0.0, "byte"))
        wb, wu = m.get("dram__bytes_write.sum", (0.0, "byte"))
        a = agg[m["name"]]
        a[0] += 1
        a[1] += t * UNIT_T.get(tu, 1e-9)
        a[2] += rb * UNIT_B.get(ru, 1) + wb * UNIT_B.get(wu, 1)
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": n, "total_ms": t * 1e3, "mean_us": t / n * 1e6, "share": t / tot,
                    "dram_bytes_per_launch": b / n, "dram_gbs": b / t / 1e9 if t else 0.0})
    return tot, out


if __name__ == "__main__":
    tot, out = summarise(load(sys.argv[1]))
    print(f"total GPU time {tot * 1e3:.3f} ms over {sum(o['launches'] for o in out)} launches\n")
    print("| kernel | launches | total ms | mean µs | share | DRAM B/launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|")
    for o in out:
        print(f"| {o['kernel']} | {o['launches']} | {o['total_ms']:.3f} | {o['mean_us']:.2f} | {o['share']:.1%} | "
              f"{o['dram_bytes_per_launch']:.3g} | {o['dram_gbs']:.0f} |")
    if "--json" in sys.argv:
        json.dump({"total_ms": tot * 1e3, "kernels": out}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
