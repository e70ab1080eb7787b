"""Key metrics of every kernel in `ncu --set full` reports (markdown table):
duration, DRAM bytes read+written (the roofline `traffic`), DRAM and SM
throughput, occupancy, IPC, and the top warp-stall reasons.
  python scripts/ncu_full_summary.py rep1.ncu-rep [rep2 ...]"""
import collections
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
STALL = "smsp__pcsamp_warps_issue_stalled_"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "nsecond": 1e-9}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, row, units)}


def num(x):
    v, u = x
    try:
        return float(v.replace(",", "")) * UNIT.get(u, 1.0)
    except ValueError:
        return float("nan")


print("| report | kernel | grid x block | regs | duration | DRAM bytes | DRAM % peak | SM % | warps active % | IPC | top stalls |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for rep in sys.argv[1:]:
    for d in rows(rep):
        name = d["Kernel Name"][0].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        t = num(d["gpu__time_duration.sum"])
        b = num(d["dram__bytes_read.sum"]) + num(d["dram__bytes_write.sum"])
        st = {k[len(STALL):]: num(v) for k, v in d.items() if k.startswith(STALL) and not k.endswith("not_issued")
              and "_not_issued" not in k}
        tot = sum(v for v in st.values() if v == v) or 1.0
        top = ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st.items(), key=lambda x: -(x[1] if x[1] == x[1] else 0))[:3])
        print(f"| {rep.split('/')[-1]} | {name} | {d['launch__grid_size'][0]} x {d['launch__block_size'][0]} | "
              f"{d['launch__registers_per_thread'][0]} | {t * 1e6:.1f} µs | {b:.3g} | "
              f"{num(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
              f"{num(d['sm__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
              f"{num(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
              f"{num(d['sm__inst_executed.avg.per_cycle_active']):.2f} | {top} |")
