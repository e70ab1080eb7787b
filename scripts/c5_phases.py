"""Config-5 phase timings only (K7 / K1 / 50 BiCGSTAB per active fraction), the
bench's own c5_sweep without the config-2 workload — for kernel tuning runs:
  python scripts/c5_phases.py 1.0,0.05 [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2008_01539_b200 as pkg  # noqa: E402

fr = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1.0").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.8
for r in bench.c5_sweep(pkg, fr, reps, hbm):
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
