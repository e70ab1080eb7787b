"""Device-resident time of one config-2 localized run (bench per_config.c2 workload):
median of 5 runs after 3 warm-ups, CUDA events; env knobs (RSIM_DSM_*) pass through."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2008_01539_b200 as pkg
cfg = int(os.environ.get("C2T_CONFIG", "2"))
R = bench.GpuRun(pkg, cfg, "localized")
for _ in range(3):
    R.run_dev()
ms = []
for _ in range(5):
    t, r = R.timed_dev()
    ms.append(t)
print(json.dumps({"config": cfg, "ms": float(np.median(ms)), "min": float(np.min(ms)), "lin": r["lin_iters"],
                  "sum_na": r["sum_na"], "rate": r["sum_na"] / (np.median(ms) / 1e3),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("RSIM_")}}), flush=True)
