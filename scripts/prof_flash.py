"""PR flash on 1M cells of the bench's Case-3 field (profiler-friendly, no timing):
  ncu --set full -k regex:k_flash python scripts/prof_flash.py [shuffled]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2008_01539_b200 as pkg  # noqa: E402

p, z, rng = bench.flash_field(1 << 20)
if len(sys.argv) > 1 and sys.argv[1] == "shuffled":
    perm = rng.permutation(len(p))
    p, z = p[perm], z.reshape(-1, 2)[perm].reshape(-1)
o = pkg.eos_flash(pkg.eos_case3(), 340.0, p, z.reshape(-1, 2))
print("two-phase fraction", float((o["status"] == 2).mean()), "mean iterations", float(o["iters"].mean()))
