#!/bin/bash
# c4 full size through the case runner for several limiter settings; per-iteration logs in gpurun_out/c4sweep/
mkdir -p gpurun_out/c4sweep
for L in "$@"; do
  d=gpurun_out/c4sweep/${L/,/_}
  RSIM_C4_LIMITER=$L timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import paper_2008_01539_b200 as pkg
m = pkg.simulate(4, 'localized', '$d', write_fields=False)
print('$L', json.dumps(m))"
done
