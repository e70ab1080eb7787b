#!/bin/bash
# cluster-Krylov layout sweep: RSIM_DSM_MINLRC in {6,7,8}
for l in 6 7 8; do
  RSIM_DSM_MINLRC=$l RSIM_KTRACE=1 timeout 300 python scripts/ktrace.py > gpurun_out/ktrace_l$l.log 2>&1
  RSIM_DSM_MINLRC=$l timeout 300 python bench.py --steps 3 --warmup 3 --c5 "" --no-cpu > gpurun_out/bench_l$l.json 2>&1
done
timeout 300 python scripts/micro_krylov.py > gpurun_out/micro_krylov3.log 2>&1
