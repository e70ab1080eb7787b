#!/bin/bash
# A/B: ktrace phase cycles + c2 bench for the base library and the working tree.
mkdir -p gpurun_out/ab
for v in base new; do
  if [ $v = base ]; then export RSIM_LIB=$PWD/paper_2008_01539_b200/lib/librsim_base.so; else unset RSIM_LIB; fi
  RSIM_KTRACE=1 timeout 300 python scripts/ktrace.py > gpurun_out/ab/ktrace_$v.log 2>&1
  timeout 300 python bench.py --steps 3 --warmup 3 --c5 "${C5:-}" --no-cpu > gpurun_out/ab/bench_$v.json 2>&1
done
