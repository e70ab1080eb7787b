#!/bin/bash
# A/B of the c2 headline workload: base library (RSIM_LIB) vs working tree, 2 alternating rounds
mkdir -p gpurun_out/ab
for k in 1 2; do
for v in base new; do
  if [ $v = base ]; then export RSIM_LIB=$PWD/paper_2008_01539_b200/lib/librsim_base.so; else unset RSIM_LIB; fi
  timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --c5 "" > gpurun_out/ab/c2_${v}_$k.json 2>&1
done
done
