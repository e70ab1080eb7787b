#!/bin/bash
mkdir -p gpurun_out/ab
for g in 0 16 32 64 128; do
  if [ $g = 0 ]; then unset RSIM_K7_COOP_GRID; else export RSIM_K7_COOP_GRID=$g; fi
  timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --c5 "" > gpurun_out/ab/k7g_$g.json 2>&1
done
