#!/bin/bash
mkdir -p gpurun_out/ab
for v in base new; do
  if [ $v = base ]; then export RSIM_LIB=$PWD/paper_2008_01539_b200/lib/librsim_base.so; else unset RSIM_LIB; fi
  timeout 600 python bench.py --no-cpu --steps 1 --warmup 3 --c5-ilu "" --c5 "${C5:-0.05,0.2,1.0}" > gpurun_out/ab/c5_$v.json 2>&1
done
