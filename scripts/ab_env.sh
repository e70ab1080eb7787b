#!/bin/bash
# A/B of one tuning env variable on config-5 phases: ab_env.sh VAR "v1 v2 ..." [fractions]
mkdir -p gpurun_out/ab
VAR=$1; VALS=$2; FR=${3:-0.05,0.2,1.0}
for v in $VALS; do
  env $VAR=$v timeout 600 python scripts/c5_phases.py $FR 3 > gpurun_out/ab/env_${VAR}_$v.json 2>&1
done
