#!/bin/bash
# c2 headline under several cluster-kernel environment settings
mkdir -p gpurun_out/ab
for cfg in "default:" "lrc7:RSIM_DSM_MINLRC=7" "lrc8:RSIM_DSM_MINLRC=8" "lrc9:RSIM_DSM_MINLRC=9"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 --c5 "" > gpurun_out/ab/env_$name.json 2>&1
done
