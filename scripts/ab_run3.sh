#!/bin/bash
mkdir -p gpurun_out/ab
RSIM_LIB=$PWD/paper_2008_01539_b200/lib/librsim_base.so timeout 300 python scripts/ktrace_c2.py > gpurun_out/ab/kc2_base.log 2>&1
for cfg in "default:" "t512:RSIM_DSM_MINT=512" "lrc7:RSIM_DSM_MINLRC=7" "lrc8:RSIM_DSM_MINLRC=8"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 python scripts/ktrace_c2.py > gpurun_out/ab/kc2_$name.log 2>&1
done
