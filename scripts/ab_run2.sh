#!/bin/bash
# ktrace under several cluster-kernel settings (env), one log each
mkdir -p gpurun_out/ab
for cfg in "default:" "t512:RSIM_DSM_MINT=512" "lrc7:RSIM_DSM_MINLRC=7" "lrc8:RSIM_DSM_MINLRC=8"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs RSIM_KTRACE=1 timeout 300 python scripts/ktrace.py > gpurun_out/ab/kt_$name.log 2>&1
done
