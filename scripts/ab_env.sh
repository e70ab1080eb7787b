#!/bin/bash
# whole c3 / c4 localized runs under environment-variable tuning overrides:
#   scripts/ab_env.sh "RSIM_FUSE_MAX_ROWS=0" "RSIM_FUSE_MAX_ROWS=300000" ...
O=gpurun_out/ab5; mkdir -p $O
{
for e in "X=1" "$@" "X=2"; do
  for c in ${CONFIGS:-3 4}; do env $e python scripts/full_runs.py $c localized 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$e', 'c$c', d['wall_s'], d['iterations'], d['lin_iters'])"; done
done
} > $O/env.log 2>&1
cat $O/env.log
