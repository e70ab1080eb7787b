#!/bin/bash
# whole config-4 adaptive-DD runs under environment-variable tuning overrides
O=gpurun_out/ab6; mkdir -p $O
{
for e in "X=1" "$@"; do
  env $e python scripts/full_runs.py 4 adaptive_dd 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$e', 'c4dd', d['wall_s'], d['iterations'], d['lin_iters'])"
done
} > $O/envdd.log 2>&1
cat $O/envdd.log
