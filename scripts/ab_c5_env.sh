#!/bin/bash
# config-5 Krylov micro (50 iterations) at several active fractions under env overrides:
#   scripts/ab_c5_env.sh "RSIM_KALT=1" ...
O=gpurun_out/ab5; mkdir -p $O
{
for f in ${FRACS:-0.05 0.2 0.5 1.0}; do
  for e in "X=1" "$@"; do
    env $e KC4_CONFIG=5 KC4_FRAC=$f python scripts/krylov_c4.py 50 3 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$e', '$f', round(d['ms'], 3), round(d['alg_GBs']), d['x_sha'])"
  done
done
} > $O/c5env.log 2>&1
cat $O/c5env.log
