#!/bin/bash
# config-5 Krylov micro (50 iterations) at several active fractions: HEAD vs lib/ab variants
O=gpurun_out/ab5; mkdir -p $O
{
for f in ${FRACS:-0.05 0.2 0.5 1.0}; do
  KC4_CONFIG=5 KC4_FRAC=$f python scripts/krylov_c4.py 50 3 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('head', '$f', round(d['ms'], 3), round(d['alg_GBs']), d['x_sha'])"
  for v in "$@"; do
    RSIM_LIB=$PWD/paper_2008_01539_b200/lib/ab/librsim_$v.so KC4_CONFIG=5 KC4_FRAC=$f python scripts/krylov_c4.py 50 3 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('$v', '$f', round(d['ms'], 3), round(d['alg_GBs']), d['x_sha'])"
  done
done
} > $O/c5.log 2>&1
cat $O/c5.log
