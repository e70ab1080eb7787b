#!/bin/bash
# Optional comparison tree: git worktree add _prev a831c67 && (cd _prev && python -c "from paper_2008_01539_b200 import build; build.build()")
# A/B on one box: GPU test suite, then whole c3 / c4 localized runs of HEAD against the
# tree of commit a831c67 (_prev/, when present) and optional lib/ab/librsim_<name>.so variants.
O=gpurun_out/ab5; mkdir -p $O
run() { # name dir env
  ( cd $2; for c in 3 4; do env $3 python scripts/full_runs.py $c localized 2>&1 | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$1', 'c$c', d['wall_s'], d['iterations'], d['lin_iters'])"; done )
}
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $O/pytest.log
{
[ -d _prev ] && run prev _prev X=1
run head . X=1
for v in "$@"; do run $v . RSIM_LIB=$PWD/paper_2008_01539_b200/lib/ab/librsim_$v.so; done
[ -d _prev ] && run prev2 _prev X=1
run head2 . X=1
} > $O/runs.log 2>&1
cat $O/pytest.log $O/runs.log
