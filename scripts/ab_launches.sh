#!/bin/bash
# Needs the comparison tree: git worktree add _prev a831c67 && (cd _prev && python -c "from paper_2008_01539_b200 import build; build.build()")
# per-launch durations of the grid BiCGSTAB over the whole config-4 run, HEAD vs _prev
O=gpurun_out/ab5; mkdir -p $O
for d in . _prev; do
  n=$( [ $d = . ] && echo head || echo prev )
  ( cd $d; timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bicgstab -c 2000 --csv \
      --log-file /tmp/l_$n.csv python scripts/full_runs.py 4 localized > /tmp/l_$n.log 2>&1 )
  cp /tmp/l_$n.csv $O/launch_$n.csv; gzip -f $O/launch_$n.csv
done
ls -la $O
