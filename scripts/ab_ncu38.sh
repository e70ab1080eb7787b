#!/bin/bash
# Needs the comparison tree: git worktree add _prev a831c67 && (cd _prev && python -c "from paper_2008_01539_b200 import build; build.build()")
# full ncu capture of the 39th grid-BiCGSTAB launch of the config-4 run (head/prev ratio 1.5)
O=gpurun_out/ab5; mkdir -p $O
for d in . _prev; do
  n=$( [ $d = . ] && echo head || echo prev )
  ( cd $d; timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab --launch-skip 38 -c 1 \
      -o /tmp/ncu38_$n -f python scripts/full_runs.py 4 localized --steps 8 > /tmp/n_$n.log 2>&1; tail -3 /tmp/n_$n.log )
  cp /tmp/ncu38_$n.ncu-rep $O/
done
ls -la $O
