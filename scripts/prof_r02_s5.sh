#!/bin/bash
# Round-2 evidence after the planar-ELL / pressure-only-block change: Krylov
# micro timings (config 4 / 3 first Newton systems, config 5 at 20 / 50 / 100 %),
# launch list of the headline bench command and full captures (with source) of
# the grid BiCGSTAB on the config-4 system and on config 5.
set -x
O=gpurun_out/r02s5; mkdir -p $O
{
python scripts/krylov_c4.py 100 3
KC4_CONFIG=3 python scripts/krylov_c4.py 100 3
for f in 0.05 0.2 0.5 1.0; do KC4_CONFIG=5 KC4_FRAC=$f python scripts/krylov_c4.py 50 3; done
} > $O/krylov_micro.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 1 --warmup 3 --configs '' --c5 '' --flash-cells 0 --direct 0 --paper 0 --no-cpu > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c4.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab --launch-skip 1 -c 1 \
    -o $O/ncu_c4_krylov python scripts/krylov_c4.py 20 1 > $O/ncu_c4.log 2>&1
for f in 1.0 0.2; do
KC4_CONFIG=5 KC4_FRAC=$f timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab --launch-skip 1 -c 1 \
    -o $O/ncu_c5_krylov_$f python scripts/krylov_c4.py 10 1 > $O/ncu_c5_$f.log 2>&1
done
ls -la $O
