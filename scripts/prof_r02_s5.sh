#!/bin/bash
# Round-2 final evidence: GPU tests, bench lines (both arms), launch list of the headline
# bench command, full captures (with source) of the grid BiCGSTAB: the 39th solve of the
# config-4 run (mid-run system) and config 5 at 100 % / 20 %, K1 at 50 %.
set -x
O=gpurun_out/r02s5; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 1 --warmup 3 --configs '' --c5 '' --flash-cells 0 --direct 0 --paper 0 --no-cpu > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c4.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab --launch-skip 38 -c 1 \
    -o $O/ncu_c4_krylov -f python scripts/full_runs.py 4 localized --steps 8 > $O/ncu_c4.log 2>&1
for f in 1.0 0.2; do
KC4_CONFIG=5 KC4_FRAC=$f timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab --launch-skip 1 -c 1 \
    -o $O/ncu_c5_krylov_$f -f python scripts/krylov_c4.py 10 1 > $O/ncu_c5_$f.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble_row" -c 1 \
    -o $O/ncu_c5_k1_0.5 -f python scripts/prof_workload.py c5 0.5 > $O/ncu_c5_k1.log 2>&1
ls -la $O
