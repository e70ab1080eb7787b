#!/bin/bash
# Round-1 evidence refresh after the grid-Krylov pass fusions (x/r/next-p pass,
# s recompute, staged commits): gpu tests, bench JSON, ncu launch list of the
# bench command, full captures of the config-5 grid Krylov at 5 / 50 / 100 %
# and of the partial-set K1 row kernel.
set -x
O=gpurun_out/r01s4; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --c5 "" --flash-cells 0 > $O/ncu_launch.log 2>&1
for f in 1.0 0.5 0.05; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_assemble_row|k_assemble_full1|k_bicgstab" -c 2 \
    -o $O/full_c5_$f python scripts/prof_workload.py c5 $f > $O/ncu_c5_$f.log 2>&1
done
ls -la $O
