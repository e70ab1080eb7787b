#!/bin/bash
# Round-1 evidence refresh with the final K1 tile / K7 bitmap / grid-Krylov kernels.
#   A: gpu tests, bench JSON, ncu launch list of the bench command, c2 cluster-Krylov capture
#   B: full captures of the config-5 kernels at 100 % and 5 %
set -x
O=gpurun_out/r01g; mkdir -p $O
if [ "$1" = A ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --c5 "" > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_krylov_dsm -s 60 -c 1 -o $O/full_c2_krylov_dsm \
    python scripts/prof_workload.py c2 30 > $O/ncu_c2.log 2>&1
else
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reset_seed|k_dilate_bits|k_keep_rg|k_count_merge_rg|k_scan_tiles|k_scatter_kb|k_assemble_full1|k_bicgstab" -c 9 \
    -o $O/full_c5_100 python scripts/prof_workload.py c5 1.0 > $O/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_reset_seed|k_dilate_bits|k_keep_rg|k_count_merge_rg|k_scan_tiles|k_scatter_kb|k_assemble_row|k_bicgstab" -c 9 \
    -o $O/full_c5_05 python scripts/prof_workload.py c5 0.05 > $O/ncu_c5b.log 2>&1
fi
ls -la $O
