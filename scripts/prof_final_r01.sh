#!/bin/bash
# Round-1 evidence (two calls, each < 64 MiB of output):
#   part A: bench JSON, ncu launch list of the bench command, full capture of the
#           c2 dominant kernel (cluster Krylov);
#   part B: full captures of config-5 K1 / K7 / grid Krylov and c2 K1/K6/K7.
set -x
O=gpurun_out/r01f; mkdir -p $O
if [ "$1" = A ]; then
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --c5 "" > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_krylov_dsm -s 60 -c 1 -o $O/full_c2_krylov_dsm \
    python scripts/prof_workload.py c2 30 > $O/ncu_c2.log 2>&1
else
ncu --set full --clock-control none --import-source on -k regex:"k_assemble|k_update|k_scatter|k_dilate" -s 200 -c 4 -o $O/full_c2_other \
    python scripts/prof_workload.py c2 30 > $O/ncu_c2b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_assemble_row|k_bicgstab|k_dilate_rg|k_scatter_rg|k_reset_seed|k_scan_tiles" -c 7 \
    -o $O/full_c5 python scripts/prof_workload.py c5 1.0 > $O/ncu_c5.log 2>&1
fi
ls -la $O
