set -x
mkdir -p gpurun_out/r01p
python scripts/prof_workload.py c2 8 > gpurun_out/r01p/plain_c2.log 2>&1 || exit 1
python scripts/prof_workload.py c5 1.0 > gpurun_out/r01p/plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01p/launches_c2.csv python scripts/prof_workload.py c2 8 > gpurun_out/r01p/ncu_list_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01p/launches_c5.csv python scripts/prof_workload.py c5 1.0 > gpurun_out/r01p/ncu_list_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_assemble_row|k_bicgstab|k_dilate|k_scan_tiles|k_scatter' -c 6 -o gpurun_out/r01p/full_c5 python scripts/prof_workload.py c5 1.0 > gpurun_out/r01p/ncu_full_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_krylov_dsm|k_assemble|k_scatter' -s 200 -c 6 -o gpurun_out/r01p/full_c2 python scripts/prof_workload.py c2 4 > gpurun_out/r01p/ncu_full_c2.log 2>&1
ls -la gpurun_out/r01p
