set -x
mkdir -p gpurun_out/r01p
ncu --set full --clock-control none --import-source on -k regex:'k_krylov_dsm' -s 60 -c 1 -o gpurun_out/r01p/full_c2_dsm_v2 python scripts/prof_workload.py c2 30 > gpurun_out/r01p/ncu_full_c2_dsm.log 2>&1
ls -la gpurun_out/r01p
