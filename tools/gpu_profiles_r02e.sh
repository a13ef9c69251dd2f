# Tile-centred form (R18j): ncu of the LSE and direct-width Gaussian kernels, and the launch list
# of one tile-centred call.
mkdir -p gpurun_out/r02e
python tools/profile_run.py --what lse --reps 2 > gpurun_out/r02e/plain_lse.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lse_local -s 1 -c 1 -o gpurun_out/r02e/ncu_lse_local python tools/profile_run.py --what lse --reps 2 > gpurun_out/r02e/ncu_lse.log 2>&1
python tools/ncu_summary.py gpurun_out/r02e/ncu_lse_local.ncu-rep gpurun_out/r02e/r02_ncu_lse_local.md > /dev/null 2>&1
ncu -i gpurun_out/r02e/ncu_lse_local.ncu-rep --page source --csv > gpurun_out/r02e/lse_local_source.csv 2>/dev/null
ncu -i gpurun_out/r02e/ncu_lse_local.ncu-rep --page raw --csv > gpurun_out/r02e/r02_ncu_lse_local_raw.csv 2>/dev/null; rm -f gpurun_out/r02e/ncu_lse_local.ncu-rep
ncu --set full --clock-control none -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02e/ncu_gauss_local python tools/profile_run.py --what gauss --scale 0.05 --reps 2 > gpurun_out/r02e/ncu_gauss_local.log 2>&1
python tools/ncu_summary.py gpurun_out/r02e/ncu_gauss_local.ncu-rep gpurun_out/r02e/r02_ncu_gauss_local.md > /dev/null 2>&1
ncu -i gpurun_out/r02e/ncu_gauss_local.ncu-rep --page raw --csv > gpurun_out/r02e/r02_ncu_gauss_local_raw.csv 2>/dev/null; rm -f gpurun_out/r02e/ncu_gauss_local.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e/launches_local.csv python tools/profile_run.py --what gauss --scale 0.05 --reps 1 > gpurun_out/r02e/launches_local.log 2>&1
