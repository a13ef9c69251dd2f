# Round-2 measurement pass: bench lines, ncu --set full of the main kernels, launch lists.
set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02/smi.txt
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02/bench_c$c.log 2>&1; done
timeout 900 python bench.py --config 2 --dist GMM3 --steps 10 --warmup 3 > gpurun_out/r02/bench_c2_gmm.log 2>&1
for n in 1 8 32; do timeout 600 python bench.py --config 6 --edge-n $n --steps 10 --warmup 3 > gpurun_out/r02/bench_edge$n.log 2>&1; done
timeout 900 python bench.py --mode jshard --config 7 --steps 5 --warmup 3 > gpurun_out/r02/bench_j7.log 2>&1
timeout 900 python bench.py --mode jshard --config 8 --steps 5 --warmup 3 > gpurun_out/r02/bench_j8.log 2>&1
# ncu (each command ran clean above or right before)
python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/r02/plain_fused.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02/ncu_fused python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/r02/ncu_fused.log 2>&1
python tools/profile_run.py --what lse --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02/plain_lse.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lse_kernel -s 1 -c 1 -o gpurun_out/r02/ncu_lse python tools/profile_run.py --what lse --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02/ncu_lse.log 2>&1
python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02/plain_gauss.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02/ncu_gauss python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02/ncu_gauss.log 2>&1
python tools/profile_run.py --what gauss --M 1000 --N 1000 --reps 3 > gpurun_out/r02/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sum_small -s 1 -c 1 -o gpurun_out/r02/ncu_c1 python tools/profile_run.py --what gauss --M 1000 --N 1000 --reps 3 > gpurun_out/r02/ncu_c1.log 2>&1
python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 2 > gpurun_out/r02/plain_knn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:knn_tc -s 1 -c 1 -o gpurun_out/r02/ncu_knn python tools/profile_run.py --what argk --M 10000 --N 60000 --D 784 --K 10 --reps 2 > gpurun_out/r02/ncu_knn.log 2>&1
# summaries on the box (the .ncu-rep files are large: gpurun brings back at most 64 MiB)
for r in fused lse gauss c1 knn; do
  if [ -f gpurun_out/r02/ncu_$r.ncu-rep ]; then
    python tools/ncu_summary.py gpurun_out/r02/ncu_$r.ncu-rep gpurun_out/r02/r02_ncu_$r.md > /dev/null 2>&1
    ncu -i gpurun_out/r02/ncu_$r.ncu-rep --page raw --csv > gpurun_out/r02/r02_ncu_${r}_raw.csv 2>/dev/null
    ncu -i gpurun_out/r02/ncu_$r.ncu-rep --page source --csv > gpurun_out/r02/r02_ncu_${r}_source.csv 2>/dev/null
    gzip -f gpurun_out/r02/r02_ncu_${r}_source.csv
    sz=$(stat -c %s gpurun_out/r02/ncu_$r.ncu-rep); if [ $sz -gt 12000000 ]; then rm -f gpurun_out/r02/ncu_$r.ncu-rep; fi
  fi
done
# launch list of C1 bench steps
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02/plain_c1bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_c1.csv python bench.py --config 1 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02/ncu_c1bench.log 2>&1
