set -x
for lib in build/var/libgenred_hh2.so build/var/libgenred_hh8.so paper_2004_11127_b200/libgenred.so; do
  GENRED_LIB=$lib python tools/ktime.py fused:gauss_sum_gradx:sum:1e5:1e5:0.5 fused2:gauss_sum_gradx:sum:4e5:4e5:0.5 >> gpurun_out/rp2.log 2>&1
done
python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/plain_fused.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02_fused_rp python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/ncu_fused.log 2>&1
