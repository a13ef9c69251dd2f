for lib in build/var/libgenred_*.so; do
  GENRED_LIB=$lib python tools/ktime.py fused:gauss_sum_gradx:sum:1e5:1e5:0.5 fused2:gauss_sum_gradx:sum:4e5:4e5:0.5 dfused:gauss_sum_gradx:sum:4e5:4e5:0.05 >> gpurun_out/rp3.log 2>&1
done
