set -x
for lib in build/var/libgenred_rp0.so build/var/libgenred_rp1.so; do
  GENRED_LIB=$lib python tools/ktime.py fused:gauss_sum_gradx:sum:1e5:1e5:0.5 fused2:gauss_sum_gradx:sum:4e5:4e5:0.5 gradx:gauss_gradx:sum:4e5:4e5:0.5 >> gpurun_out/rp.log 2>&1
done
timeout 900 python -m pytest tests -q -m gpu -rf -k "grad or fused or autograd or c2 or c1 or range or random or lse" > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest2.log
