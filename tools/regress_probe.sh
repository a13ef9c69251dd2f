# round-1 library vs the current one on the same box: small M, pack, k-means, CG-shaped direct sum
for lib in build/var/libgenred_r1.so paper_2004_11127_b200/libgenred.so; do
  export GENRED_LIB=$lib
  echo "== $lib" >> gpurun_out/regress.log
  timeout 300 python tools/small_m_probe.py 2>&1 | head -6 >> gpurun_out/regress.log
  timeout 300 python tools/kmeans_probe.py >> gpurun_out/regress.log 2>&1
  timeout 300 python tools/ktime.py direct1e5:gauss:sum:1e5:1e5:0.05 gauss1e5:gauss:sum:1e5:1e5:0.5 >> gpurun_out/regress.log 2>&1
done
