timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest3.log
python tools/ktime.py fused:gauss_sum_gradx:sum:1e5:1e5:0.5 gradx:gauss_gradx:sum:1e5:1e5:0.5 gauss:gauss:sum:1e5:1e5:0.5 > gpurun_out/kt_e.log 2>&1
