python tools/ktime.py gauss:gauss:sum:1e5:1e5:0.5 fused:gauss_sum_gradx:sum:1e5:1e5:0.5 gradx:gauss_gradx:sum:1e5:1e5:0.5 gauss3e5:gauss:sum:3e5:3e5:0.5 gauss2e4:gauss:sum:2e4:2e4:0.5 direct1e5:gauss:sum:1e5:1e5:0.05 > gpurun_out/var19.log 2>&1
timeout 900 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/bench_c2.log 2>&1
