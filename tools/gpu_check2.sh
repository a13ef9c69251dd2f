timeout 900 python -m pytest tests -q -m gpu -rf -k "small or fused or expanded or gradient or c1 or smoke or tiny" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_small.log
for st in 20 200; do timeout 600 python bench.py --config 1 --steps $st --warmup 5 --no-cpu > gpurun_out/bench_c1_$st.log 2>&1; done
python tools/host_overhead_probe.py > gpurun_out/c1_host_probe.txt 2>&1
