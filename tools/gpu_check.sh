# Round-2 GPU check: full -m gpu suite, then bench lines of C2/C3/C4/C1 and C5 (short) -> gpurun_out/
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
for c in 2 3 4 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_c$c.log 2>&1; done
