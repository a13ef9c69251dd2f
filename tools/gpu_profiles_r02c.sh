# Round-2 measurement pass (c): the fused Sum + grad kernel (C2, final build) under ncu --set full,
# the full -m gpu suite on the final build, and the C2 / C3 / C1 bench lines.
mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02c/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02c/pytest.log
python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/r02c/plain_fused.log 2>&1 && \
ncu --set full --clock-control none -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02c/ncu_fused python tools/profile_run.py --what fused --M 100000 --N 100000 --reps 2 > gpurun_out/r02c/ncu_fused.log 2>&1
python tools/ncu_summary.py gpurun_out/r02c/ncu_fused.ncu-rep gpurun_out/r02c/r02_ncu_fused.md > /dev/null 2>&1
ncu -i gpurun_out/r02c/ncu_fused.ncu-rep --page raw --csv > gpurun_out/r02c/r02_ncu_fused_raw.csv 2>/dev/null; rm -f gpurun_out/r02c/ncu_fused.ncu-rep
for c in 2 3 1; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02c/bench_c$c.log 2>&1; done
