# Round-2 final measurement pass: the driver's sequence (tests, smoke, reference arm, default bench)
# plus ncu of the final Gaussian kernel and the config lines.
mkdir -p gpurun_out/r02d
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02d/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02d/pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02d/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02d/smoke.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02d/ref.log 2>&1
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02d/bench.log 2>&1
for c in 1 2 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02d/bench_c$c.log 2>&1; done
timeout 900 python bench.py --config 5 --dist GMM3 --steps 3 --warmup 3 > gpurun_out/r02d/bench_c5_gmm.log 2>&1
timeout 900 python bench.py --mode jshard --config 7 --steps 5 --warmup 3 > gpurun_out/r02d/bench_j7.log 2>&1
python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02d/plain_gauss.log 2>&1 && \
ncu --set full --clock-control none -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02d/ncu_gauss python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02d/ncu_gauss.log 2>&1
python tools/ncu_summary.py gpurun_out/r02d/ncu_gauss.ncu-rep gpurun_out/r02d/r02_ncu_gauss.md > /dev/null 2>&1
ncu -i gpurun_out/r02d/ncu_gauss.ncu-rep --page raw --csv > gpurun_out/r02d/r02_ncu_gauss_raw.csv 2>/dev/null; rm -f gpurun_out/r02d/ncu_gauss.ncu-rep
timeout 1200 python tools/bench_next.py > gpurun_out/r02d/bench_next.jsonl 2> gpurun_out/r02d/bench_next.err
timeout 900 python tools/bench_paper_table.py > gpurun_out/r02d/paper_table.jsonl 2> gpurun_out/r02d/paper_table.err
