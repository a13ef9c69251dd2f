# Round-2 measurement pass (b): C5 launch list, ncu of the Gaussian / LSE kernels at their final
# occupancy, the reference arm, and the side measurements (8(f) items, paper table, small M).
set -x
mkdir -p gpurun_out/r02b
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02b/plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02b/ncu_c5.log 2>&1
python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02b/plain_gauss.log 2>&1 && \
ncu --set full --clock-control none -k regex:sum_kernel -s 1 -c 1 -o gpurun_out/r02b/ncu_gauss python tools/profile_run.py --what gauss --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02b/ncu_gauss.log 2>&1
python tools/profile_run.py --what lse --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02b/plain_lse.log 2>&1 && \
ncu --set full --clock-control none -k regex:lse_kernel -s 1 -c 1 -o gpurun_out/r02b/ncu_lse python tools/profile_run.py --what lse --M 1000000 --N 1000000 --reps 2 > gpurun_out/r02b/ncu_lse.log 2>&1
for r in gauss lse; do python tools/ncu_summary.py gpurun_out/r02b/ncu_$r.ncu-rep gpurun_out/r02b/r02_ncu_$r.md > /dev/null 2>&1; ncu -i gpurun_out/r02b/ncu_$r.ncu-rep --page raw --csv > gpurun_out/r02b/r02_ncu_${r}_raw.csv 2>/dev/null; rm -f gpurun_out/r02b/ncu_$r.ncu-rep; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b/bench_reference.log 2>&1
timeout 1200 python tools/bench_next.py > gpurun_out/r02b/bench_next.jsonl 2> gpurun_out/r02b/bench_next.err
timeout 900 python tools/bench_paper_table.py > gpurun_out/r02b/paper_table.jsonl 2> gpurun_out/r02b/paper_table.err
timeout 900 python tools/small_m_probe.py > gpurun_out/r02b/small_m.jsonl 2> gpurun_out/r02b/small_m.err
du -sh gpurun_out/r02b
