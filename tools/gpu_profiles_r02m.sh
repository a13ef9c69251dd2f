# Round-2 last pass (after the edge tiles, the split-major planner and the host gather): the driver's sequence (tests, smoke, reference
# arm, default bench) and the config lines.
mkdir -p gpurun_out/r02m
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r02m/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02m/pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02m/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02m/smoke.log
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02m/ref.log 2>&1
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02m/bench.log 2>&1
for c in 1 2 3 4 9; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r02m/bench_c$c.log 2>&1; done
timeout 900 python bench.py --config 5 --dist GMM3 --steps 3 --warmup 3 > gpurun_out/r02m/bench_c5_gmm.log 2>&1
timeout 900 python bench.py --config 5 --shape 2000000,2000000 --scale 0.05 --steps 5 --warmup 3 > gpurun_out/r02m/bench_direct.log 2>&1
timeout 900 python bench.py --mode jshard --config 7 --steps 5 --warmup 3 > gpurun_out/r02m/bench_j7.log 2>&1
timeout 900 python bench.py --mode jshard --config 8 --steps 5 --warmup 3 > gpurun_out/r02m/bench_j8.log 2>&1
for n in 1 8 32; do timeout 600 python bench.py --config 6 --edge-n $n --steps 10 --warmup 3 > gpurun_out/r02m/bench_edge$n.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-e2e --shape 2000000,2000000 > gpurun_out/r02m/launches_c5.log 2>&1
timeout 1200 python tools/bench_next.py > gpurun_out/r02m/bench_next.jsonl 2> gpurun_out/r02m/bench_next.err
timeout 900 python tools/bench_paper_table.py > gpurun_out/r02m/paper_table.jsonl 2> gpurun_out/r02m/paper_table.err
