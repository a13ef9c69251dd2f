#!/bin/bash
# Round-end refresh of every bench line and side measurement into gpurun_out/ (no ncu here).
set -x
python bench.py > gpurun_out/r01_bench_c5.json 2> gpurun_out/r01_bench_c5.err
python bench.py --config 2 > gpurun_out/r01_bench_c2.json 2> gpurun_out/r01_bench_c2.err
python bench.py --config 3 > gpurun_out/r01_bench_c3.json 2> gpurun_out/r01_bench_c3.err
python bench.py --config 4 > gpurun_out/r01_bench_c4.json 2> gpurun_out/r01_bench_c4.err
python bench.py --config 1 --steps 20 --warmup 5 > gpurun_out/r01_bench_c1.json 2> gpurun_out/r01_bench_c1.err
python bench.py --config 6 --edge-n 1 > gpurun_out/r01_bench_edge1.json 2> gpurun_out/r01_bench_edge1.err
python bench.py --config 6 --edge-n 8 > gpurun_out/r01_bench_edge8.json 2> gpurun_out/r01_bench_edge8.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01_bench_reference.json 2> gpurun_out/r01_bench_reference.err
python tools/bench_next.py > gpurun_out/r01_bench_next.jsonl 2> gpurun_out/r01_bench_next.err
python tools/bench_paper_table.py > gpurun_out/r01_paper_table.jsonl 2> gpurun_out/r01_paper_table.err
python tools/small_m_probe.py > gpurun_out/r01_small_m.jsonl 2> gpurun_out/r01_small_m.err
python tools/argk_small_m_probe.py > gpurun_out/r01_argk_small_m.jsonl 2> gpurun_out/r01_argk_small_m.err
