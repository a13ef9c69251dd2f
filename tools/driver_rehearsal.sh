# What the driver runs at round end (1 GPU): pytest -m gpu, smoke(), the reference arm, the default bench
mkdir -p gpurun_out/rehearsal
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/rehearsal/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/rehearsal/pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/rehearsal/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/rehearsal/smoke.log
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/rehearsal/ref.log 2>&1
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/rehearsal/bench.log 2>&1
