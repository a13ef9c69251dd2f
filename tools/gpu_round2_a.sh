set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest1.log
timeout 300 python bench.py --mode jshard --config 7 --steps 3 --warmup 3 > gpurun_out/j7.log 2>&1; echo rc=$? >> gpurun_out/j7.log
timeout 300 python bench.py --mode jshard --config 8 --steps 3 --warmup 3 > gpurun_out/j8.log 2>&1; echo rc=$? >> gpurun_out/j8.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 2 --dist-backend gloo --one-device --steps 3 --warmup 3 > gpurun_out/ish2.log 2>&1; echo rc=$? >> gpurun_out/ish2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --mode jshard --config 8 --dist-backend gloo --one-device --steps 3 --warmup 3 > gpurun_out/jsh2.log 2>&1; echo rc=$? >> gpurun_out/jsh2.log
