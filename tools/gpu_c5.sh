python -c "
import torch, synth
from paper_2004_11127_b200 import genred
x = torch.from_numpy(synth.uniform3(10000, 1)).cuda(); y = torch.from_numpy(synth.uniform3(10000000, 2)).cuda()
genred.eval('sqdist', 'lse', x, y, None, scale=0.05, out_dtype='float64'); print('lse 1e4 x 1e7 plan', genred.last_plan())
lib = genred.load()
" > gpurun_out/r02/lse_plan.txt 2>&1
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r02/bench_c5.log 2>&1
timeout 1500 python bench.py --steps 3 --warmup 3 --dist GMM3 > gpurun_out/r02/bench_c5_gmm.log 2>&1
