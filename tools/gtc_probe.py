"""One Gaussian Sum at M = N = n on the selected path (GENRED_GAUSS_TC), with SM clocks sampled."""
import os, sys, json, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
from paper_2004_11127_b200 import genred as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = torch.from_numpy(synth.uniform3(n, 1005)).cuda(); y = torch.from_numpy(synth.uniform3(n, 2005)).cuda()
b = torch.from_numpy(synth.signal(n, 3005)).cuda()
a = G.eval("gauss", "sum", x, y, b, scale=0.5); torch.cuda.synchronize()
clk = []
stop = False
def samp():
    try:
        import pynvml
        pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop:
            clk.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.05)
    except Exception as e:
        clk.append(str(e))
th = threading.Thread(target=samp); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    a = G.eval("gauss", "sum", x, y, b, scale=0.5)
e1.record(); torch.cuda.synchronize()
stop = True; th.join()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"n": n, "path": G.last_plan()["path"], "ms": ms, "pairs_per_s": n * n / (ms * 1e-3),
                  "clocks": clk[len(clk)//4: len(clk)//4 + 8]}), flush=True)
