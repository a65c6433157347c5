"""Config-1 expression at larger sizes: single launch, back to back, and the
SM clock / power while it runs (debugging the large-n reduction rate)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A, B, C, Dm = (dm.Matrix(n, n, fill="randu") for _ in range(4))
r = D.ShardedReduction("accu", 2 * A + B % C - dm.exp(Dm))
for _ in range(3): r.launch()
torch.cuda.synchronize()
one = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); r.launch(); e.record(); e.synchronize(); one.append(s.elapsed_time(e))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): r.launch()
e.record()
time.sleep(0.005)
clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
reasons = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
e.synchronize()
bt = s.elapsed_time(e) / 50
print(f"n={n}: single {min(one)*1e3:.1f} us ({16*n*n/min(one)/1e6:.0f} GB/s), back-to-back {bt*1e3:.1f} us "
      f"({16*n*n/bt/1e6:.0f} GB/s), sm {clk} MHz, {pw:.0f} W, reasons {reasons:#x}")
