import sys, time, pathlib
sys.path.insert(0, "/root/repo")
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
nrow, ncol = 1 << 20, 1024
X = dm.Matrix(nrow, ncol, fill="randn")
w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
def fused():
    return dm.evaluate_many(r_e, X.t() @ r_e)
fused(); torch.cuda.synchronize()
import cProfile, pstats
t0 = time.perf_counter()
for _ in range(20): fused()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host enqueue per call {1e3*(t1-t0)/20:.3f} ms, total per call {1e3*(t2-t0)/20:.3f} ms")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): fused()
e.record(); e.synchronize(); print(f"back-to-back device per call {s.elapsed_time(e)/20:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(20): fused()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
