"""Where the host time of one fused logistic step goes (cProfile, tottime)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
nrow, ncol = 1 << 16, 1024
X = dm.Matrix(nrow, ncol, fill="randn")
w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
def step():
    r, g = dm.evaluate_many(r_e, X.t() @ r_e)
    return dm.accu(r)
for _ in range(20): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): step()
print(f"host per step (small X, GPU not the bound): {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile(); pr.enable()
for _ in range(200): step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
