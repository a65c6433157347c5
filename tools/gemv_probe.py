"""X @ w and X.t() @ r on 2^20 x 1024 f32 (config 5's two GEMVs), device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
nrow, ncol = 1 << 20, 1024
X = dm.Matrix(nrow, ncol, fill="randn")
w = dm.Matrix(ncol, 1, fill="randn")
r = dm.Matrix(nrow, 1, fill="randn")
for name, fn in (("X @ w", lambda: dm.evaluate(X @ w)), ("X.t() @ r", lambda: dm.evaluate(X.t() @ r))):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5): fn()
        e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 5)
    print(f"{name}: {best:.3f} ms  {4 * nrow * ncol / best / 1e6:.0f} GB/s", flush=True)
