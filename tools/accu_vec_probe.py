"""accu / min / max over a 2^30 f32 Col, back-to-back device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
n = 1 << 30
dm.set_seed(2)
a = dm.Col(n, fill="randu")
for name in ("accu", "min", "max"):
    r = D.ShardedReduction(name, a)
    for _ in range(3): r.launch()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3): r.launch()
        e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 3)
    print(f"{name} 2^30: {best:.3f} ms  {4 * n / best / 1e6:.0f} GB/s", flush=True)
