import sys, pathlib
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
for n in (4096, 8192, 16384):
    A, B, C, Dm = (dm.Matrix(n, n, fill="randu") for _ in range(4))
    for name, r, nb in (("cfg1", D.ShardedReduction("accu", 2 * A + B % C - dm.exp(Dm)), 16), ("dot", D.ShardedReduction("dot", A, B), 8), ("accu1", D.ShardedReduction("accu", A), 4)):
        for _ in range(5): r.launch()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20): r.launch()
            e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 20)
        print(f"n={n} {name}: {best*1e3:.1f} us  {nb*n*n/best/1e6:.0f} GB/s", flush=True)
    del A, B, C, Dm
