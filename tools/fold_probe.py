"""Fixed-cost probe for the flat reduction (GPU box): accu of a 1-input f32
vector at several sizes, timed with CUDA events.  Run once normally and once
with BM_DEBUG_NOFOLD=1 to isolate the final fold."""
import json
import os
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    dm.init("b200")
    D.bind_torch_stream()
    out = {"nofold": os.environ.get("BM_DEBUG_NOFOLD")}
    for lg in (13, 17, 20, 22, 24, 26):
        n = 1 << lg
        a = dm.Col.from_numpy(np.random.default_rng(0).random(n, dtype=np.float32))
        r = D.ShardedReduction("accu", a)
        for _ in range(5):
            r.launch()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(50):
                r.launch()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e) / 50)
        out[f"2^{lg}_us"] = round(best * 1e3, 2)
    print(json.dumps(out))
    dm.shutdown()


if __name__ == "__main__":
    main()
