"""Single isolated launch of the config-1 reduction (GPU box): L2 flushed and
the device idle before every launch, CUDA events around the one launch,
median of 30.  Knobs come from the environment (BM_DEBUG_NOFOLD,
BM_REDUCE_WARPS, ...), so the fold / ramp / tail costs can be told apart.
Prints one JSON line."""
import json
import os
import pathlib
import statistics
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    dm.init("b200")
    D.bind_torch_stream()
    rng = np.random.default_rng(0)
    A, B, C, Dm = (dm.Matrix.from_numpy(rng.random((4096, 4096), dtype=np.float32)) for _ in range(4))
    cases = {"cfg1": (D.ShardedReduction("accu", 2 * A + B % C - dm.exp(Dm)), 4 << 26),
             "accu_1in": (D.ShardedReduction("accu", A), 1 << 26),
             "dot_2in": (D.ShardedReduction("dot", A, B), 2 << 26)}
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    out = {k: os.environ.get(k) for k in ("BM_DEBUG_NOFOLD", "BM_REDUCE_WARPS", "BM_REDUCE_GRAB")}
    for name, (r, nb) in cases.items():
        for _ in range(5):
            r.launch()
        torch.cuda.synchronize()
        iso = []
        for _ in range(30):
            flush.sum()                 # read-only flush: L2 left holding clean lines
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)   # ~100 us of device work: the launch below is queued behind it
            s.record()
            r.launch()
            e.record()
            e.synchronize()
            iso.append(s.elapsed_time(e))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            r.launch()
        e.record()
        e.synchronize()
        pipe = s.elapsed_time(e) / 50
        out[name] = {"isolated_us": round(statistics.median(iso) * 1e3, 2), "min_us": round(min(iso) * 1e3, 2),
                     "pipelined_us": round(pipe * 1e3, 2), "isolated_GBs": round(nb / statistics.median(iso) / 1e6, 1),
                     "value": float(r.value())}
    print(json.dumps(out))
    dm.shutdown()


if __name__ == "__main__":
    main()
