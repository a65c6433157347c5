"""Time the config-1 fused eOp+accu kernel (and a few single-input
reductions) under the reduction-geometry knobs given in the environment
(BM_REDUCE_WARPS / BM_REDUCE_MODE / BM_REDUCE_CTAS / BM_UNIT_UNROLL).
Prints one JSON line.  Used for tuning sweeps on the GPU box."""
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
    out = {k: os.environ.get(k) for k in ("BM_REDUCE_WARPS", "BM_REDUCE_MODE", "BM_REDUCE_CTAS", "BM_UNIT_UNROLL")}
    rng = np.random.default_rng(0)
    A, B, C, Dm = (dm.Matrix.from_numpy(rng.random((4096, 4096), dtype=np.float32)) for _ in range(4))
    cases = {"cfg1": D.ShardedReduction("accu", 2 * A + B % C - dm.exp(Dm)),
             "cfg1_noexp": D.ShardedReduction("accu", 2 * A + B % C - Dm),
             "accu_1in": D.ShardedReduction("accu", A),
             "dot_2in": D.ShardedReduction("dot", A, B)}
    bytes_ = {"cfg1": 4, "cfg1_noexp": 4, "accu_1in": 1, "dot_2in": 2}
    import time
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM))
    out["clk_before"] = clk()
    warm = float(os.environ.get("WARM_S", "0"))
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < warm:
        for _ in range(20):
            cases["cfg1"].launch()
        torch.cuda.synchronize()
    out["clk_after_warm"] = clk()
    for name, r in cases.items():
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
        import time
        t0 = time.perf_counter()
        for _ in range(50):
            r.launch()
        out[name + "_cpu_issue_us"] = round((time.perf_counter() - t0) / 50 * 1e6, 2)
        torch.cuda.synchronize()
        out[name + "_us"] = round(best * 1e3, 2)
        out[name + "_GBs"] = round(bytes_[name] * 4 * 4096 * 4096 / (best * 1e-3) / 1e9, 1)
    out["check"] = float(cases["cfg1"].value())
    print(json.dumps(out), flush=True)
    dm.shutdown()


if __name__ == "__main__":
    main()
