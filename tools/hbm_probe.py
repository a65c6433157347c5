"""Calibrate this box: torch copy bandwidth (like MEASURED_PEAKS.json) and a
torch sum over 256 MiB, timed with CUDA events."""
import json
import torch


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / reps)
    return best


a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
ms = t(lambda: b.copy_(a), 5)
x = torch.rand(4 * 4096 * 4096, device="cuda")
ms2 = t(lambda: x.sum())
y = torch.rand(4096 * 4096 * 8, device="cuda")
ms3 = t(lambda: torch.dot(y[: len(y) // 2], y[len(y) // 2:]))
print(json.dumps({"copy_GBs": 2 * a.numel() * 2 / ms / 1e6, "sum256MiB_us": ms2 * 1e3,
                  "sum256MiB_GBs": x.numel() * 4 / ms2 / 1e6, "dot2x256MiB_GBs": y.numel() * 4 / ms3 / 1e6}))
