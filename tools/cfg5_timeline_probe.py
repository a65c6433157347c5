"""Config-5 fused step on the GPU box: host time of each API call and the
device timeline around them (CUDA events on the library's stream), medians
over 50 steps.  Tells host latency before the kernel apart from device work.
Usage: python tools/cfg5_timeline_probe.py"""
import pathlib
import statistics
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2308_03120_b200 as dm  # noqa: E402
from paper_2308_03120_b200 import dist as D  # noqa: E402


def main():
    dm.init("b200")
    D.bind_torch_stream()
    nrow, ncol = 1 << 20, 1024
    dm.set_seed(5)
    X = dm.Matrix(nrow, ncol, fill="randn")
    w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
    y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
    r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
    rows = []
    for it in range(60):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e[0].record()
        r, g = dm.evaluate_many(r_e, X.t() @ r_e)
        t1 = time.perf_counter()
        e[1].record()
        s = dm.accu(r)
        t2 = time.perf_counter()
        e[2].record()
        torch.cuda.synchronize()
        if it >= 10:
            rows.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t2 - t0) * 1e3, e[0].elapsed_time(e[1]),
                         e[1].elapsed_time(e[2])))
    names = ("host evaluate_many", "host accu (incl. sync)", "host step", "dev e0->e1 (lgrad+finish)",
             "dev e1->e2 (accu)")
    for i, nm in enumerate(names):
        print(f"{nm:32s} {statistics.median(r[i] for r in rows):8.4f} ms")
    print("accu value", s)
    dm.shutdown()


if __name__ == "__main__":
    main()
