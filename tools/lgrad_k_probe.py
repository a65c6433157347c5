"""Fused logistic step vs the two-pass plan at other widths (GPU box): X of
2^30 / k rows x k f32 columns (4 GiB), median of 10 CUDA-event timings.
Prints one JSON line.  Usage: python tools/lgrad_k_probe.py [k ...]"""
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2308_03120_b200 as dm  # noqa: E402
from paper_2308_03120_b200 import dist as D  # noqa: E402


def med(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    dm.init("b200")
    D.bind_torch_stream()
    out = {}
    for k in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
        m = (1 << 30) // k
        dm.set_seed(5)
        X = dm.Matrix(m, k, fill="randn")
        w = dm.evaluate(0.03 * dm.Matrix(k, 1, fill="randn"))
        y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(m, 1, fill="randu"), "i32"), "f32"))
        r_e = 1 / (1 + dm.exp(0 - X @ w)) - y

        def fused():
            r, g = dm.evaluate_many(r_e, X.t() @ r_e)
            return dm.accu(r)

        def two_pass():
            z = dm.evaluate(X @ w)
            r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - y)
            dm.evaluate(X.t() @ r)
            return dm.accu(r)

        tf, tt = med(fused), med(two_pass)
        nb = 4 * m * k
        out[k] = {"rows": m, "fused_ms": round(tf, 4), "two_pass_ms": round(tt, 4),
                  "fused_GBs": round(nb / tf / 1e6, 1), "plan": [s.kernel for s in dm.plan(X.t() @ r_e).steps]}
        del X, w, y, r_e
    print(json.dumps(out))
    dm.shutdown()


if __name__ == "__main__":
    main()
