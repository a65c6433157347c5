"""GEMM prologue / epilogue fusion vs the reference's plan (GPU box): median
CUDA-event time of 10 evaluations at 8192^3 for f32 (3xTF32) and f64 (DMMA).
Prints one JSON line.  Usage: python tools/fusion_probe.py [n]"""
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
    return round(statistics.median(ts), 3)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dm.init("b200")
    D.bind_torch_stream()
    out = {"n": n}
    for elem in sys.argv[2].split(",") if len(sys.argv) > 2 else ("f32", "f64"):
        dm.set_seed(3)
        A = dm.Matrix(n, n, fill="randu", elem_type=elem)
        B = dm.Matrix(n, n, fill="randu", elem_type=elem)
        C = dm.Matrix(n, n, fill="randu", elem_type=elem)
        r = {"plain A@B.t()": med(lambda: dm.evaluate(A @ B.t()))}
        pro = (2 * A + 1) @ (B - 3).t()
        r["prologue fused"] = med(lambda: dm.evaluate(pro))
        r["prologue unfused"] = med(lambda: dm.evaluate(pro, fuse=False))
        epi = dm.exp((A @ B.t()) / n) - C
        r["epilogue fused"] = med(lambda: dm.evaluate(epi))
        r["epilogue unfused"] = med(lambda: dm.evaluate(epi, fuse=False))
        triv = (A @ B.t()) * 1
        r["epilogue trivial fused"] = med(lambda: dm.evaluate(triv))
        sub = (A @ B.t()) - C
        r["epilogue minus C fused"] = med(lambda: dm.evaluate(sub))
        ex = dm.exp((A @ B.t()) / n)
        r["epilogue exp fused"] = med(lambda: dm.evaluate(ex))
        r["epilogue exp unfused"] = med(lambda: dm.evaluate(ex, fuse=False))
        r["plans"] = {"prologue": [s.kernel for s in dm.plan(pro).steps],
                      "epilogue": [s.kernel for s in dm.plan(epi).steps]}
        out[elem] = r
        del A, B, C
    print(json.dumps(out))
    dm.shutdown()


if __name__ == "__main__":
    main()
