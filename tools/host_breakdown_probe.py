"""Host-side cost breakdown of the config-5 fused step (GPU box): wraps the
runtime / planner entry points with perf_counter accumulators and reports
microseconds per step for each.  Usage: python tools/host_breakdown_probe.py"""
import collections
import functools
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2308_03120_b200 as dm  # noqa: E402
from paper_2308_03120_b200 import dist as D  # noqa: E402
from paper_2308_03120_b200 import expr as E  # noqa: E402
from paper_2308_03120_b200 import runtime as R  # noqa: E402

ACC = collections.defaultdict(float)
MARK = {"t0": None, "first": []}


def wrap(obj, name, label):
    f = getattr(obj, name)

    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            ACC[label] += time.perf_counter() - t
    setattr(obj, name, g)


class LibProxy:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, n):
        f = getattr(self._lib, n)
        if not callable(f):
            return f

        def g(*a):
            t = time.perf_counter()
            if n == "bm_enqueue" and MARK["t0"] is not None:
                MARK["first"].append(t - MARK["t0"])
                MARK["t0"] = None
            try:
                return f(*a)
            finally:
                ACC["C " + n] += time.perf_counter() - t
        return g


def main():
    dm.init("b200")
    D.bind_torch_stream()
    nrow, ncol = 1 << 20, 1024
    dm.set_seed(5)
    X = dm.Matrix(nrow, ncol, fill="randn")
    w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
    y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
    r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
    rt = R.get_runtime()

    def step():
        MARK["t0"] = time.perf_counter()
        r, g = dm.evaluate_many(r_e, X.t() @ r_e)
        return dm.accu(r)

    for _ in range(5):
        step()
    wrap(E, "evaluate_many", "evaluate_many")
    wrap(E, "execute_plan", "execute_plan")
    wrap(E, "plan_reduce", "plan_reduce")
    wrap(E._Lowerer, "lower", "Lowerer.lower (recursive, inclusive)")
    wrap(R, "build_invocation", "build_invocation")
    wrap(rt, "acquire_memory", "acquire_memory")
    wrap(rt, "_validate", "_validate")
    wrap(rt, "release_deferred", "release_deferred")
    wrap(rt, "enqueue", "enqueue (incl. C)")
    rt._lib = LibProxy(rt._lib)
    dm.evaluate_many = E.evaluate_many
    n = 50
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    wall = (time.perf_counter() - t0) / n
    for k, v in sorted(ACC.items(), key=lambda kv: -kv[1]):
        print(f"{k:40s} {v / n * 1e6:9.1f} us/step")
    print(f"{'wall':40s} {wall * 1e6:9.1f} us/step")
    import statistics
    print(f"{'step start -> bm_enqueue (median)':40s} {statistics.median(MARK['first']) * 1e6:9.1f} us")
    dm.shutdown()


if __name__ == "__main__":
    main()
