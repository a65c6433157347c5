"""Epilogues that read another m x n matrix (exp(AB^T/n) - C, 2 AB^T + 3 C) fused
into the GEMM's store against the reference's plan, interleaved in one process
so the power / thermal state is shared (GPU box).  Run with BM_GEMM_PERSIST=0|1.
Usage: python tools/epi_mem_probe.py [n] [rounds] [f32|f64]"""
import json
import os
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2308_03120_b200 as dm  # noqa: E402
from paper_2308_03120_b200 import dist as D  # noqa: E402
from paper_2308_03120_b200 import expr as E  # noqa: E402


def once(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    elem = sys.argv[3] if len(sys.argv) > 3 else "f32"
    dm.init("b200")
    D.bind_torch_stream()
    dm.set_seed(3)
    A, B, C = (dm.Matrix(n, n, fill="randu", elem_type=elem) for _ in range(3))
    e1 = dm.exp((A @ B.t()) / n) - C
    e2 = 2 * (A @ B.t()) + 3 * C
    E._EPI_MEM_INPUTS = True
    variants = {"plain": lambda: dm.evaluate(A @ B.t()),
                "exp-C fused": lambda: dm.evaluate(e1), "exp-C unfused": lambda: dm.evaluate(e1, fuse=False),
                "axpby fused": lambda: dm.evaluate(e2), "axpby unfused": lambda: dm.evaluate(e2, fuse=False)}
    plans = {"exp-C": [s.kernel for s in dm.plan(e1).steps], "axpby": [s.kernel for s in dm.plan(e2).steps]}
    ts = {k: [] for k in variants}
    for fn in variants.values():
        fn()
    torch.cuda.synchronize()
    for _ in range(rounds):
        for k, fn in variants.items():
            ts[k].append(once(fn))
    out = {"n": n, "elem": elem, "persist": os.environ.get("BM_GEMM_PERSIST", "0"), "plans": plans}
    out.update({k: round(statistics.median(v), 3) for k, v in ts.items()})
    print(json.dumps(out))
    dm.shutdown()


if __name__ == "__main__":
    main()
