"""32768^3 NT f32 GEMM: time one configuration (env BM_GEMM_GROUP / BM_GEMM_KPASS
are read once per process, so the sweep runs one process per setting).
Usage: python tools/gemm32k_sweep.py [n] -> prints 'n group kpass ms TF/s'"""
import os
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2308_03120_b200 as dm  # noqa: E402
from paper_2308_03120_b200 import dist as D  # noqa: E402
from paper_2308_03120_b200 import runtime as R  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dm.init("b200")
    D.bind_torch_stream()
    dm.set_seed(3)
    A = dm.Matrix(n, n, fill="randu")
    B = dm.Matrix(n, n, fill="randu")
    C = dm.Matrix(n, n)
    inv = dm.KernelInvocation("gemm", (R.BlockView(A.mem, 0, n, n, n), R.BlockView(B.mem, 0, n, n, n)),
                              R.BlockView(C.mem, 0, n, n, n), (), {"trans_a": 0, "trans_b": 1})
    rt = R.get_runtime()
    rt.enqueue(inv)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rt.enqueue(inv)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    print(n, os.environ.get("BM_GEMM_GROUP", "def"), os.environ.get("BM_GEMM_KPASS", "def"),
          f"{ms:.2f}", f"{2 * n ** 3 / ms / 1e9:.1f}", flush=True)
    dm.shutdown()


if __name__ == "__main__":
    main()
