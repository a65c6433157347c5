"""Where the config-5 fused step's time goes on the host (GPU box):
cProfile of evaluate_many + accu over a few steps, and CUDA-event time of the
step vs its kernels."""
import cProfile
import pathlib
import pstats
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

    def step():
        r, g = dm.evaluate_many(r_e, X.t() @ r_e)
        return dm.accu(r)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        step()
    torch.cuda.synchronize()
    print("step wall ms", (time.perf_counter() - t0) / 50 * 1e3)
    # host-only cost of planning (no launch): plan() of the same tree
    t0 = time.perf_counter()
    for _ in range(50):
        dm.plan(X.t() @ r_e)
    print("plan() ms", (time.perf_counter() - t0) / 50 * 1e3)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        step()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
    dm.shutdown()


if __name__ == "__main__":
    main()
