"""cProfile of the config-5 fused step's host side (GPU box): 300 steps of
r, g = evaluate_many(r_e, X.t() @ r_e); accu(r), top functions by own time.
Usage: python tools/cfg5_cprofile.py"""
import cProfile
import pathlib
import pstats
import sys

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

    for _ in range(10):
        step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(300):
        step()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(45)
    dm.shutdown()


if __name__ == "__main__":
    main()
