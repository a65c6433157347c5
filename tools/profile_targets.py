"""Run one hot-path workload a few times so ncu can capture its kernel.
Usage: python tools/profile_targets.py cfg1|accu1|logistic|logistic_fused|gemm_f32|gemm_f64|rdim0|rdim1|rdim0_fused|rdim1_fused|dot"""
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main(which: str) -> None:
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import runtime as R
    dm.init("b200")
    rt = R.get_runtime()
    if which == "cfg1":
        rng = np.random.default_rng(0)
        A, B, C, D = (dm.Matrix.from_numpy(rng.random((4096, 4096), dtype=np.float32)) for _ in range(4))
        for _ in range(4):
            dm.accu(2 * A + B % C - dm.exp(D))
    elif which == "accu1":
        rng = np.random.default_rng(0)
        A = dm.Matrix.from_numpy(rng.random((4096, 4096), dtype=np.float32))
        for _ in range(4):
            dm.accu(A)
    elif which == "logistic":
        nrow, ncol = 1 << 20, 1024
        X = dm.Matrix(nrow, ncol, fill="randn")
        w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
        y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
        for _ in range(3):
            z = dm.evaluate(X @ w)
            r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - y)
            g = dm.evaluate(X.t() @ r)
            dm.accu(r)
    elif which == "logistic_fused":
        nrow, ncol = 1 << 20, 1024
        X = dm.Matrix(nrow, ncol, fill="randn")
        w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
        y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
        r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
        for _ in range(3):
            r, g = dm.evaluate_many(r_e, X.t() @ r_e)
    elif which in ("gemm_f32", "gemm_f64", "gemm32k_f32", "gemm32k_f64"):
        elem = which[-3:]
        n = 32768 if "32k" in which else 8192
        A = dm.Matrix(n, n, fill="randu", elem_type=elem)
        B = dm.Matrix(n, n, fill="randu", elem_type=elem)
        for _ in range(3):
            dm.evaluate(A @ B.t())
    elif which == "epi_axpby":
        n = 8192
        A, B, C = (dm.Matrix(n, n, fill="randu") for _ in range(3))
        e = 2 * (A @ B.t()) + 3 * C
        for _ in range(3):
            dm.evaluate(e)
    elif which in ("epi_exp", "epi_exp_minus_c"):
        # the fused-epilogue pair GEMM at 8192^3: exp(AB^T/n), and exp(AB^T/n) - C with C
        # read in the store (BM_GEMM_EPI_INPUTS forced on)
        from paper_2308_03120_b200 import expr as E
        E._EPI_MEM_INPUTS = True
        n = 8192
        A, B, C = (dm.Matrix(n, n, fill="randu") for _ in range(3))
        e = dm.exp((A @ B.t()) / n) - C if which == "epi_exp_minus_c" else dm.exp((A @ B.t()) / n)
        for _ in range(3):
            dm.evaluate(e)
    elif which in ("rdim0", "rdim1"):
        m = dm.Matrix(16384, 16384, fill="randu", elem_type="f64")
        for op in ("sum", "max"):
            for _ in range(2):
                dm.evaluate(getattr(dm, op)(m, int(which[-1])))
    elif which in ("rdim0_fused", "rdim1_fused"):
        a = dm.Matrix(16384, 16384, fill="randu", elem_type="f64")
        b = dm.Matrix(16384, 16384, fill="randu", elem_type="f64")
        for _ in range(2):
            dm.evaluate(dm.sum(2 * a + b, int(which[4])))
    elif which == "dot":
        a = dm.Col(1 << 30, fill="randu")
        b = dm.Col(1 << 30, fill="randu")
        for _ in range(3):
            dm.dot(a, b)
    dm.synchronise()
    dm.shutdown()


if __name__ == "__main__":
    main(sys.argv[1])
