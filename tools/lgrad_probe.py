"""Time the config-5 logistic step: two-pass (reference plan) vs fused."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    dm.init("b200")
    D.bind_torch_stream()
    nrow, ncol = 1 << 20, 1024
    X = dm.Matrix(nrow, ncol, fill="randn")
    w = dm.evaluate(0.03 * dm.Matrix(ncol, 1, fill="randn"))
    y = dm.evaluate(dm.conv_to(dm.conv_to(2 * dm.Matrix(nrow, 1, fill="randu"), "i32"), "f32"))
    r_e = 1 / (1 + dm.exp(0 - X @ w)) - y

    def fused():
        return dm.evaluate_many(r_e, X.t() @ r_e)

    def twopass():
        z = dm.evaluate(X @ w)
        r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - y)
        return r, dm.evaluate(X.t() @ r)

    for name, fn in (("two-pass", twopass), ("fused", fused)):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        print(f"{name}: {best:.3f} ms  ({4 * nrow * ncol / best / 1e6:.0f} GB/s per pass over X)")
    dm.shutdown()


if __name__ == "__main__":
    main()
