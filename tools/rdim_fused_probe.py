"""Time sum/mean/min/max(2*A + B, dim) on 16384^2 f64: fused (one kernel over A
and B) against the reference's plan (materialise 2*A + B, then reduce)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    dm.init("b200")
    D.bind_torch_stream()
    n = 16384
    A = dm.Matrix(n, n, fill="randu", elem_type="f64")
    B = dm.Matrix(n, n, fill="randu", elem_type="f64")

    def timeit(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        return best

    for dim in (0, 1):
        for op in ("sum", "mean", "min", "max"):
            f = getattr(dm, op)
            fused = timeit(lambda: dm.evaluate(f(2 * A + B, dim)))
            unfused = timeit(lambda: dm.evaluate(f(dm.evaluate(2 * A + B), dim)))
            print(f"{op}(2*A + B, {dim}): fused {fused:.3f} ms ({16 * n * n / fused / 1e6:.0f} GB/s of inputs), "
                  f"materialise + reduce {unfused:.3f} ms", flush=True)
    dm.shutdown()


if __name__ == "__main__":
    main()
