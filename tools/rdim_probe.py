"""Time sum/min/max along dims 0 and 1 of a 16384^2 f64 matrix (config 2)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    from paper_2308_03120_b200 import expr as E
    from paper_2308_03120_b200 import runtime as R
    dm.init("b200")
    D.bind_torch_stream()
    m = dm.Matrix(16384, 16384, fill="randu", elem_type="f64")
    rt = R.get_runtime()
    for op in ("sum", "min", "max"):
        for dim in (0, 1):
            p = E.plan(getattr(dm, op)(m, dim))
            step = p.steps[0]
            res = dm.Matrix(*(1, 16384) if dim == 0 else (16384, 1), elem_type="f64")
            inv = dm.KernelInvocation(step.kernel, tuple(E._step_views(p, step, {})),
                                      E._make_view(res.mem, res.n_rows, res.n_cols, "flat"), (), step.params)
            rt.enqueue(inv)
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(3):
                    rt.enqueue(inv)
                e.record()
                e.synchronize()
                best = min(best, s.elapsed_time(e) / 3)
            print(f"{op} dim{dim}: {best:.3f} ms  {8 * 16384 ** 2 / best / 1e6:.0f} GB/s")
    dm.shutdown()


if __name__ == "__main__":
    main()
