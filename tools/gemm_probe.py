"""Time the NT GEMM (C = A * B^T) at several sizes on the GPU box."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main(sizes, elems):
    import torch
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import runtime as R
    from paper_2308_03120_b200 import dist as D
    dm.init("b200")
    D.bind_torch_stream()
    rt = R.get_runtime()
    for elem in elems:
        for n in sizes:
            A = dm.Matrix(n, n, fill="randu", elem_type=elem)
            B = dm.Matrix(n, n, fill="randu", elem_type=elem)
            C = dm.Matrix(n, n, elem_type=elem)
            inv = dm.KernelInvocation("gemm", (R.BlockView(A.mem, 0, n, n, n), R.BlockView(B.mem, 0, n, n, n)),
                                      R.BlockView(C.mem, 0, n, n, n), (), {"trans_a": 0, "trans_b": 1})
            rt.enqueue(inv)
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3 if n <= 16384 else 1):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                rt.enqueue(inv)
                e.record()
                e.synchronize()
                best = min(best, s.elapsed_time(e))
            print(f"{elem} {n}^3: {best:.3f} ms  {2 * n ** 3 / best / 1e9:.1f} TFLOP/s", flush=True)
            del A, B, C
    dm.shutdown()


if __name__ == "__main__":
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,16384,32768").split(",")]
    elems = (sys.argv[2] if len(sys.argv) > 2 else "f32").split(",")
    main(sizes, elems)
