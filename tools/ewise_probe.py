"""Element-wise store bandwidth: evaluate(2*A + B % C - exp(D)) (config 1's
tree materialised: 4 inputs read, 1 output written) and a 1-input scale."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
from paper_2308_03120_b200 import expr as E
from paper_2308_03120_b200 import runtime as R
dm.init("b200"); D.bind_torch_stream()
rt = R.get_runtime()
for n in (4096, 8192, 16384):
    A, B, C, Dm = (dm.Matrix(n, n, fill="randu") for _ in range(4))
    out = dm.Matrix(n, n)
    for name, node, nin in (("cfg1_tree", 2 * A + B % C - dm.exp(Dm), 4), ("scale", 2 * A, 1)):
        p = E.plan(node)
        st = p.steps[0]
        views = E._step_views(p, st, {})
        inv = dm.KernelInvocation(st.kernel, tuple(views), E._make_view(out.mem, n, n, "flat"), st.scalars, st.params)
        rt.enqueue(inv); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(10): rt.enqueue(inv)
            e.record(); e.synchronize(); best = min(best, s.elapsed_time(e) / 10)
        print(f"n={n} {name}: {best*1e3:.1f} us  {(nin + 1) * 4 * n * n / best / 1e6:.0f} GB/s", flush=True)
    del A, B, C, Dm, out
