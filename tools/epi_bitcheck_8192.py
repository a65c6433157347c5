"""Fused GEMM epilogues at 8192^3 (GPU box): fused vs unfused plan, bit for bit,
with both result matrices held while compared.  Usage: python tools/epi_bitcheck_8192.py"""
import sys, torch
sys.path.insert(0, '.')
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
n = 8192
A, B, C = (dm.Matrix(n, n, fill="randu") for _ in range(3))
for e in (2 * (A @ B.t()) + 3 * C, dm.exp((A @ B.t()) / n), dm.exp((A @ B.t()) / n) - C):
    f, u = dm.evaluate(e), dm.evaluate(e, fuse=False)
    tf, tu = D.torch_view(f), D.torch_view(u)
    print([s.kernel for s in dm.plan(e).steps], torch.equal(tf, tu), int((tf != tu).sum()))
dm.shutdown()
