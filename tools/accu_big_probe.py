"""Single-launch vs back-to-back timing of a large unit-mode accu (debugging
the large-n reduction rate)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import dist as D
dm.init("b200"); D.bind_torch_stream()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = dm.Matrix(n, n, fill="randu")
extra = [dm.Matrix(n, n, fill="randu") for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0)]
r = D.ShardedReduction("accu", A)
for _ in range(3): r.launch()
torch.cuda.synchronize()
one = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); r.launch(); e.record(); e.synchronize(); one.append(s.elapsed_time(e))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): r.launch()
e.record(); e.synchronize()
print(f"n={n}: single {min(one)*1e3:.1f} us, back-to-back {s.elapsed_time(e)/20*1e3:.1f} us, value {r.value()}")
