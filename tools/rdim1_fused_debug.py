import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2308_03120_b200 as dm
dm.init("b200")
rng = np.random.default_rng(0)
a = rng.standard_normal((8192, 40)).astype(np.float32); b = rng.standard_normal((8192, 40)).astype(np.float32)
A, B = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
case = sys.argv[1]
if case == "one":
    got = dm.evaluate(dm.sum(2 * A + 1, 1)).to_numpy(); ref = (2 * a + 1).sum(axis=1, dtype=np.float32)
elif case == "two":
    got = dm.evaluate(dm.sum(A + B, 1)).to_numpy(); ref = (a + b).sum(axis=1)
else:
    got = dm.evaluate(dm.sum(A + B + A * B + B, 1)).to_numpy(); ref = None
print(case, "ok", None if ref is None else float(np.abs(got.ravel() - ref).max()))
