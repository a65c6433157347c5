import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2308_03120_b200 as dm
import oracle as O
dm.init("b200")
for shape in ((4, 3), (16, 5), (8, 1000), (128, 2), (64, 1)):
    rng = np.random.default_rng(1)
    a = rng.random(shape, dtype=np.float32); b = rng.random(shape, dtype=np.float32)
    A, B = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    ks = [s.kernel for s in dm.plan(dm.sum(2 * A + B, 1)).steps]
    try:
        got = dm.evaluate(dm.sum(2 * A + B, 1)).to_numpy()
        mat = dm.evaluate(2 * A + B).to_numpy()
        ok = np.array_equal(got, O.rdim("sum", mat, 1))
        print(shape, ks, "ok" if ok else "MISMATCH")
    except Exception as e:
        print(shape, ks, "ERROR", repr(e)[:150])
