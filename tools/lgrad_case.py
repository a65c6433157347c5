import sys, numpy as np, pathlib
sys.path.insert(0, "/root/repo")
import paper_2308_03120_b200 as dm
m, k = int(sys.argv[1]), int(sys.argv[2])
dm.init("b200")
rng = np.random.default_rng(1)
X = rng.standard_normal((m, k), dtype=np.float32); w = (0.03*rng.standard_normal((k,1))).astype(np.float32); y = (rng.random((m,1))<0.5).astype(np.float32)
mX, mw, my = dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(w), dm.Matrix.from_numpy(y)
r_e = 1/(1+dm.exp(0 - mX @ mw)) - my
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
for _ in range(reps):
    r, g = dm.evaluate_many(r_e, mX.t() @ r_e)
    dm.synchronise()
gf = X.T.astype(np.float64) @ (1/(1+np.exp(-(X.astype(np.float64)@w))) - y)
print(m, k, "ok", np.abs(g.to_numpy()-gf).max()/np.abs(gf).max(), flush=True)
