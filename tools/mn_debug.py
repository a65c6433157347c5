"""Debug the MN-major GEMM path (BM_GEMM_MN=1): structured inputs, print what comes out."""
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2308_03120_b200 as dm  # noqa: E402

dm.init("b200")
m = n = 256
k = 32
rng = np.random.default_rng(0)
a = rng.integers(0, 4, (m, k)).astype(np.float32)
b = rng.integers(0, 4, (n, k)).astype(np.float32)
ma, mb = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
got = dm.evaluate(ma @ mb.t()).to_numpy()
ref = a @ b.T
print("max|got|", np.abs(got).max(), "max|ref|", np.abs(ref).max(), "nonzero frac", (got != 0).mean())
print("got[:4,:4]\n", got[:4, :4], "\nref[:4,:4]\n", ref[:4, :4])
# unit probes: A = e_i e_k^T-ish, B = ones -> C[i, :] = count
for (i, kk) in [(0, 0), (1, 0), (0, 1), (33, 0), (0, 9), (0, 17), (130, 3)]:
    a1 = np.zeros((m, k), np.float32)
    a1[i, kk] = 1
    b1 = np.zeros((n, k), np.float32)
    b1[:, kk] = np.arange(n, dtype=np.float32) + 1
    c1 = dm.evaluate(dm.Matrix.from_numpy(a1) @ dm.Matrix.from_numpy(b1).t()).to_numpy()
    nz = np.argwhere(c1 != 0)
    print(f"A[{i},{kk}]=1, B[:,{kk}]=1..n: nonzeros {len(nz)}; rows {sorted(set(nz[:, 0].tolist()))[:8]}; "
          f"C[row, 0:4] {c1[nz[0][0], :4] if len(nz) else None}")
dm.shutdown()
