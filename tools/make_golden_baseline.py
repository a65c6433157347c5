"""Golden values of the UNMODIFIED reference at the exact BASELINE shapes and
seeds, written to tests/golden/baseline.npz.

Run in the build container (where /root/reference exists; ~3 minutes on 8
cores, ~20 GB of host memory):

    python tools/make_golden_baseline.py

The inputs are NOT stored (gigabytes); they are regenerated from the seeds by
tests/test_gpu_baseline_shapes.py and bench.py (``baseline_inputs`` below is
the single definition both import).  Stored: the reference's results, or for
the 8192^3 GEMMs a fixed sample of entries plus f64 row sums of C.
"""
from __future__ import annotations

import os
import pathlib
import sys
import tempfile
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = pathlib.Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden" / "baseline.npz"
sys.path.insert(0, str(ROOT))

from tools.baseline_inputs import (cfg1_inputs, cfg2_input, cfg3_inputs, cfg4_inputs, cfg5_inputs,  # noqa: E402
                                   gemm_sample_index)


def main() -> None:
    os.environ["KERNEL_CACHE_DIR"] = tempfile.mkdtemp(prefix="devmat-cache-")
    sys.path.insert(0, str(REF))
    import devmat as dm  # noqa: E402

    dm.init("parallel", worker_count=os.cpu_count())
    M = dm.Matrix.from_numpy
    g = {}
    t0 = time.time()

    # config 1: accu(2*A + B*C - exp(D)) on 4096^2 f32, default_rng(0)
    A, B, C, D = (M(x) for x in cfg1_inputs())
    g["cfg1_accu_exp"] = np.float32(dm.accu(2 * A + B * C - dm.exp(D)))
    g["cfg1_accu_noexp"] = np.float32(dm.accu(2 * A + B * C - D))
    del A, B, C, D
    print("cfg1", g["cfg1_accu_exp"], time.time() - t0, flush=True)

    # config 2: f64 sum / min / max along both dims of 16384^2, default_rng(1)
    X = M(cfg2_input())
    for op in ("sum", "min", "max"):
        for dim in (0, 1):
            g[f"cfg2_{op}{dim}"] = dm.evaluate(getattr(dm, op)(X, dim)).to_numpy().reshape(-1)
    del X
    print("cfg2", time.time() - t0, flush=True)

    # config 3: dot and 2-norm of 2^30-element f32 Col vectors, default_rng(2)
    a, b = cfg3_inputs()
    ca, cb = M(a.reshape(-1, 1)), M(b.reshape(-1, 1))   # (Col.from_numpy fails in the reference)
    del a, b
    g["cfg3_dot"] = np.float32(dm.dot(ca, cb))
    g["cfg3_norm2"] = np.float64(dm.norm(ca, 2))
    del ca, cb
    print("cfg3", g["cfg3_dot"], g["cfg3_norm2"], time.time() - t0, flush=True)

    # config 4: C = A * trans(B) at 8192^3, f32 and f64, default_rng(3)
    ii, jj = gemm_sample_index(8192)
    for elem in ("f32", "f64"):
        a, b = cfg4_inputs(8192, elem)
        c = dm.evaluate(M(a) @ M(b).t()).to_numpy()
        g[f"cfg4_{elem}_samples"] = c[ii, jj]
        g[f"cfg4_{elem}_rowsum"] = c.astype(np.float64).sum(axis=1)
        del a, b, c
        print("cfg4", elem, time.time() - t0, flush=True)

    # config 5: logistic-regression step on 2^20 x 1024 f32, default_rng(5)
    x, w, y = cfg5_inputs()
    mX, mw, my = M(x), M(w), M(y)
    del x
    z = dm.evaluate(mX @ mw)
    r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - my)
    gr = dm.evaluate(mX.t() @ r)
    g["cfg5_g"] = gr.to_numpy().reshape(-1)
    g["cfg5_s"] = np.float32(dm.accu(r))
    g["cfg5_r_head"] = r.to_numpy().reshape(-1)[:65536]
    print("cfg5", time.time() - t0, flush=True)

    dm.shutdown()
    np.savez_compressed(OUT, **g)
    print("wrote", OUT, {k: v.shape for k, v in g.items()})


if __name__ == "__main__":
    main()
