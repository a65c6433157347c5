"""Parity at the exact BASELINE shapes and seeds (VERDICT r1
"weak" 1): the device path against the unmodified reference's results
(tests/golden/baseline.npz, tools/make_golden_baseline.py) on inputs
regenerated from the same seeds (tools/baseline_inputs.py), plus f64 host
truth where the reference itself is only within tolerance.

Bars: bit-exact for the IEEE-exact config-1 variant and the per-dimension
reductions; 1e-5 (f32) / 1e-12 (f64) relative for dot, norm, GEMM and the
logistic step, the reference's own metric (tests/dag_util.py:84-95).
"""
import numpy as np
import pytest

from conftest import golden
from tools.baseline_inputs import (cfg1_inputs, cfg2_input, cfg3_inputs, cfg4_inputs, cfg5_inputs,
                                   gemm_sample_index)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _rel(got, want) -> float:
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1.0))


@pytest.fixture(scope="module")
def gb():
    return golden("baseline")


def test_config1_4096_default_rng0(dm, gb):
    """accu(2*A + B % C - exp(D)) at 4096^2: the reference's -7857368.0.  The
    exp-free variant's bits are the reference's (same arithmetic, same order)."""
    A, B, C, D = (dm.Matrix.from_numpy(x) for x in cfg1_inputs())
    got = np.float32(dm.accu(2 * A + B % C - dm.exp(D)))
    assert _rel(got, gb["cfg1_accu_exp"]) <= 1e-5, (got, gb["cfg1_accu_exp"])
    assert got == np.float32(-7857368.0)
    noexp = np.float32(dm.accu(2 * A + B % C - D))
    assert noexp.tobytes() == np.float32(gb["cfg1_accu_noexp"]).tobytes()


def test_config2_16384_f64_bit_exact(dm, gb):
    X = dm.Matrix.from_numpy(cfg2_input())
    for op in ("sum", "min", "max"):
        for dim in (0, 1):
            got = dm.evaluate(getattr(dm, op)(X, dim)).to_numpy().reshape(-1)
            want = gb[f"cfg2_{op}{dim}"]
            assert got.tobytes() == want.tobytes(), (op, dim, _rel(got, want))


def test_config3_2pow30_dot_norm(dm, gb):
    a, b = cfg3_inputs()
    ca, cb = dm.Matrix.from_numpy(a.reshape(-1, 1)), dm.Matrix.from_numpy(b.reshape(-1, 1))
    # f64 truth in 64 chunks (host memory stays bounded)
    step = 1 << 24
    truth_dot = sum(float(np.dot(a[i:i + step].astype(np.float64), b[i:i + step].astype(np.float64)))
                    for i in range(0, a.size, step))
    truth_nrm = np.sqrt(sum(float(np.dot(a[i:i + step].astype(np.float64), a[i:i + step].astype(np.float64)))
                            for i in range(0, a.size, step)))
    del a, b
    d = dm.dot(ca, cb)
    nrm = dm.norm(ca, 2)
    assert _rel(d, gb["cfg3_dot"]) <= 1e-5 and _rel(d, truth_dot) <= 1e-5, (d, gb["cfg3_dot"], truth_dot)
    assert _rel(nrm, gb["cfg3_norm2"]) <= 1e-5 and _rel(nrm, truth_nrm) <= 1e-5, (nrm, gb["cfg3_norm2"])


@pytest.mark.parametrize("elem,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_config4_8192_full_matrix(dm, gb, elem, tol):
    """C = A * trans(B) at 8192^3: the whole matrix normwise against an f64
    host product, the reference's own entries and its row sums."""
    a, b = cfg4_inputs(8192, elem)
    C = dm.evaluate(dm.Matrix.from_numpy(a) @ dm.Matrix.from_numpy(b).t()).to_numpy()
    truth = a.astype(np.float64) @ b.astype(np.float64).T
    assert _rel(C, truth) <= tol
    ii, jj = gemm_sample_index(8192)
    assert _rel(C[ii, jj], gb[f"cfg4_{elem}_samples"]) <= tol
    assert _rel(C.astype(np.float64).sum(axis=1), gb[f"cfg4_{elem}_rowsum"]) <= tol


@pytest.mark.parametrize("fused", [False, True])
def test_config5_logistic_step_1M(dm, gb, fused):
    """z = X w, r = 1/(1+exp(-z)) - y, g = X^T r, s = accu(r) on 2^20 x 1024
    f32: the reference's g and s, and an f64 host step."""
    x, w, y = cfg5_inputs()
    X, W, Y = (dm.Matrix.from_numpy(v) for v in (x, w, y))
    if fused:
        r_e = 1 / (1 + dm.exp(0 - X @ W)) - Y
        r, g = dm.evaluate_many(r_e, X.t() @ r_e)
    else:
        z = dm.evaluate(X @ W)
        r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - Y)
        g = dm.evaluate(X.t() @ r)
    s = dm.accu(r)
    x64 = x.astype(np.float64)
    r64 = 1 / (1 + np.exp(-(x64 @ w.astype(np.float64)))) - y
    g64 = (x64.T @ r64).reshape(-1)
    del x64
    gg = g.to_numpy().reshape(-1)
    assert _rel(gg, gb["cfg5_g"]) <= 1e-5 and _rel(gg, g64) <= 1e-5
    assert _rel(s, gb["cfg5_s"]) <= 1e-5 and _rel(s, r64.sum()) <= 1e-5
    assert _rel(r.to_numpy().reshape(-1)[:65536], gb["cfg5_r_head"]) <= 1e-6
