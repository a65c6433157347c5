"""The seeded host inputs of the BASELINE configs, one
definition shared by tools/make_golden_baseline.py (reference side),
tests/test_gpu_baseline_shapes.py and bench.py (device side)."""
from __future__ import annotations

import numpy as np

CFG1_N = 4096
CFG2_N = 16384
CFG3_N = 1 << 30
CFG5_M, CFG5_K = 1 << 20, 1024


def cfg1_inputs(n: int = CFG1_N):
    """A, B, C, D = default_rng(0).random((n, n), f32), in that order."""
    rng = np.random.default_rng(0)
    return [rng.random((n, n), dtype=np.float32) for _ in range(4)]


def cfg2_input(n: int = CFG2_N):
    """default_rng(1).random((n, n)) (f64)."""
    return np.random.default_rng(1).random((n, n))


def cfg3_inputs(n: int = CFG3_N):
    """a, b = default_rng(2).random(n, f32), sequentially."""
    rng = np.random.default_rng(2)
    a = rng.random(n, dtype=np.float32)
    b = rng.random(n, dtype=np.float32)
    return a, b


def cfg4_inputs(n: int, elem: str):
    """A, B = default_rng(3).random((n, n)).astype(dtype)."""
    rng = np.random.default_rng(3)
    dt = np.float32 if elem == "f32" else np.float64
    a = rng.random((n, n)).astype(dt)
    b = rng.random((n, n)).astype(dt)
    return a, b


def gemm_sample_index(n: int, count: int = 4096):
    """Fixed (i, j) entries of C checked at full size."""
    rng = np.random.default_rng(34)
    return rng.integers(0, n, count), rng.integers(0, n, count)


def cfg5_inputs(m: int = CFG5_M, k: int = CFG5_K):
    """X = default_rng(5).standard_normal((m, k), f32); w = 0.03 N(0,1) (k x 1);
    y ~ Bernoulli(0.5) in {0, 1} (m x 1), drawn in that order."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((m, k), dtype=np.float32)
    w = (0.03 * rng.standard_normal((k, 1))).astype(np.float32)
    y = (rng.random((m, 1)) < 0.5).astype(np.float32)
    return x, w, y
