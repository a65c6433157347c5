"""The oracle (oracle/devmat_oracle.py) must reproduce the unmodified
reference on its golden vectors (tests/golden, made by tools/make_golden.py),
and the summation order the device implements must be numpy's."""
import numpy as np
import pytest

import oracle as O
from conftest import golden


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    assert a.tobytes() == b.tobytes()


def test_chains_match_reference():
    g = golden("chains")
    prog_exp = (("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("load", 2),
                ("glue", "eglue_schur"), ("glue", "eglue_plus"), ("load", 3), ("unary", "eop_exp", None),
                ("glue", "eglue_minus"))
    for tag in ("a", "b", "c"):
        A, B, C, D = (g[f"{tag}_{x}"] for x in "ABCD")
        vals = [x.reshape(-1, order="F") for x in (A, B, C, D)]
        got = O.run_program(prog_exp, vals, np.float32).reshape(A.shape, order="F")
        _same(got, g[f"{tag}_chain_exp"])
        _same(O.reduce_accu(got.reshape(-1, order="F")), g[f"{tag}_accu_exp"])
        noexp = O.run_program(prog_exp[:7] + (("glue", "eglue_minus"),), vals, np.float32)
        _same(O.reduce_accu(noexp), g[f"{tag}_accu_noexp"])


def test_unary_ops_match_reference():
    g = golden("ops")
    for name in ("exp", "log", "log10", "sqrt", "square", "abs", "cos", "sin", "tan", "acos", "asin", "atan"):
        for dt, x in (("f32", g["xf"]), ("f64", g["xd"])):
            _same(O.apply_unary(f"eop_{name}", x, None, x.dtype), g[f"{dt}_{name}"])
    _same(O.apply_unary("eop_pow", g["xf"], 3, np.float32), g["f32_pow3"])
    _same(O.apply_unary("eop_pow", g["xd"], 2.5, np.float64), g["f64_pow2_5"])


def test_integer_ops_match_reference():
    g = golden("ops")
    xi, yi, xu = g["xi"], g["yi"], g["xu"]
    i32 = np.int32
    chain = O.apply_glue("eglue_minus", O.apply_scalar("eop_scalar_plus", O.apply_glue("eglue_schur", xi, xi, i32),
                                                       3, i32),
                         O.apply_scalar("eop_scalar_times", yi, 7, i32), i32)
    _same(chain, g["i32_chain"])
    _same(O.apply_scalar("eop_scalar_div_post", xi, 7, i32), g["i32_div_scalar"])
    sq = O.apply_scalar("eop_scalar_plus", O.apply_glue("eglue_schur", yi, yi, i32), 1, i32)
    _same(O.apply_scalar("eop_scalar_div_pre", sq, 1000, i32), g["i32_div_pre"])
    _same(O.apply_glue("eglue_div", xi, yi, i32), g["i32_div_glue"])
    _same(O.apply_unary("eop_square", O.apply_scalar("eop_scalar_times", xi, 1000, i32), None, i32), g["i32_square"])
    _same(O.apply_unary("eop_abs", yi, None, i32), g["i32_abs"])
    _same(O.apply_unary("eop_pow", yi, 3, i32), g["i32_pow"])
    _same(O.apply_unary("eop_sqrt", O.apply_unary("eop_abs", xi, None, i32), None, i32), g["i32_sqrt"])
    u = np.uint64
    c = O.apply_glue("eglue_minus", O.apply_scalar("eop_scalar_plus", O.apply_scalar("eop_scalar_times", xu, 3, u),
                                                    7, u),
                     O.apply_scalar("eop_scalar_div_post", xu, 5, u), u)
    _same(c, g["u64_chain"])
    _same(O.apply_scalar("eop_scalar_minus_pre", xu, 5, u), g["u64_minus_pre"])
    _same(O.apply_glue("eglue_div", xu, np.zeros_like(xu), u), g["u64_div0"])


def test_casts_match_reference():
    g = golden("casts")
    for src in ("edge", "edge_f32", "iv", "uv"):
        x = g["edge_f64"] if src == "edge" else g[src]
        for key in [k for k in g if k.startswith(src + "_to_")]:
            t = key.rsplit("_", 1)[1]
            _same(O.cast_out(x, O.NP_DTYPE[t]), g[key])


def test_reductions_match_reference():
    g = golden("reduce")
    for key in [k for k in g if k.endswith("_accu") and k[0] == "f"]:
        base = key[: -len("_accu")]
        x, y = g[base + "_x"], g[base + "_y"]
        _same(O.reduce_accu(x), g[key])
        _same(O.reduce_dot(x, y), g[base + "_dot"])
        assert O.norm_vector(x, 2) == float(g[base + "_norm2"])
        assert O.norm_vector(x, "inf") == float(g[base + "_norminf"])
        assert O.norm_vector(x, "-inf") == float(g[base + "_normm"])
        assert O.norm_vector(x, 3) == float(g[base + "_norm3"])
    assert int(O.reduce_accu(g["i32_x"])) == int(g["i32_accu"])
    assert int(O.reduce_accu(g["u64_x"])) == int(g["u64_accu"])
    for case in ("nan_first", "nan_second_block", "nan_two"):
        x = g[f"mm_{case}_x"]
        _same(np.float32(O.reduce_min(x)), g[f"mm_{case}_reduce_min"])
        _same(np.float32(O.reduce_max(x)), g[f"mm_{case}_reduce_max"])


def test_rdim_match_reference():
    g = golden("rdim")
    for key in [k for k in g if k.count("_") == 1]:
        a = g[key]
        for op in ("sum", "min", "max", "mean", "var", "stddev"):
            for dim in (0, 1):
                want = g.get(f"{key}_{op}{dim}")
                if want is None:
                    continue
                if op == "stddev":
                    got = O.stage_cast(np.sqrt(O.rdim("var", a, dim)), a.dtype)
                else:
                    got = O.rdim(op, a, dim)
                _same(got, want)


def test_gemm_match_reference():
    g = golden("gemm")
    for dt in ("f32", "f64"):
        a, b, bt = g[f"{dt}_a"], g[f"{dt}_b"], g[f"{dt}_bt"]
        _same(O.gemm(a, b), g[f"{dt}_ab"])
        # the reference materialises the transpose, then gemm (expr.py:543-547)
        _same(O.gemm(a, np.ascontiguousarray(bt.T)), g[f"{dt}_abt"])
    _same(O.gemm(g["i32_a"], g["i32_a"]), g["i32_aa"])


def test_misc_match_reference():
    g = golden("misc")
    for kind in ("fro", "inf", "-inf"):
        assert O.norm_matrix(g["mx"], kind) == float(g[f"mx_norm_{kind}"])
        assert O.norm_matrix(g["big"], kind) == float(g[f"big_norm_{kind}"])
    # RNG: the set_seed stream counter restarts at 0; randu is stream 0, randn stream 1
    for seed, dt in ((123, np.float32), (777, np.float64)):
        u = O.uniform_stream(seed, 0, 0, 40 * 25).astype(dt).reshape(40, 25, order="F")
        _same(u, g[f"randu_{seed}"])
        z = O.normal_stream(seed, 1, 0, 33 * 17).astype(dt).reshape(33, 17, order="F")
        _same(z, g[f"randn_{seed}"])
    gr, r, s = O.logistic_step(g["lr_X"], g["lr_w"], g["lr_y"])
    _same(r, g["lr_r"])
    np.testing.assert_allclose(gr, g["lr_g"], rtol=1e-5, atol=1e-6)
    _same(s, g["lr_s"])


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_numpy_pairwise_order_is_ndarray_sum(dt):
    """The device's summation order (bm_reduce.cuh) is numpy's pairwise sum."""
    rng = np.random.default_rng(7)
    for n in list(range(0, 140)) + [255, 256, 257, 1000, 2047, 2048, 4100, 8191, 8192, 8200]:
        a = (rng.standard_normal(n) * np.exp2(rng.integers(-20, 20, n))).astype(dt)
        _same(O.numpy_pairwise_sum(a), a.sum(dtype=dt))
    z = np.full(20, -0.0, dtype=dt)
    _same(O.numpy_pairwise_sum(z), z.sum(dtype=dt))


def test_row_sums_are_sequential_and_column_sums_pairwise():
    """rdim order (kernels.py:502-531): dim 1 folds columns left to right,
    dim 0 is numpy's pairwise sum down each column."""
    rng = np.random.default_rng(8)
    a = (rng.standard_normal((64, 333)) * np.exp2(rng.integers(-20, 20, (64, 333)))).astype(np.float32)
    row = O.rdim("sum", a, 1).reshape(-1)
    seq = np.zeros(64, dtype=np.float32)
    for j in range(a.shape[1]):
        seq = seq + a[:, j]
    _same(row, seq)
    col = O.rdim("sum", a, 0).reshape(-1)
    _same(col, np.array([O.numpy_pairwise_sum(np.ascontiguousarray(a[:, j])) for j in range(a.shape[1])]))


def test_combine_pairwise_is_hierarchical_over_aligned_groups():
    """Folding aligned power-of-two groups first, then their results, equals
    one combine_pairwise -- the property the device's CTA / rank split uses."""
    rng = np.random.default_rng(9)
    add = lambda a, b: np.float32(a + b)  # noqa: E731
    for n in (1, 2, 3, 7, 8, 9, 31, 64, 100, 257, 1000, 4099):
        parts = list((rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))).astype(np.float32))
        whole = O.combine_pairwise(parts, add)
        for g in (1, 2, 4, 8, 16, 64):
            groups = [O.combine_pairwise(parts[i:i + g], add) for i in range(0, n, g)]
            _same(O.combine_pairwise(groups, add), whole)
    for op in (O.py_min, O.py_max):
        parts = [1.0, np.nan, 3.0, 0.5, np.nan, 2.0, 7.0]
        whole = O.combine_pairwise(parts, op)
        for g in (1, 2, 4):
            groups = [O.combine_pairwise(parts[i:i + g], op) for i in range(0, len(parts), g)]
            got = O.combine_pairwise(groups, op)
            assert (np.isnan(got) and np.isnan(whole)) or got == whole


def test_cast_edge_cases():
    """numpy's x86 float->int casts that the device emulates (bm_common.cuh)."""
    x = np.array([np.nan, np.inf, -np.inf, 3e9, -3e9, -1.5, 2.7, 1e20, 2.0 ** 63, 2.0 ** 64])
    with np.errstate(invalid="ignore"):
        i32 = x.astype(np.int32)
        u64 = x.astype(np.uint64)
    imin = np.int32(-2147483648)
    assert list(i32) == [imin, imin, imin, imin, imin, -1, 2, imin, imin, imin]
    assert [int(v) for v in u64] == [2 ** 63, 0, 2 ** 63, 3000000000, 2 ** 64 - 3000000000, 2 ** 64 - 1, 2, 0,
                                     2 ** 63, 0]


def test_predicates_match_reference_golden():
    g = golden("pred")
    for elem in ("f32", "f64", "i32", "u64"):
        a = g[f"{elem}_x"]
        flat = np.asfortranarray(a).reshape(-1, order="F")
        for name, op in (("gt", ">"), ("lt", "<"), ("ge", ">="), ("le", "<=")):
            for ti, thr in enumerate((0.5, 2, -0.25)):
                want = g[f"{elem}_find_{name}_{ti}"]
                got = O.find_indices(a, op, thr)
                assert np.array_equal(got, want), (elem, op, thr)
                mask = O.predicate_mask(flat, op, thr)
                assert bool(mask.all()) == bool(g[f"{elem}_all_{name}_{ti}"])
                assert bool(mask.any()) == bool(g[f"{elem}_any_{name}_{ti}"])
        assert np.array_equal(O.find_indices(a), g[f"{elem}_find_nonzero"])
    assert list(g["eye_find"]) == [0, 4, 8]
