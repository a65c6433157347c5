"""GPU parity: the CUDA path against the reference's golden vectors and the
CPU oracle on the same seeded inputs.

Bars: IEEE-exact element-wise ops, integer ops, casts and the
reduction *order* are bit-exact; transcendental ops are ULP-bounded
(rtol 2e-6, the reference's own test precedent, tests/test_kernels.py:36-45);
dot/norm within 1e-5 (f32) / 1e-12 (f64); GEMM normwise within 1e-5 / 1e-12.
"""
import numpy as np
import pytest

import oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu


def same_nan(a, b):
    """Bit-identical except that NaNs only have to be NaN on both sides: a NaN
    produced by device arithmetic (0x7fffffff) and numpy's reductions (the
    operand's payload on some paths, 0x7fc00000 on its SIMD paths) need not
    share a payload."""
    a, b = np.asarray(a), np.asarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape, (a.dtype, b.dtype, a.shape, b.shape)
    na, nb = np.isnan(a), np.isnan(b)
    assert np.array_equal(na, nb), "NaN positions differ"
    same(np.where(na, 0, a).astype(a.dtype), np.where(nb, 0, b).astype(b.dtype))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.dtype == b.dtype, (a.dtype, b.dtype)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.tobytes() != b.tobytes():
        bad = np.argwhere(a.reshape(-1).view(np.uint8) != b.reshape(-1).view(np.uint8))
        raise AssertionError(f"not bit-identical; first differing byte {bad[:3].ravel()} "
                             f"{a.reshape(-1)[:4]} vs {b.reshape(-1)[:4]}")


def ulp_close(a, b, rtol):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    np.testing.assert_allclose(a, b, rtol=rtol, atol=0)


def normwise(got, want, tol):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    err = np.abs(got - want).max() / max(np.abs(want).max(), 1.0)
    assert err <= tol, err


def rel_err(got, want):
    return abs(float(got) - float(want)) / max(abs(float(want)), 1.0)


# ---- element-wise ----------------------------------------------------------------------------

def test_config1_chain_and_accu_vs_reference(dm):
    g = golden("chains")
    for tag in ("a", "b", "c"):
        A, B, C, D = (dm.Matrix.from_numpy(g[f"{tag}_{x}"]) for x in "ABCD")
        same(dm.evaluate(2 * A + B % C - D).to_numpy(), g[f"{tag}_chain_noexp"])
        # exp differs from numpy's SIMD expf by ulps; cancellation in 2A+BC-exp(D)
        # makes a relative-per-element bound meaningless, so use the reference's
        # own metric (tests/dag_util.py:84-95): max|err| / max(max|want|, 1)
        normwise(dm.evaluate(2 * A + B % C - dm.exp(D)).to_numpy(), g[f"{tag}_chain_exp"], 1e-6)
        # the reduction order is the reference's: bit-exact without transcendentals
        same(np.float32(dm.accu(2 * A + B % C - D)), g[f"{tag}_accu_noexp"])
        assert rel_err(dm.accu(2 * A + B % C - dm.exp(D)), g[f"{tag}_accu_exp"]) <= 1e-5
        # sqrt and the arithmetic are IEEE-exact: bit-identical
        same(dm.evaluate(dm.sqrt(dm.absolute(A - 0.5) + 1.0) / (B + 1) * 3 - C % D + 0.25).to_numpy(),
             g[f"{tag}_deep"])


@pytest.mark.parametrize("name", ["exp", "log", "log10", "sqrt", "square", "abs", "cos", "sin", "tan", "acos",
                                  "asin", "atan"])
def test_unary_vs_reference(dm, name):
    g = golden("ops")
    fn = getattr(dm, "absolute" if name == "abs" else name)
    for dt, key in (("f32", "xf"), ("f64", "xd")):
        got = dm.evaluate(fn(dm.Matrix.from_numpy(g[key]))).to_numpy()
        if name in ("sqrt", "square", "abs"):
            same(got, g[f"{dt}_{name}"])
        else:
            ulp_close(got, g[f"{dt}_{name}"], 2e-6 if dt == "f32" else 1e-12)
    ulp_close(dm.evaluate(dm.power(dm.Matrix.from_numpy(g["xf"]), 3)).to_numpy(), g["f32_pow3"], 1e-6)
    ulp_close(dm.evaluate(dm.power(dm.Matrix.from_numpy(g["xd"]), 2.5)).to_numpy(), g["f64_pow2_5"], 1e-13)


def test_integer_ops_bit_exact(dm):
    g = golden("ops")
    mi, mj, mu = (dm.Matrix.from_numpy(g[k]) for k in ("xi", "yi", "xu"))
    same(dm.evaluate(mi % mi + 3 - mj * 7).to_numpy(), g["i32_chain"])
    same(dm.evaluate(mi / 7).to_numpy(), g["i32_div_scalar"])
    same(dm.evaluate(1000 / (mj % mj + 1)).to_numpy(), g["i32_div_pre"])
    same(dm.evaluate(mi / mj).to_numpy(), g["i32_div_glue"])
    same(dm.evaluate(dm.square(mi * 1000)).to_numpy(), g["i32_square"])
    same(dm.evaluate(dm.absolute(mj)).to_numpy(), g["i32_abs"])
    same(dm.evaluate(dm.power(mj, 3)).to_numpy(), g["i32_pow"])
    same(dm.evaluate(dm.sqrt(dm.absolute(mi))).to_numpy(), g["i32_sqrt"])
    same(dm.evaluate(mu * 3 + 7 - mu / 5).to_numpy(), g["u64_chain"])
    same(dm.evaluate(5 - mu).to_numpy(), g["u64_minus_pre"])
    same(dm.evaluate(mu / dm.evaluate(mu * 0)).to_numpy(), g["u64_div0"])


def test_casts_bit_exact(dm):
    g = golden("casts")
    for src, key in (("edge_f64", "edge"), ("edge_f32", "edge_f32"), ("iv", "iv"), ("uv", "uv")):
        m = dm.Matrix.from_numpy(g[src])
        for k in [k for k in g if k.startswith(key + "_to_")]:
            t = k.rsplit("_", 1)[1]
            got = dm.evaluate(dm.conv_to(m, t)).to_numpy()
            want = g[k]
            if want.dtype.kind == "f":
                # NaN payloads differ between x86 and the GPU; compare NaN-aware
                np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
                ok = ~np.isnan(want)
                same(got[ok], want[ok])
            else:
                same(got, want)


def test_fused_two_way_conversion_equals_convert_after(dm):
    rng = np.random.default_rng(17)
    a = dm.Matrix.from_numpy(rng.random((9, 9), dtype=np.float32))
    scaled = 10 * a + 1
    for target in ("f64", "i32", "u64"):
        fused = dm.evaluate(dm.conv_to(scaled, target)).to_numpy()
        plain = dm.evaluate(scaled)
        conv = dm.evaluate(dm.conv_to(plain, target), fuse=False).to_numpy()
        same(fused, conv)


def test_strided_views(dm):
    rng = np.random.default_rng(3)
    x = rng.random((40, 30), dtype=np.float32)
    m = dm.Matrix.from_numpy(x)
    same(dm.evaluate(2 * m.submat(3, 4, 33, 24) + 1).to_numpy(),
         O.apply_scalar("eop_scalar_plus", O.apply_scalar("eop_scalar_times", x[3:34, 4:25], 2, np.float32), 1,
                        np.float32))
    same(dm.evaluate(m.row(5) * 3).to_numpy(), (x[5:6, :] * np.float32(3)))
    same(dm.evaluate(m.diag() + 0).to_numpy(), np.diagonal(x).reshape(-1, 1).copy())


def test_large_vector_vectorised_and_tail(dm):
    n = (1 << 16) * 2 + 17
    rng = np.random.default_rng(5)
    v = rng.random(n, dtype=np.float32)
    mv = dm.Matrix.from_numpy(v.reshape(-1, 1))
    same(dm.evaluate(2 * mv).to_numpy().reshape(-1), v * np.float32(2))


# ---- scalar reductions ------------------------------------------------------------------------

def test_accu_dot_norm_vs_reference(dm):
    g = golden("reduce")
    for key in [k for k in g if k.endswith("_accu") and k[0] == "f"]:
        base = key[: -len("_accu")]
        x, y = g[base + "_x"], g[base + "_y"]
        mx, my = dm.Matrix.from_numpy(x.reshape(-1, 1)), dm.Matrix.from_numpy(y.reshape(-1, 1))
        tol = 1e-5 if x.dtype == np.float32 else 1e-12
        same(np.array(dm.accu(mx), dtype=x.dtype), g[key])          # numpy order reproduced
        assert rel_err(dm.dot(mx, my), g[base + "_dot"]) <= tol
        assert rel_err(dm.norm(mx, 2), g[base + "_norm2"]) <= tol
        assert dm.norm(mx, "inf") == float(g[base + "_norminf"])
        assert dm.norm(mx, "-inf") == float(g[base + "_normm"])
        assert rel_err(dm.norm(mx, 3), g[base + "_norm3"]) <= (1e-5 if x.dtype == np.float32 else 1e-12)
    assert dm.accu(dm.Matrix.from_numpy(g["i32_x"].reshape(-1, 1))) == int(g["i32_accu"])
    assert dm.accu(dm.Matrix.from_numpy(g["u64_x"].reshape(-1, 1))) == int(g["u64_accu"])


def test_min_max_nan_semantics(dm):
    g = golden("reduce")
    for case in ("nan_first", "nan_second_block", "nan_two"):
        m = dm.Matrix.from_numpy(g[f"mm_{case}_x"].reshape(-1, 1))
        for op, key in (("min", "reduce_min"), ("max", "reduce_max")):
            got = np.float32(getattr(dm, f"reduce_{op}")(m))
            want = g[f"mm_{case}_{key}"]
            assert (np.isnan(got) and np.isnan(want)) or got == want, (case, op, got, want)


def test_min_max_empty_raises(dm):
    e = dm.Col(0)
    with pytest.raises(ValueError):
        dm.reduce_min(e)
    assert dm.accu(dm.Matrix(0, 0)) == 0


@pytest.mark.parametrize("n", [1, 5, 127, 128, 129, 2047, 2048, 2049, 8192 * 5 + 3, 1 << 20, (1 << 20) + 999])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_accu_bit_exact_sizes(dm, n, dt):
    rng = np.random.default_rng(n)
    v = (rng.standard_normal(n) * np.exp2(rng.integers(-16, 16, n))).astype(dt)
    m = dm.Matrix.from_numpy(v.reshape(-1, 1))
    same(np.array(dm.accu(m), dtype=dt), O.reduce_accu(v))


def test_accu_fused_expression_bit_exact_large(dm):
    rng = np.random.default_rng(0)
    A, B, C, D = (rng.random((1024, 1024), dtype=np.float32) for _ in range(4))
    mA, mB, mC, mD = (dm.Matrix.from_numpy(x) for x in (A, B, C, D))
    flat = [x.reshape(-1, order="F") for x in (A, B, C, D)]
    prog = (("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("load", 2), ("glue", "eglue_schur"),
            ("glue", "eglue_plus"), ("load", 3), ("glue", "eglue_minus"))
    same(np.float32(dm.accu(2 * mA + mB % mC - mD)), O.reduce_accu(O.run_program(prog, flat, np.float32)))


# ---- per-dimension reductions ------------------------------------------------------------------

def test_rdim_vs_reference(dm):
    g = golden("rdim")
    for key in [k for k in g if k.count("_") == 1]:
        a = g[key]
        m = dm.Matrix.from_numpy(a)
        for op in ("sum", "min", "max", "mean", "var", "stddev"):
            for dim in (0, 1):
                want = g.get(f"{key}_{op}{dim}")
                if want is None:
                    continue
                got = dm.evaluate(getattr(dm, op)(m, dim)).to_numpy()
                if op in ("var", "stddev"):
                    tol = 1e-5 if a.dtype == np.float32 else 1e-12
                    np.testing.assert_allclose(got, want, rtol=tol, atol=tol)
                else:
                    same(got, want)


@pytest.mark.parametrize("shape", [(16384, 64), (2048, 3000), (1000, 1000), (4096, 4096)])
def test_rdim_large_bit_exact(dm, shape):
    rng = np.random.default_rng(1)
    a = rng.random(shape)
    m = dm.Matrix.from_numpy(a)
    for op in ("sum", "min", "max"):
        for dim in (0, 1):
            same(dm.evaluate(getattr(dm, op)(m, dim)).to_numpy(), O.rdim(op, a, dim))


@pytest.mark.parametrize("dt,shape", [(np.float32, (4096, 300)), (np.float32, (1024, 7)), (np.float64, (512, 1500)),
                                      (np.float64, (8192, 1))])
def test_rdim0_sum_mean_streamed_bit_exact(dm, dt, shape):
    """column lengths that are a power-of-two number of half-units take the
    streamed dim-0 path; sum and mean stay bit-exact with the reference"""
    a = (np.random.default_rng(7).random(shape) - 0.25).astype(dt)
    m = dm.Matrix.from_numpy(a)
    for op in ("sum", "mean"):
        same(dm.evaluate(getattr(dm, op)(m, 0)).to_numpy(), O.rdim(op, a, 0))


@pytest.mark.parametrize("dt,shape", [(np.float64, (4096, 37)), (np.float32, (8192, 20)), (np.float64, (12288, 9)),
                                      (np.int32, (8192, 5))])
def test_rdim0_minmax_cta_path_nan(dm, dt, shape):
    """columns of a multiple of 8 half-units take the CTA-per-column dim-0
    path; min/max propagate NaN like numpy and are exact"""
    rng = np.random.default_rng(11)
    if np.issubdtype(dt, np.integer):
        a = rng.integers(-10**6, 10**6, size=shape).astype(dt)
    else:
        a = rng.standard_normal(shape).astype(dt)
        a[shape[0] - 1, 0] = np.nan
        a[3 * shape[0] // 4, shape[1] - 1] = np.nan
    m = dm.Matrix.from_numpy(a)
    for op in ("min", "max"):
        same(dm.evaluate(getattr(dm, op)(m, 0)).to_numpy(), O.rdim(op, a, 0))


@pytest.mark.parametrize("dt,shape", [(np.float32, (8192, 40)), (np.float64, (4096, 37)), (np.float32, (4096, 300)),
                                      (np.float64, (1000, 33)), (np.float32, (999, 17)), (np.int32, (2048, 9)),
                                      (np.float64, (12288, 11))])
def test_fused_dim0_reduction_of_a_tree(dm, dt, shape):
    """sum / mean / min / max(·, 0) of an element-wise tree run as one fused
    kernel and give the bits of reducing the materialised tree (the
    reference's two steps), NaNs included"""
    rng = np.random.default_rng(shape[0] + shape[1])
    if np.issubdtype(dt, np.integer):
        a = rng.integers(-1000, 1000, size=shape).astype(dt)
        b = rng.integers(-1000, 1000, size=shape).astype(dt)
    else:
        a = rng.standard_normal(shape).astype(dt)
        b = rng.standard_normal(shape).astype(dt)
        b[shape[0] // 3, 0] = np.nan
    A, B = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    tree = lambda: 3 * A + B % A - 2
    launches = []
    for op in ("sum", "mean", "min", "max"):
        assert [s.kernel for s in dm.plan(getattr(dm, op)(tree(), 0)).steps] == ["fused_rdim"]
        c0 = dm.counters().launches
        got = dm.evaluate(getattr(dm, op)(tree(), 0)).to_numpy()
        launches.append(dm.counters().launches - c0)
        mat = dm.evaluate(tree()).to_numpy()
        same(got, O.rdim(op, mat, 0))
    assert launches == [1, 1, 1, 1]
    if np.issubdtype(dt, np.floating):
        mat = dm.evaluate(tree()).to_numpy()
        tol = 1e-5 if dt == np.float32 else 1e-12
        for op in ("var", "stddev"):
            assert [s.kernel for s in dm.plan(getattr(dm, op)(tree(), 0)).steps][0] == "fused_rdim"
            got = dm.evaluate(getattr(dm, op)(tree(), 0)).to_numpy().astype(np.float64)
            want = O.rdim("var", mat, 0).astype(np.float64)
            if op == "stddev":
                want = np.sqrt(want)
            ok = np.isnan(want) == np.isnan(got)
            assert ok.all()
            m = ~np.isnan(want)
            np.testing.assert_allclose(got[m], want[m], rtol=tol, atol=tol)


@pytest.mark.parametrize("dt,shape", [(np.float32, (8192, 40)), (np.float64, (4096, 37)), (np.float32, (300, 1000)),
                                      (np.float64, (1000, 33)), (np.int32, (2048, 9)), (np.float32, (130, 70)),
                                      (np.float32, (64 * 5 + 1, 20)), (np.float32, (999, 17)), (np.float32, (4, 3)),
                                      (np.float32, (16, 5)), (np.float64, (8, 1000))])
def test_fused_dim1_reduction_of_a_tree(dm, dt, shape):
    """sum / mean / min / max(·, 1) of an element-wise tree: one TMA-staged
    kernel where the rows allow it (16-B columns, no lone-row block), the
    reference's two steps otherwise -- the bits of reducing the materialised
    tree either way, NaNs included"""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    if np.issubdtype(dt, np.integer):
        a = rng.integers(-1000, 1000, size=shape).astype(dt)
        b = rng.integers(-1000, 1000, size=shape).astype(dt)
    else:
        a = rng.standard_normal(shape).astype(dt)
        b = rng.standard_normal(shape).astype(dt)
        b[0, shape[1] // 2] = np.nan
    A, B = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    tree = lambda: 3 * A + B % A - 2
    fusable = (shape[0] * a.itemsize) % 16 == 0 and shape[0] % 64 != 1
    for op in ("sum", "mean", "min", "max"):
        kernels = [s.kernel for s in dm.plan(getattr(dm, op)(tree(), 1)).steps]
        assert (kernels == ["fused_rdim"]) == fusable, kernels
        got = dm.evaluate(getattr(dm, op)(tree(), 1)).to_numpy()
        mat = dm.evaluate(tree()).to_numpy()
        (same_nan if np.issubdtype(dt, np.floating) else same)(got, O.rdim(op, mat, 1))
    if np.issubdtype(dt, np.floating):
        mat = dm.evaluate(tree()).to_numpy()
        tol = 1e-5 if dt == np.float32 else 1e-12
        got = dm.evaluate(dm.var(tree(), 1)).to_numpy().astype(np.float64)
        want = O.rdim("var", mat, 1).astype(np.float64)
        assert (np.isnan(want) == np.isnan(got)).all()
        m = ~np.isnan(want)
        np.testing.assert_allclose(got[m], want[m], rtol=tol, atol=tol)


@pytest.mark.parametrize("nin,dt", [(1, np.float32), (3, np.float32), (4, np.float32), (5, np.float32),
                                    (8, np.float32), (8, np.float64), (9, np.float32)])
def test_fused_dim1_input_counts(dm, nin, dt):
    """1-8 inputs run the fused TMA row fold (64 / 32 / 16 / 8-column tiles); a
    ninth input keeps the reference's two steps; the bits match either way"""
    rng = np.random.default_rng(40 + nin)
    arrs = [rng.standard_normal((448, 37)).astype(dt) for _ in range(nin)]
    ms = [dm.Matrix.from_numpy(x) for x in arrs]
    tree = 2 * ms[0] + 1
    for m_ in ms[1:]:
        tree = tree * m_ + 1
    kernels = [s.kernel for s in dm.plan(dm.sum(tree, 1)).steps]
    assert (kernels == ["fused_rdim"]) == (nin <= 8), kernels
    got = dm.evaluate(dm.sum(tree, 1)).to_numpy()
    same(got, O.rdim("sum", dm.evaluate(tree).to_numpy(), 1))


# ---- GEMM ----------------------------------------------------------------------------------------

def test_gemm_vs_reference(dm):
    g = golden("gemm")
    for dt, tol in (("f32", 1e-5), ("f64", 1e-12)):
        a, b, bt = (dm.Matrix.from_numpy(g[f"{dt}_{k}"]) for k in ("a", "b", "bt"))
        for got, key in ((dm.gemm(a, b), "ab"), (dm.evaluate(a @ bt.t()), "abt")):
            want = g[f"{dt}_{key}"]
            err = np.abs(got.to_numpy().astype(np.float64) - want).max() / np.abs(want).max()
            assert err <= tol, (dt, key, err)
    same(dm.gemm(dm.Matrix.from_numpy(g["i32_a"]), dm.Matrix.from_numpy(g["i32_a"])).to_numpy(), g["i32_aa"])
    z = dm.evaluate(dm.Matrix(3, 0) @ dm.Matrix(0, 4)).to_numpy()
    same(z, g["f32_inner0"])


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (512, 384, 1024), (1000, 777, 333), (128, 128, 4096)])
@pytest.mark.parametrize("tb", [0, 1])
def test_gemm_shapes(dm, dt, m, n, k, tb):
    rng = np.random.default_rng(m + n + k)
    a = rng.random((m, k)).astype(dt)
    b = rng.random((n, k) if tb else (k, n)).astype(dt)
    ma, mb = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    got = dm.evaluate(ma @ (mb.t() if tb else mb)).to_numpy().astype(np.float64)
    ref = a.astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= (1e-5 if dt == np.float32 else 1e-12), err


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("m,n,k", [(384, 256, 320), (333, 258, 129), (334, 257, 130)])
@pytest.mark.parametrize("tb", [0, 1])
def test_gemm_trans_a_and_offset_views(dm, dt, m, n, k, tb):
    """trans(A) operands and operands that start at an odd element offset
    (the f64 kernel's 16-byte pair copies must fall back to 8-byte copies)"""
    rng = np.random.default_rng(m * n + k)
    a = rng.random((k, m)).astype(dt)
    b = rng.random((n, k) if tb else (k, n)).astype(dt)
    ref = a.T.astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    ma, mb = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    got = dm.evaluate(ma.t() @ (mb.t() if tb else mb)).to_numpy().astype(np.float64)
    tol = 1e-5 if dt == np.float32 else 1e-12
    assert np.abs(got - ref).max() / np.abs(ref).max() <= tol
    # through a subview (materialised first) ...
    wa = np.concatenate([rng.random((k, 1)).astype(dt), a], axis=1)
    big = dm.Matrix.from_numpy(wa)
    got = dm.evaluate(dm.trans(big.cols(1, m)) @ (mb.t() if tb else mb)).to_numpy().astype(np.float64)
    assert np.abs(got - ref).max() / np.abs(ref).max() <= tol
    # ... and straight through the operator ABI with op(A) = A stored one
    # column into a wider buffer (odd base offset when m is odd) and B the
    # same way (odd when its row count is odd)
    from paper_2308_03120_b200 import runtime as R
    at = np.ascontiguousarray(a.T)
    rb, cb = b.shape
    wa2 = dm.Matrix.from_numpy(np.concatenate([np.zeros((m, 1), dt), at], axis=1))
    wb2 = dm.Matrix.from_numpy(np.concatenate([np.zeros((rb, 1), dt), b], axis=1))
    out = dm.Matrix(m, n, elem_type=mb.elem_type)
    inv = dm.KernelInvocation("gemm", (R.BlockView(wa2.mem, m, m, k, m), R.BlockView(wb2.mem, rb, rb, cb, rb)),
                              R.BlockView(out.mem, 0, m, n, m), (), {"trans_a": 0, "trans_b": tb})
    R.get_runtime().enqueue(inv)
    got = out.to_numpy().astype(np.float64)
    assert np.abs(got - ref).max() / np.abs(ref).max() <= tol


def test_logistic_step_vs_reference(dm):
    g = golden("misc")
    X, w, y = (dm.Matrix.from_numpy(g[k]) for k in ("lr_X", "lr_w", "lr_y"))
    z = dm.evaluate(X @ w)
    r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - y)
    gr = dm.evaluate(X.t() @ r)
    ulp_close(r.to_numpy(), g["lr_r"], 1e-5)
    np.testing.assert_allclose(gr.to_numpy(), g["lr_g"], rtol=1e-4, atol=1e-5)
    assert rel_err(dm.accu(r), g["lr_s"]) <= 1e-4


def test_rng_bit_exact(dm):
    g = golden("misc")
    for seed, elem in ((123, "f32"), (777, "f64")):
        dm.set_seed(seed)
        same(dm.Matrix(40, 25, fill="randu", elem_type=elem).to_numpy(), g[f"randu_{seed}"])
        got = dm.Matrix(33, 17, fill="randn", elem_type=elem).to_numpy()
        ulp_close(got, g[f"randn_{seed}"], 1e-6 if elem == "f32" else 1e-13)


@pytest.mark.slow
def test_large_reductions_external_fold(dm):
    """n large enough that the final fold runs as separate chunk kernels."""
    n = (1 << 28) + 12345
    rng = np.random.default_rng(11)
    v = rng.random(n, dtype=np.float32)
    w = rng.random(n, dtype=np.float32)
    mv, mw = dm.Matrix.from_numpy(v.reshape(-1, 1)), dm.Matrix.from_numpy(w.reshape(-1, 1))
    same(np.float32(dm.accu(mv)), O.reduce_accu(v))
    same(np.float32(dm.reduce_max(mv)), np.float32(O.reduce_max(v)))
    same(np.float32(dm.reduce_min(mv)), np.float32(O.reduce_min(v)))
    assert rel_err(dm.dot(mv, mw), O.reduce_dot(v, w)) <= 1e-5
    vd = v[: 1 << 27].astype(np.float64)
    same(np.float64(dm.accu(dm.Matrix.from_numpy(vd.reshape(-1, 1)))), O.reduce_accu(vd))


def test_beyond_2_31_elements(dm):
    """64-bit element indexing end to end: 2^31 + 1000 f64 elements (17 GB,
    generated on the device) through a fused store, accu, min/max, dot and a
    dim-0 sum; every value is exact in f64, so the results are known."""
    n = (1 << 31) + 1000
    x = dm.Matrix(n, 1, fill="ones", elem_type="f64")
    assert dm.accu(x) == float(n)
    assert dm.reduce_min(x) == 1.0 and dm.reduce_max(x) == 1.0
    assert dm.dot(x, x) == float(n)
    y = dm.evaluate(2 * x + 1)
    assert dm.accu(y) == 3.0 * n
    assert dm.accu(y - 3) == 0.0
    del y
    m = dm.Matrix(1 << 16, (1 << 15) + 3, fill="ones", elem_type="f64")   # 2^31 + 3 * 2^16 elements
    s = dm.evaluate(dm.sum(m, 0)).to_numpy()
    assert s.shape == (1, (1 << 15) + 3) and np.all(s == float(1 << 16))
    assert dm.accu(m) == float(m.n_elem)


def test_back_to_back_reductions_stay_ordered_with_stores(dm):
    """Reductions launch as programmatic dependents (PDL) and overlap their
    predecessor's final fold.  Interleave stores that rewrite the reduced
    matrix with device-resident reductions and no host synchronisation: every
    reduction must see exactly the store before it, and consecutive
    reductions must not corrupt each other's scratch."""
    import torch
    from paper_2308_03120_b200 import dist as D
    D.bind_torch_stream()   # torch's partial tensors and the kernels on one stream
    n = 2048
    base = np.random.default_rng(3).random((n, n), dtype=np.float32)
    A = dm.Matrix.from_numpy(base)
    X = dm.Matrix(n, n)
    reds = []
    for k in range(24):
        dm.evaluate(A * float(k + 1), out=X)
        r = D.ShardedReduction("accu", X)
        r.launch()
        r2 = D.ShardedReduction("accu", A * float(k + 1) + 1.0)   # back-to-back reduction, no store between
        r2.launch()
        reds.append((k, r, r2))
    torch.cuda.synchronize()
    flat = base.reshape(-1, order="F")
    for k, r, r2 in reds:
        scaled = (flat * np.float32(k + 1)).astype(np.float32)
        same(np.float32(r.partial.cpu().numpy()[0]), O.reduce_accu(scaled))
        same(np.float32(r2.partial.cpu().numpy()[0]), O.reduce_accu((scaled + np.float32(1)).astype(np.float32)))


def test_sharded_helpers_at_world_size_one(dm):
    """dist helpers on one GPU (no process group): the zero-copy torch view,
    dim-0/dim-1 reductions, the NT GEMM block and the logistic step."""
    import torch
    from paper_2308_03120_b200 import dist as D
    D.bind_torch_stream()
    a = np.random.default_rng(8).random((300, 200))
    m = dm.Matrix.from_numpy(a)
    t = D.torch_view(m)
    assert t.numel() == a.size and t.dtype == torch.float64
    same(t.cpu().numpy(), np.asfortranarray(a).reshape(-1, order="F"))
    t.mul_(2.0)
    torch.cuda.synchronize()
    same(m.to_numpy(), 2 * a)
    for op in ("sum", "min", "max"):
        for dim in (0, 1):
            same(D.sharded_reduce_dim(op, m, dim).to_numpy(), O.rdim(op, 2 * a, dim))
    b = np.random.default_rng(9).random((64, 200))
    c = D.sharded_gemm_nt(m, dm.Matrix.from_numpy(b)).to_numpy()
    normwise(c, (2 * a) @ b.T, 1e-12)
    rng = np.random.default_rng(10)
    X = rng.standard_normal((4096, 256)).astype(np.float32)
    w = (0.03 * rng.standard_normal((256, 1))).astype(np.float32)
    y = (rng.random((4096, 1)) < 0.5).astype(np.float32)
    g, s = D.sharded_logistic_step(dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(w), dm.Matrix.from_numpy(y))
    rf = 1 / (1 + np.exp(-(X.astype(np.float64) @ w))) - y
    normwise(g.to_numpy(), X.T.astype(np.float64) @ rf, 1e-5)
    assert rel_err(s, rf.sum()) <= 1e-5


@pytest.mark.slow
@pytest.mark.parametrize("elem,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_gemm_nt_32768_sampled(dm, elem, tol):
    """Config 4 at full size: C = A * B^T at 32768^3 (3xTF32 / DMMA), checked
    on sampled entries against f64 dot products of the operand rows
    (the CPU reference at this size costs minutes)."""
    n = 32768
    dm.set_seed(3)
    A = dm.Matrix(n, n, fill="randu", elem_type=elem)
    B = dm.Matrix(n, n, fill="randu", elem_type=elem)
    C = dm.evaluate(A @ B.t())
    rng = np.random.default_rng(12)
    for i, j in zip(rng.integers(0, n, 12), rng.integers(0, n, 12)):
        a = dm.evaluate(A.row(int(i))).to_numpy().astype(np.float64).reshape(-1)
        b = dm.evaluate(B.row(int(j))).to_numpy().astype(np.float64).reshape(-1)
        ref = float(a @ b)
        got = C.at(int(i), int(j))
        assert abs(got - ref) / abs(ref) <= tol, (i, j, got, ref)


@pytest.mark.slow
@pytest.mark.parametrize("elem,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_gemm_nt_32768_full_normwise(dm, elem, tol):
    """Config 4 at full size, every entry: C = A * B^T at 32768^3 against an
    f64 cuBLAS product of the same operands on this GPU (max-normalised error;
    the 4 K-pass 3xTF32 path and the DMMA path)."""
    import torch
    from paper_2308_03120_b200 import dist as D
    n = 32768
    dm.set_seed(3)
    A = dm.Matrix(n, n, fill="randu", elem_type=elem)
    B = dm.Matrix(n, n, fill="randu", elem_type=elem)
    C = dm.evaluate(A @ B.t())
    dm.synchronise()
    ta = D.torch_view(A).view(n, n).t().double()      # column-major storage -> (row, col)
    tb = D.torch_view(B).view(n, n).t().double()
    truth = ta @ tb.t()
    del ta, tb
    got = D.torch_view(C).view(n, n).t().double()
    err = float((got - truth).abs().max() / truth.abs().max())
    del got, truth
    torch.cuda.empty_cache()
    assert err <= tol, err


# ---- predicates: find / all / any (ops.py:202-262) ----------------------------------------------

def test_predicates_vs_reference(dm):
    g = golden("pred")
    for elem in ("f32", "f64", "i32", "u64"):
        a = g[f"{elem}_x"]
        m = dm.Matrix.from_numpy(a)
        for name, op in (("gt", ">"), ("lt", "<"), ("ge", ">="), ("le", "<=")):
            for ti, thr in enumerate((0.5, 2, -0.25)):
                rel = {">": m > thr, "<": m < thr, ">=": m >= thr, "<=": m <= thr}[op]
                idx = dm.find(rel)
                assert idx.elem_type == "u64"
                same(idx.to_numpy().reshape(-1), g[f"{elem}_find_{name}_{ti}"])
                assert dm.all(rel) == bool(g[f"{elem}_all_{name}_{ti}"])
                assert dm.any(rel) == bool(g[f"{elem}_any_{name}_{ti}"])
        same(dm.find(m).to_numpy().reshape(-1), g[f"{elem}_find_nonzero"])
        assert dm.all(m) == bool(g[f"{elem}_all_nonzero"]) and dm.any(m) == bool(g[f"{elem}_any_nonzero"])
    same(dm.find(dm.Matrix(3, 3, fill="eye")).to_numpy().reshape(-1), g["eye_find"])
    same(dm.find(dm.Matrix.from_numpy(g["f32_x"]) * 2 - 1 > 0.25).to_numpy().reshape(-1), g["expr_find"])


def test_predicate_conventions_and_transfers(dm):
    """tests/test_kernels.py:235-274 of the reference."""
    assert dm.find(dm.Matrix(3, 3, fill="zeros")).n_rows == 0
    m = dm.Matrix(4, 4, fill="ones")
    assert dm.all(m) and dm.any(m) and dm.all(m < 2) and not dm.any(m > 5)
    z = dm.Matrix(4, 4, fill="zeros")
    assert not dm.any(z) and not dm.all(z)
    e = dm.Matrix(0, 0)
    assert dm.all(e) is True and dm.any(e) is False
    dm.set_seed(33)
    r = dm.Matrix(1000, 1000, fill="randu")
    host = r.to_numpy()
    dm.synchronise()
    before = dm.counters()
    count = dm.find(r > 0.3).n_rows
    delta = dm.counters() - before
    assert count == int((host > np.float32(0.3)).sum())
    assert delta.transfers_d2h <= 2
    idx = dm.find(dm.Matrix(3, 3, fill="eye"))
    assert dm.accu(idx) == 12


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 1 << 20, (1 << 24) + 77])
def test_find_large_vs_oracle(dm, n):
    rng = np.random.default_rng(n)
    v = rng.random(n, dtype=np.float32)
    v[rng.random(n) < 0.01] = np.nan
    m = dm.Matrix.from_numpy(v.reshape(-1, 1))
    for op, thr in ((">", 0.7), ("<=", 0.01), ("!=", 0.5)):
        rel = {">": m > thr, "<=": m <= thr}.get(op)
        if rel is None:
            from paper_2308_03120_b200.expr import Relational
            rel = Relational(op, m, thr)
        same(dm.find(rel).to_numpy().reshape(-1), O.find_indices(v, op, thr))


# ---- fused single-pass logistic step (bm_lgrad.cuh) -------------------------------------------------

def test_fused_logistic_step_vs_reference(dm):
    """r, g = evaluate_many(F(X@w, y), X.t() @ F(...)) is one fused kernel
    reading X once; same tolerances as the unfused reference step."""
    g = golden("misc")
    X, w, y = (dm.Matrix.from_numpy(g[k]) for k in ("lr_X", "lr_w", "lr_y"))
    r_e = 1 / (1 + dm.exp(0 - X @ w)) - y
    p = dm.plan(X.t() @ r_e)
    assert [s.kernel for s in p.steps] == ["logistic_grad"]
    r, gr = dm.evaluate_many(r_e, X.t() @ r_e)
    ulp_close(r.to_numpy(), g["lr_r"], 1e-5)
    np.testing.assert_allclose(gr.to_numpy(), g["lr_g"], rtol=1e-4, atol=1e-5)
    assert rel_err(dm.accu(r), g["lr_s"]) <= 1e-4
    # the single-expression form (no r returned)
    np.testing.assert_allclose(dm.evaluate(X.t() @ r_e).to_numpy(), g["lr_g"], rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("m,k", [(1 << 16, 1024), (4100, 300), (4096 * 3 + 16, 1000), (16, 16), (1024, 513),
                                 (2052, 1), (1 << 15, 1500), (8192 + 64, 2048), (20000, 4096), (4096, 3000)])
def test_fused_logistic_step_large(dm, m, k):
    rng = np.random.default_rng(m + k)
    X = rng.standard_normal((m, k), dtype=np.float32)
    w = (0.03 * rng.standard_normal((k, 1))).astype(np.float32)
    y = (rng.random((m, 1)) < 0.5).astype(np.float32)
    mX, mw, my = dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(w), dm.Matrix.from_numpy(y)
    r_e = 1 / (1 + dm.exp(0 - mX @ mw)) - my
    assert [s.kernel for s in dm.plan(mX.t() @ r_e).steps] == ["logistic_grad"]
    r, gr = dm.evaluate_many(r_e, mX.t() @ r_e)
    # unfused device path (GEMV + chain + GEMV) and an f64 host reference
    r2 = dm.evaluate(1 / (1 + dm.exp(0 - dm.evaluate(mX @ mw))) - my)
    g2 = dm.evaluate(mX.t() @ r2)
    rf = 1 / (1 + np.exp(-(X.astype(np.float64) @ w))) - y
    gf = X.T.astype(np.float64) @ rf
    normwise(r.to_numpy(), rf, 1e-5)
    normwise(gr.to_numpy(), gf, 1e-5)
    normwise(gr.to_numpy(), g2.to_numpy(), 1e-5)
    # deterministic: a second run is bit-identical
    r3, g3 = dm.evaluate_many(r_e, mX.t() @ r_e)
    same(g3.to_numpy(), gr.to_numpy())
    same(r3.to_numpy(), r.to_numpy())


@pytest.mark.parametrize("m,k", [(1 << 20, 64), (8192 * 3 + 128 * 5 + 64, 96), (8192 * 2, 32), (100, 8),
                                 (4100, 300), (64 * 37, 16), (8192 * 4 + 4, 2500)])
def test_fused_logistic_accu_side_output_bit_exact(dm, m, k):
    """The logistic kernel also folds accu(r) in the reference's order (numpy
    leaves inside the kernel, blocks + combine_pairwise in lgrad_finish), and
    accu() of the returned r reads it: bit-identical to the oracle's
    reduce_accu of the same r, with no reduction launched."""
    rng = np.random.default_rng(m ^ k)
    X = rng.standard_normal((m, k), dtype=np.float32)
    w = (0.05 * rng.standard_normal((k, 1))).astype(np.float32)
    y = (rng.random((m, 1)) < 0.5).astype(np.float32)
    mX, mw, my = dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(w), dm.Matrix.from_numpy(y)
    r_e = 1 / (1 + dm.exp(0 - mX @ mw)) - my
    r, gr = dm.evaluate_many(r_e, mX.t() @ r_e)
    rv = r.to_numpy().reshape(-1, order="F")
    want = O.reduce_accu(rv)
    dm.synchronise()
    before = dm.counters()
    got = dm.accu(r)
    assert (dm.counters() - before).launches == 0          # served from the sum cache
    assert np.float32(got).tobytes() == np.float32(want).tobytes(), (got, want)
    # a second step with the same operands gives the same bits
    r2, _ = dm.evaluate_many(r_e, mX.t() @ r_e)
    assert np.float32(dm.accu(r2)).tobytes() == np.float32(want).tobytes()


def test_sum_cache_forgets_on_write(dm):
    """Any write to the matrix drops the cached accu: element writes,
    evaluate(out=...), host copies and torch views."""
    from paper_2308_03120_b200 import dist as D
    m, k = 8192 * 2 + 64, 48
    rng = np.random.default_rng(7)
    X = rng.standard_normal((m, k), dtype=np.float32)
    w = (0.05 * rng.standard_normal((k, 1))).astype(np.float32)
    y = (rng.random((m, 1)) < 0.5).astype(np.float32)
    mX, mw, my = dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(w), dm.Matrix.from_numpy(y)
    r_e = 1 / (1 + dm.exp(0 - mX @ mw)) - my

    def fresh():
        r, _ = dm.evaluate_many(r_e, mX.t() @ r_e)
        return r

    def check(r):
        v = r.to_numpy().reshape(-1, order="F")
        assert np.float32(dm.accu(r)).tobytes() == np.float32(O.reduce_accu(v)).tobytes()

    r = fresh()
    r[5, 0] = 1000.0
    check(r)
    r = fresh()
    dm.evaluate(2 * my, out=r)
    check(r)
    r = fresh()
    dm.runtime.get_runtime().copy_h2d(np.ones(m, np.float32), r.mem)
    check(r)
    r = fresh()
    D.torch_view(r).fill_(0.25)
    check(r)
    r = fresh()
    r2 = r
    del r
    check(r2)


def test_plan_recipes_rebind_leaves(dm):
    """A recipe (plan + invocations built once per DAG shape) serves later
    calls with other matrices of the same shapes: results equal a fresh plan
    of each call, including aliasing outputs, shared leaves, reductions and
    evaluate_many duplicates."""
    from paper_2308_03120_b200 import expr as E
    rng = np.random.default_rng(11)
    mats = [dm.Matrix.from_numpy(rng.random((300, 200), dtype=np.float32)) for _ in range(6)]
    hosts = [m.to_numpy() for m in mats]
    rt = dm.runtime.get_runtime()
    for it in range(3):
        a, b, c = mats[it], mats[it + 1], mats[it + 2]
        ha, hb, hc = hosts[it], hosts[it + 1], hosts[it + 2]
        e = 2 * a + b % c - a                                  # a shared leaf
        got = dm.evaluate(e).to_numpy()
        want = O.run_program((("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("load", 2),
                              ("glue", "eglue_schur"), ("glue", "eglue_plus"), ("load", 0), ("glue", "eglue_minus")),
                             [x.reshape(-1, order="F") for x in (ha, hb, hc)], np.float32)
        same(got.reshape(-1, order="F"), want)
        s = dm.accu(2 * a + b)
        assert np.float32(s).tobytes() == np.float32(O.reduce_accu(
            O.run_program((("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("glue", "eglue_plus")),
                          [ha.reshape(-1, order="F"), hb.reshape(-1, order="F")], np.float32))).tobytes()
        x, y, z = dm.evaluate_many(a + b, a + b, c)            # a duplicate and a bare leaf
        same(x.to_numpy(), y.to_numpy())
        same(z.to_numpy(), hc)
        d = dm.Matrix.from_numpy(ha)
        dm.evaluate(d + b, out=d)                              # output aliases an operand
        same(d.to_numpy(), (ha + hb).astype(np.float32))
    assert len(rt._recipes) > 0
    # the same calls without recipes give the same bits
    E._RECIPES_ON = False
    try:
        same(dm.evaluate(2 * mats[0] + mats[1] % mats[2] - mats[0]).to_numpy(),
             dm.evaluate(2 * mats[0] + mats[1] % mats[2] - mats[0]).to_numpy())
    finally:
        E._RECIPES_ON = True


@pytest.mark.parametrize("m,n,k,ta,tb", [(512, 384, 256, 0, 1), (1000, 700, 300, 0, 0), (300, 257, 129, 1, 1),
                                         (2048, 1024, 512, 1, 0)])
def test_gemm_fused_operand_chains_f64(dm, m, n, k, ta, tb, monkeypatch):
    """f64 (2A + 1) @ op(exp(B/4) - 3): the operand programs run in the DMMA
    kernel's register-staged producer -- one launch, bit-identical to
    materialising the operands and running the plain DMMA kernel (same K
    order per accumulator)."""
    rng = np.random.default_rng(m * n + k)
    a = rng.random((k, m) if ta else (m, k))
    b = rng.random((n, k) if tb else (k, n))
    mA, mB = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    ea = 2 * mA + 1
    eb = dm.exp(mB / 4) - 3
    expr = (ea.t() if ta else ea) @ (eb.t() if tb else eb)
    from paper_2308_03120_b200 import expr as E
    monkeypatch.setattr(E, "_F64_PROLOGUE", True)          # off by default (measured slower, bm_gemm_tc.cuh)
    assert [s.kernel for s in dm.plan(expr).steps] == ["gemm_fused"]
    dm.synchronise()
    before = dm.counters()
    got = dm.evaluate(expr).to_numpy()
    assert (dm.counters() - before).launches == 1
    ua, ub = dm.evaluate(ea), dm.evaluate(eb)
    ref_dev = dm.evaluate((ua.t() if ta else ua) @ (ub.t() if tb else ub)).to_numpy()
    same(got, ref_dev)
    oa, ob = ua.to_numpy(), ub.to_numpy()
    normwise(got, (oa.T if ta else oa) @ (ob.T if tb else ob), 1e-12)


def test_plan_recipes_keep_generators_fresh_and_follow_shapes(dm):
    """Recipes never freeze device-generated values (each call draws the next
    counter-RNG stream, like a fresh plan), and a matrix whose shape changes
    between calls gets a new recipe, not a stale one."""
    a = dm.Matrix.from_numpy(np.ones((64, 32), np.float32))
    x1 = dm.evaluate(dm.randu(64, 32) + a).to_numpy()
    x2 = dm.evaluate(dm.randu(64, 32) + a).to_numpy()
    assert not np.array_equal(x1, x2)
    assert np.all((x1 >= 1) & (x1 < 2)) and np.all((x2 >= 1) & (x2 < 2))
    s1 = dm.accu(dm.randn(1000, 1))
    s2 = dm.accu(dm.randn(1000, 1))
    assert s1 != s2
    # the same matrix, reshaped between two evaluations of one expression shape
    m = dm.Matrix.from_numpy(np.arange(12, dtype=np.float32).reshape(3, 4))
    y = dm.evaluate(2 * m).to_numpy()
    same(y, 2 * np.arange(12, dtype=np.float32).reshape(3, 4))
    dm.evaluate(dm.Matrix.from_numpy(np.ones((6, 2), np.float32)), out=m)
    y = dm.evaluate(2 * m).to_numpy()
    assert y.shape == (6, 2)
    same(y, 2 * np.ones((6, 2), np.float32))


def test_plan_recipes_under_threads_and_eviction(dm, monkeypatch):
    """Several user threads evaluating while the recipe cache evicts (a small
    capacity forces it): every result stays right."""
    import threading
    from paper_2308_03120_b200 import expr as E
    monkeypatch.setattr(E, "_RECIPE_MAX", 4)
    errors = []

    def work(tid):
        try:
            rng = np.random.default_rng(tid)
            for it in range(12):
                r, c = 8 + (tid + it) % 7, 3 + it % 5
                a = rng.random((r, c), dtype=np.float32)
                b = rng.random((r, c), dtype=np.float32)
                ma, mb = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
                got = dm.evaluate(2 * ma + mb).to_numpy()
                if got.tobytes() != (np.float32(2) * a + b).astype(np.float32).tobytes():
                    errors.append((tid, it, "evaluate"))
                s = dm.accu(ma % mb)
                want = O.reduce_accu((a * b).reshape(-1, order="F"))
                if np.float32(s).tobytes() != np.float32(want).tobytes():
                    errors.append((tid, it, "accu"))
        except Exception as ex:  # noqa: BLE001
            errors.append((tid, repr(ex)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]


# ---- GEMM epilogue fusion ------------------------------------------------------------------------

@pytest.mark.parametrize("elem,m,n,k,ta,tb", [("f32", 512, 384, 256, 0, 1), ("f32", 1000, 700, 300, 0, 0),
                                              ("f32", 2048, 2048, 1024, 1, 1), ("f32", 256, 256, 20000, 0, 1),
                                              ("f32", 4096, 4352, 600, 0, 1),   # persistent pairs (272 tiles)
                                              ("f64", 300, 200, 100, 1, 0), ("f64", 512, 512, 512, 0, 1),
                                              ("f64", 1030, 770, 64, 0, 0)])
def test_gemm_epilogue_bit_identical_to_unfused(dm, elem, m, n, k, ta, tb):
    """F(op(A) op(B)) with F in the GEMM's store: one launch, and the same
    bits as the reference's plan (the product materialised, then the chain),
    which the unfused device plan reproduces; k = 20000 runs three K passes
    with the epilogue on the last."""
    rng = np.random.default_rng(m + n + k)
    dt = np.float32 if elem == "f32" else np.float64
    a = rng.random((k, m) if ta else (m, k)).astype(dt)
    b = rng.random((n, k) if tb else (k, n)).astype(dt)
    c = rng.random((m, n)).astype(dt)
    mA, mB, mC = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b), dm.Matrix.from_numpy(c)
    prod = (mA.t() if ta else mA) @ (mB.t() if tb else mB)
    e = dm.exp(prod / 64) * 3 - prod % prod / 1000
    assert [s.kernel for s in dm.plan(e).steps] == ["gemm_epi"]
    dm.synchronise()
    before = dm.counters()
    got = dm.evaluate(e).to_numpy()
    assert (dm.counters() - before).launches == 1
    want = dm.evaluate(e, fuse=False).to_numpy()
    same(got, want)
    # and the product itself is the usual GEMM (max-normalised vs f64)
    pa = (a.T if ta else a).astype(np.float64)
    pb = (b.T if tb else b).astype(np.float64)
    normwise(dm.evaluate(prod).to_numpy(), pa @ pb, 1e-5 if elem == "f32" else 1e-12)


@pytest.mark.parametrize("m,n,k,tb", [(1024, 768, 512, 1), (1001, 700, 300, 0), (512, 512, 20000, 1),
                                      (2052, 1030, 256, 1), (1024, 1024, 384, 1)])
def test_gemm_epilogue_with_memory_input(dm, m, n, k, tb, monkeypatch):
    """alpha AB + beta C, exp(AB / k) - C and AB - C^T with C read in the GEMM's
    store (the f32 input staged through the idle TMA ring; m % 4 != 0 makes the
    launcher run the unfused plan instead): the same bits as the reference's plan."""
    from paper_2308_03120_b200 import expr as E
    monkeypatch.setattr(E, "_EPI_MEM_INPUTS", True)
    rng = np.random.default_rng(m * 7 + n + k)
    a = rng.random((m, k)).astype(np.float32)
    b = rng.random((n, k) if tb else (k, n)).astype(np.float32)
    c = rng.random((m, n)).astype(np.float32)
    mA, mB, mC = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b), dm.Matrix.from_numpy(c)
    prod = mA @ (mB.t() if tb else mB)
    exprs = [2 * prod + 3 * mC, dm.exp(prod / k) - mC]
    if m == n:
        exprs.append(prod - mC.t())      # the input a materialised transpose (a slot, not a leaf)
    for e in exprs:
        assert [s.kernel for s in dm.plan(e).steps][-1] == "gemm_epi"
        got = dm.evaluate(e).to_numpy()
        want = dm.evaluate(e, fuse=False).to_numpy()
        same(got, want)


def _random_epilogue(dm, rng, prod, mats, depth):
    """A random element-wise tree over the product and the matrices in `mats`
    (rng: a random.Random)."""
    if depth == 0 or rng.random() < 0.25:
        return prod if (not mats or rng.random() < 0.6) else rng.choice(mats)
    kind = rng.randrange(6)
    a = _random_epilogue(dm, rng, prod, mats, depth - 1)
    if kind == 0:
        return a * rng.choice([0.5, 2.0, -1.5, 3.0])
    if kind == 1:
        return a + rng.choice([1.0, -2.0, 0.25])
    if kind == 2:
        return rng.choice([dm.exp, dm.square, dm.abs])(a / 512.0)
    b = _random_epilogue(dm, rng, prod, mats, depth - 1)
    return {3: lambda: a + b, 4: lambda: a - b, 5: lambda: a % b}[kind]()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gemm_epilogue_random_programs_bit_identical(dm, seed):
    """Random element-wise trees over a tensor-core product and 0-2 more matrices
    (staged, unstaged and declined shapes, odd row counts, several K passes):
    the fused plan gives the bits of the reference's plan every time."""
    import random
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    kinds = []
    for trial in range(8):
        m = rng.choice([256, 384, 516, 601, 1024])
        n = rng.choice([256, 300, 512, 777])
        k = rng.choice([64, 250, 1000, 17000])
        a = dm.Matrix.from_numpy(nrng.random((m, k), dtype=np.float32))
        b = dm.Matrix.from_numpy(nrng.random((n, k), dtype=np.float32))
        mats = [dm.Matrix.from_numpy(nrng.random((m, n), dtype=np.float32)) for _ in range(rng.randrange(3))]
        e = _random_epilogue(dm, rng, a @ b.t(), mats, 3)
        steps = [st.kernel for st in dm.plan(e).steps]
        if not any(kd in ("gemm_epi", "gemm") for kd in steps):
            continue                                  # the tree never reached the product
        kinds.append((steps[-1], len(mats)))
        got = dm.evaluate(e).to_numpy()
        want = dm.evaluate(e, fuse=False).to_numpy()
        same_nan(got, want)
    assert any(kd == "gemm_epi" for kd, _ in kinds), kinds


@pytest.mark.parametrize("seed", [4, 5])
def test_gemm_prologue_random_programs_bit_identical(dm, seed):
    """Random element-wise operand programs on both sides of a tensor-core product
    (evaluated inside the 3xTF32 split pass, no operand materialised): the bits
    of the reference's plan, which materialises the operands first."""
    import random
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    fused = 0
    for trial in range(6):
        m, n, k = rng.choice([256, 520, 777]), rng.choice([256, 384, 600]), rng.choice([128, 300, 2000])
        a = dm.Matrix.from_numpy(nrng.random((m, k), dtype=np.float32))
        b = dm.Matrix.from_numpy(nrng.random((n, k), dtype=np.float32))
        am = [dm.Matrix.from_numpy(nrng.random((m, k), dtype=np.float32)) for _ in range(rng.randrange(2))]
        bm = [dm.Matrix.from_numpy(nrng.random((n, k), dtype=np.float32)) for _ in range(rng.randrange(2))]
        e = _random_epilogue(dm, rng, a, am, 2) @ _random_epilogue(dm, rng, b, bm, 2).t()
        fused += "gemm_fused" in [st.kernel for st in dm.plan(e).steps]
        got = dm.evaluate(e).to_numpy()
        want = dm.evaluate(e, fuse=False).to_numpy()
        same_nan(got, want)
    assert fused > 0


def test_pair_gemm_repeatable_under_load(dm):
    """The pair kernel's stage / accumulator barriers are CTA-scope (no cluster-wide
    fence per chunk): any ordering hole between the MMA issuer, the TMA threads and
    the epilogue warps of the two CTAs would show up as run-to-run differences.  40
    back-to-back products (plain, fused exp, staged memory-input epilogue) at 4096^3
    with K = 5120 (two 64-K-chunk accumulators ping-ponging 80 times per tile) must
    repeat bit for bit, and match f64 normwise."""
    rng = np.random.default_rng(77)
    n, k = 4096, 5120
    a = rng.random((n, k), dtype=np.float32)
    b = rng.random((n, k), dtype=np.float32)
    c = rng.random((n, n), dtype=np.float32)
    mA, mB, mC = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b), dm.Matrix.from_numpy(c)
    prod = mA @ mB.t()
    exprs = (prod, dm.exp(prod / k), 2 * prod + 3 * mC)
    assert [s.kernel for s in dm.plan(exprs[2]).steps] == ["gemm_epi"]
    firsts = [dm.evaluate(e).to_numpy() for e in exprs]
    for i in range(40):
        e = exprs[i % 3]
        got = dm.evaluate(e).to_numpy()
        assert got.tobytes() == firsts[i % 3].tobytes(), f"run {i} of expression {i % 3} differs"
    import torch
    ta, tb = torch.from_numpy(a).cuda().double(), torch.from_numpy(b).cuda().double()
    normwise(firsts[0], (ta @ tb.t()).cpu().numpy(), 1e-5)


def test_torch_view_keeps_its_matrix_alive(dm):
    """dist.torch_view of a temporary: the tensor holds the matrix, so its buffer
    is not released (and reused by the next evaluation) under the view."""
    import gc
    import weakref
    import torch
    from paper_2308_03120_b200 import dist as D
    a = dm.Matrix.from_numpy(np.arange(1 << 16, dtype=np.float32))
    tmp = dm.evaluate(2 * a)
    alive = weakref.ref(tmp)
    v = D.torch_view(tmp)
    del tmp
    gc.collect()
    assert alive() is not None
    others = [dm.evaluate(5 * a + k) for k in range(4)]     # would reuse a released buffer
    dm.synchronise()
    assert torch.equal(v.cpu(), torch.arange(1 << 16, dtype=torch.float32) * 2)
    del v, others
    gc.collect()
    assert alive() is None


_PERSIST_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2308_03120_b200 as dm
dm.init("b200")
rng = np.random.default_rng(11)
outs = []
for m, n, k in ((4096, 4000, 2048), (2304, 5000, 700), (8192, 256, 1030)):
    a = dm.Matrix.from_numpy(rng.random((m, k), dtype=np.float32))
    b = dm.Matrix.from_numpy(rng.random((n, k), dtype=np.float32))
    prod = a @ b.t()
    outs.append(dm.evaluate(prod).to_numpy().reshape(-1))
    outs.append(dm.evaluate(dm.exp(prod / k) * 3 - 1).to_numpy().reshape(-1))
np.save(sys.argv[2], np.concatenate(outs))
dm.shutdown()
"""


def test_gemm_persistent_pairs_bit_identical(tmp_path):
    """BM_GEMM_PERSIST=1 (the default): 74 resident CTA pairs claim the 256 x 256
    tiles from a global counter (several K passes here, each with its own
    counter) -- the same bits as one pair per tile, for the plain GEMM and a
    fused epilogue, at shapes with many tiles, ragged tiles and one tile column."""
    import os
    import pathlib
    import subprocess
    import sys
    root = str(pathlib.Path(__file__).resolve().parents[1])
    outs = {}
    for p in ("0", "1"):
        env = dict(os.environ, BM_GEMM_PERSIST=p, BM_GEMM_KPASS="512")
        f = tmp_path / f"p{p}.npy"
        subprocess.run([sys.executable, "-c", _PERSIST_CHILD, root, str(f)], env=env, check=True, timeout=600)
        outs[p] = np.load(f)
    same(outs["1"], outs["0"])


# ---- GEMM prologue fusion ------------------------------------------------------------------------

@pytest.mark.parametrize("m,n,k,tb", [(512, 384, 256, 1), (1000, 700, 300, 0), (2048, 2048, 1024, 1),
                                      (4096, 4352, 512, 1)])   # the last: persistent pairs (272 tiles)
def test_gemm_fused_operand_chains(dm, m, n, k, tb):
    """(2A + 1) @ op(exp(B/4) - 3) with the operand programs inside the split
    pre-pass: same numbers as materialising the operands first."""
    rng = np.random.default_rng(m + n + k)
    a = rng.random((m, k), dtype=np.float32)
    b = rng.random((n, k) if tb else (k, n), dtype=np.float32)
    mA, mB = dm.Matrix.from_numpy(a), dm.Matrix.from_numpy(b)
    eb = dm.exp(mB / 4) - 3
    expr = (2 * mA + 1) @ (eb.t() if tb else eb)
    assert [s.kernel for s in dm.plan(expr).steps] == ["gemm_fused"]
    dm.synchronise()
    before = dm.counters()
    got = dm.evaluate(expr).to_numpy()
    assert (dm.counters() - before).launches == 1
    # unfused device path and an f64 host reference of the same operand values
    ua = dm.evaluate(2 * mA + 1)
    ub = dm.evaluate(eb)
    ref_dev = dm.evaluate(ua @ (ub.t() if tb else ub)).to_numpy()
    oa = ua.to_numpy().astype(np.float64)
    ob = ub.to_numpy().astype(np.float64)
    ref = oa @ (ob.T if tb else ob)
    normwise(got, ref, 1e-5)
    same(got, ref_dev)          # identical operand values and the same 3xTF32 kernel: bit-identical
