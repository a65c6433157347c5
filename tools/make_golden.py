"""Generate tests/golden/*.npz by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tools/make_golden.py

It imports `devmat` from /root/reference/pkg/src, evaluates the hot-path
operations of SURVEY.md section 8 on seeded inputs with the reference's own
public API (backend "reference"), and stores inputs and outputs.  The
fixtures pin tests/test_oracle.py (oracle == reference) and are the
reference-side expectations of the GPU parity tests.  Nothing on the GPU box
reads /root/reference.
"""
from __future__ import annotations

import os
import pathlib
import sys
import tempfile

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parents[1] / "tests" / "golden"


def main() -> None:
    os.environ["KERNEL_CACHE_DIR"] = tempfile.mkdtemp(prefix="devmat-cache-")
    sys.path.insert(0, str(REF))
    import devmat as dm  # noqa: E402

    dm.init("reference")
    OUT.mkdir(parents=True, exist_ok=True)
    M = dm.Matrix.from_numpy

    def ev(node):
        return dm.evaluate(node).to_numpy()

    # ---- 1. fused element-wise chains and the config-1 expression -------------------------
    g = {}
    rng = np.random.default_rng(0)
    for tag, (r, c) in {"a": (64, 48), "b": (1000, 37), "c": (4096, 4)}.items():
        A, B, C, D = (rng.random((r, c), dtype=np.float32) for _ in range(4))
        mA, mB, mC, mD = M(A), M(B), M(C), M(D)
        g[f"{tag}_A"], g[f"{tag}_B"], g[f"{tag}_C"], g[f"{tag}_D"] = A, B, C, D
        g[f"{tag}_chain_exp"] = ev(2 * mA + mB * mC - dm.exp(mD))
        g[f"{tag}_chain_noexp"] = ev(2 * mA + mB * mC - mD)
        g[f"{tag}_accu_exp"] = np.array(dm.accu(2 * mA + mB * mC - dm.exp(mD)), dtype=np.float32)
        g[f"{tag}_accu_noexp"] = np.array(dm.accu(2 * mA + mB * mC - mD), dtype=np.float32)
        g[f"{tag}_deep"] = ev(dm.sqrt(dm.absolute(mA - 0.5) + 1.0) / (mB + 1) * 3 - mC * mD + 0.25)
    np.savez_compressed(OUT / "chains.npz", **g)

    # ---- 2. unary / scalar / glue ops per element type -----------------------------------------
    g = {}
    rng = np.random.default_rng(1)
    xf = (0.05 + 0.9 * rng.random((33, 17))).astype(np.float32)
    xd = 0.05 + 0.9 * rng.random((33, 17))
    g["xf"], g["xd"] = xf, xd
    for name in ("exp", "log", "log10", "sqrt", "square", "abs", "cos", "sin", "tan", "acos", "asin", "atan"):
        fn = getattr(dm, "absolute" if name == "abs" else name)
        g[f"f32_{name}"] = ev(fn(M(xf)))
        g[f"f64_{name}"] = ev(fn(M(xd)))
    g["f32_pow3"] = ev(dm.power(M(xf), 3))
    g["f64_pow2_5"] = ev(dm.power(M(xd), 2.5))
    xi = rng.integers(-1000, 1000, (29, 11)).astype(np.int32)
    yi = rng.integers(-50, 50, (29, 11)).astype(np.int32)
    g["xi"], g["yi"] = xi, yi
    mi, mj = M(xi), M(yi)
    g["i32_chain"] = ev(mi * mi + 3 - mj * 7)
    g["i32_div_scalar"] = ev(mi / 7)
    g["i32_div_pre"] = ev(1000 / (mj * mj + 1))
    g["i32_div_glue"] = ev(mi / mj)              # includes division by zero
    g["i32_square"] = ev(dm.square(mi * 1000))   # wraps
    g["i32_abs"] = ev(dm.absolute(mj))
    g["i32_pow"] = ev(dm.power(mj, 3))
    g["i32_sqrt"] = ev(dm.sqrt(dm.absolute(mi)))
    xu = rng.integers(0, 1 << 40, (13, 9), dtype=np.uint64)
    g["xu"] = xu
    mu = M(xu)
    g["u64_chain"] = ev(mu * 3 + 7 - mu / 5)
    g["u64_minus_pre"] = ev(5 - mu)              # wraps
    g["u64_div0"] = ev(mu / dm.evaluate(mu * 0))
    np.savez_compressed(OUT / "ops.npz", **g)

    # ---- 3. conversions -------------------------------------------------------------------------
    g = {}
    edge = np.array([[np.nan, np.inf, -np.inf, 3e9, -3e9, -1.5, 2.7, 1e20, -1e20, 2.0 ** 63, 2.0 ** 64,
                      -0.0, 2147483647.9, -2147483648.5, 0.5]])
    g["edge_f64"] = edge
    me = M(edge)
    for t in ("i32", "u64", "f32"):
        g[f"edge_to_{t}"] = dm.evaluate(dm.conv_to(me, t), fuse=False).to_numpy()
    mf = M(edge.astype(np.float32))
    g["edge_f32"] = edge.astype(np.float32)
    for t in ("i32", "u64", "f64"):
        g[f"edge_f32_to_{t}"] = dm.evaluate(dm.conv_to(mf, t), fuse=False).to_numpy()
    iv = np.array([[-7, 7, -2147483648, 2147483647, 0, 123456789]], dtype=np.int32)
    g["iv"] = iv
    for t in ("f32", "f64", "u64"):
        g[f"iv_to_{t}"] = dm.evaluate(dm.conv_to(M(iv), t), fuse=False).to_numpy()
    uv = np.array([[0, 1, 2 ** 53 + 1, 2 ** 63 + 12345, 2 ** 64 - 1]], dtype=np.uint64)
    g["uv"] = uv
    for t in ("f32", "f64", "i32"):
        g[f"uv_to_{t}"] = dm.evaluate(dm.conv_to(M(uv), t), fuse=False).to_numpy()
    np.savez_compressed(OUT / "casts.npz", **g)

    # ---- 4. scalar reductions -------------------------------------------------------------------
    g = {}
    rng = np.random.default_rng(2)
    sizes = [1, 7, 8, 100, 128, 129, 1000, 2048, 8191, 8192, 8193, 3 * 8192 + 41, 65536 + 999, 100000]
    for n in sizes:
        for dt in ("f32", "f64"):
            v = (rng.standard_normal(n) * np.exp2(rng.integers(-12, 12, n))).astype(dt.replace("f", "float")
                                                                                    .replace("float32", "float32"))
            v = v.astype(np.float32 if dt == "f32" else np.float64)
            w = rng.random(n).astype(v.dtype)
            mv, mw = M(v.reshape(-1, 1)), M(w.reshape(-1, 1))
            g[f"{dt}_{n}_x"], g[f"{dt}_{n}_y"] = v, w
            g[f"{dt}_{n}_accu"] = np.array(dm.accu(mv), dtype=v.dtype)
            g[f"{dt}_{n}_dot"] = np.array(dm.dot(mv, mw), dtype=v.dtype)
            g[f"{dt}_{n}_norm2"] = np.array(dm.norm(mv, 2))
            g[f"{dt}_{n}_norminf"] = np.array(dm.norm(mv, "inf"))
            g[f"{dt}_{n}_normm"] = np.array(dm.norm(mv, "-inf"))
            g[f"{dt}_{n}_norm3"] = np.array(dm.norm(mv, 3))
    xi = rng.integers(-(1 << 30), 1 << 30, 20000).astype(np.int32)
    g["i32_x"] = xi
    g["i32_accu"] = np.array(dm.accu(M(xi.reshape(-1, 1))), dtype=np.int64)
    xu = rng.integers(0, 1 << 62, 20000, dtype=np.uint64)
    g["u64_x"] = xu
    g["u64_accu"] = np.array(dm.accu(M(xu.reshape(-1, 1))), dtype=np.uint64)
    # min/max with NaNs at chosen block positions (order-dependent combine)
    from devmat import runtime as rtm
    from devmat.runtime import FlatView, KernelInvocation
    rt = rtm.get_runtime()
    for case, pos in {"nan_first": [5], "nan_second_block": [8192 + 3], "nan_two": [10, 3 * 8192]}.items():
        v = rng.random(4 * 8192 + 7).astype(np.float32)
        v[pos] = np.nan
        mv = M(v.reshape(-1, 1))
        g[f"mm_{case}_x"] = v
        for kind in ("reduce_min", "reduce_max"):
            val = rt.execute_reduce(KernelInvocation(kind, (FlatView(mv.mem, 0, mv.n_elem),), None))
            g[f"mm_{case}_{kind}"] = np.array(val, dtype=np.float32)
    np.savez_compressed(OUT / "reduce.npz", **g)

    # ---- 5. per-dimension reductions ---------------------------------------------------------------
    g = {}
    rng = np.random.default_rng(3)
    shapes = [(37, 53), (300, 7), (64, 300), (1, 9), (9, 1), (2048, 5)]
    for (r, c) in shapes:
        for dt in ("f32", "f64", "i32"):
            if dt == "i32":
                a = rng.integers(-100, 100, (r, c)).astype(np.int32)
            else:
                a = (rng.standard_normal((r, c)) * 10).astype(np.float32 if dt == "f32" else np.float64)
            key = f"{dt}_{r}x{c}"
            g[key] = a
            ma = M(a)
            for op in ("sum", "min", "max", "mean", "var", "stddev"):
                if dt == "i32" and op in ("var", "stddev"):
                    continue
                for dim in (0, 1):
                    g[f"{key}_{op}{dim}"] = ev(getattr(dm, op)(ma, dim))
    np.savez_compressed(OUT / "rdim.npz", **g)

    # ---- 6. gemm --------------------------------------------------------------------------------------
    g = {}
    rng = np.random.default_rng(4)
    for dt in ("f32", "f64"):
        npdt = np.float32 if dt == "f32" else np.float64
        a = rng.random((96, 80)).astype(npdt)
        b = rng.random((80, 112)).astype(npdt)
        bt = rng.random((112, 80)).astype(npdt)
        g[f"{dt}_a"], g[f"{dt}_b"], g[f"{dt}_bt"] = a, b, bt
        g[f"{dt}_ab"] = dm.gemm(M(a), M(b)).to_numpy()
        g[f"{dt}_abt"] = ev(M(a) @ M(bt).t())
        g[f"{dt}_atb"] = ev(M(np.ascontiguousarray(a.T)).t() @ M(b))
    ai = np.array([[1, 2], [3, 4]], dtype=np.int32)
    g["i32_a"] = ai
    g["i32_aa"] = dm.gemm(M(ai), M(ai)).to_numpy()
    g["f32_inner0"] = dm.evaluate(dm.Matrix(3, 0) @ dm.Matrix(0, 4)).to_numpy()
    np.savez_compressed(OUT / "gemm.npz", **g)

    # ---- 7. norms of matrices, RNG pins, logistic step --------------------------------------------------
    g = {}
    rng = np.random.default_rng(5)
    x = np.array([[1.0, -2.0], [3.0, 4.0]], dtype=np.float32)
    g["mx"] = x
    for kind in ("fro", "inf", "-inf"):
        g[f"mx_norm_{kind}"] = np.array(dm.norm(M(x), kind))
    big = (rng.standard_normal((50, 70))).astype(np.float64)
    g["big"] = big
    for kind in ("fro", "inf", "-inf"):
        g[f"big_norm_{kind}"] = np.array(dm.norm(M(big), kind))
    for seed, elem in ((123, "f32"), (777, "f64")):
        dm.set_seed(seed)
        g[f"randu_{seed}"] = dm.Matrix(40, 25, fill="randu", elem_type=elem).to_numpy()
        g[f"randn_{seed}"] = dm.Matrix(33, 17, fill="randn", elem_type=elem).to_numpy()
    X = rng.standard_normal((512, 16), dtype=np.float32)
    w = (0.03 * rng.standard_normal((16, 1))).astype(np.float32)
    y = (rng.random((512, 1)) < 0.5).astype(np.float32)
    mX, mw, my = M(X), M(w), M(y)
    z = dm.evaluate(mX @ mw)
    r = dm.evaluate(1 / (1 + dm.exp(0 - z)) - my)
    gr = dm.evaluate(mX.t() @ r)
    g["lr_X"], g["lr_w"], g["lr_y"] = X, w, y
    g["lr_r"], g["lr_g"] = r.to_numpy(), gr.to_numpy()
    g["lr_s"] = np.array(dm.accu(r), dtype=np.float32)
    np.savez_compressed(OUT / "misc.npz", **g)

    # ---- 8. predicates: find / all / any (ops.py:202-262) ------------------------------------------
    g = {}
    rng = np.random.default_rng(8)
    mats = {
        "f32": rng.random((97, 61), dtype=np.float32),
        "f64": rng.standard_normal((70, 40)),
        "i32": rng.integers(-5, 6, (50, 33)).astype(np.int32),
        "u64": rng.integers(0, 9, (45, 21)).astype(np.uint64),
    }
    mats["f32"][rng.random((97, 61)) < 0.03] = np.nan
    mats["f64"][rng.random((70, 40)) < 0.03] = np.nan
    for elem, a in mats.items():
        g[f"{elem}_x"] = a
        m = M(a)
        for name, op in (("gt", ">"), ("lt", "<"), ("ge", ">="), ("le", "<=")):
            for ti, thr in enumerate((0.5, 2, -0.25)):
                rel = {">": m > thr, "<": m < thr, ">=": m >= thr, "<=": m <= thr}[op]
                g[f"{elem}_find_{name}_{ti}"] = dm.find(rel).to_numpy().reshape(-1)
                g[f"{elem}_all_{name}_{ti}"] = np.array(dm.all(rel))
                g[f"{elem}_any_{name}_{ti}"] = np.array(dm.any(rel))
        g[f"{elem}_find_nonzero"] = dm.find(m).to_numpy().reshape(-1)
        g[f"{elem}_all_nonzero"] = np.array(dm.all(m))
        g[f"{elem}_any_nonzero"] = np.array(dm.any(m))
    g["eye_find"] = dm.find(dm.Matrix(3, 3, fill="eye")).to_numpy().reshape(-1)
    g["expr_find"] = dm.find(M(mats["f32"]) * 2 - 1 > 0.25).to_numpy().reshape(-1)
    np.savez_compressed(OUT / "pred.npz", **g)
    dm.shutdown()
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
