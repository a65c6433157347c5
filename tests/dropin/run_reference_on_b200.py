"""The UNMODIFIED reference package (baseline/_ref/devmat) with the B200 device
behind its firewall (tests/dropin/b200_device.py): the reference's own
expression layer, planner and Runtime drive libb200mat.so.  Checks the hot
path against the golden outputs of the reference's CPU backend and prints a
JSON summary on the last line (run by tests/test_device_plugin.py in its own
process, so ``devmat`` here is the reference, not the alias)."""
import json
import os
import pathlib
import sys
import tempfile

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))
os.environ["KERNEL_CACHE_DIR"] = tempfile.mkdtemp(prefix="devmat-ref-cache-")

import devmat as dm  # noqa: E402  (the unmodified reference)

sys.path.insert(0, str(ROOT / "tests" / "dropin"))
import b200_device  # noqa: E402

from tools.baseline_inputs import cfg1_inputs  # noqa: E402

assert pathlib.Path(dm.__file__).resolve().is_relative_to((ROOT / "baseline" / "_ref").resolve()), dm.__file__


def golden(name):
    with np.load(ROOT / "tests" / "golden" / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def rel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1.0))


def main():
    b200_device.install(dm)
    dm.init("reference")
    rt = dm.runtime.get_runtime()
    assert type(rt._device).__name__ == "B200Device", type(rt._device)
    M = dm.Matrix.from_numpy
    res = {"checks": 0, "bit_exact": 0, "failures": []}

    def check(name, ok):
        res["checks"] += 1
        if not ok:
            res["failures"].append(name)

    def same(name, got, want):
        ok = np.asarray(got).tobytes() == np.asarray(want).tobytes()
        res["bit_exact"] += ok
        check(name, ok)

    g = golden("chains")
    for t in "abc":
        A, B, C, D = (M(g[f"{t}_{x}"]) for x in "ABCD")
        same(f"chain_noexp_{t}", dm.evaluate(2 * A + B * C - D).to_numpy(), g[f"{t}_chain_noexp"])
        same(f"accu_noexp_{t}", np.float32(dm.accu(2 * A + B * C - D)), g[f"{t}_accu_noexp"])
        check(f"chain_exp_{t}", rel(dm.evaluate(2 * A + B * C - dm.exp(D)).to_numpy(), g[f"{t}_chain_exp"]) <= 1e-6)
        check(f"accu_exp_{t}", rel(dm.accu(2 * A + B * C - dm.exp(D)), g[f"{t}_accu_exp"]) <= 1e-5)
        same(f"deep_{t}", dm.evaluate(dm.sqrt(dm.absolute(A - 0.5) + 1.0) / (B + 1) * 3 - C * D + 0.25).to_numpy(),
             g[f"{t}_deep"])

    g = golden("reduce")
    for dt in ("f32", "f64"):
        for n in (1, 7, 8, 128, 129, 2048, 8191, 8192, 8193, 24617, 66535, 100000):
            x, y = M(g[f"{dt}_{n}_x"].reshape(-1, 1)), M(g[f"{dt}_{n}_y"].reshape(-1, 1))
            same(f"accu_{dt}_{n}", np.asarray(dm.accu(x)).astype(g[f"{dt}_{n}_accu"].dtype), g[f"{dt}_{n}_accu"])
            tol = 1e-5 if dt == "f32" else 1e-12
            check(f"dot_{dt}_{n}", rel(dm.dot(x, y), g[f"{dt}_{n}_dot"]) <= tol)
            check(f"norm2_{dt}_{n}", rel(dm.norm(x, 2), g[f"{dt}_{n}_norm2"]) <= tol)
            same(f"norminf_{dt}_{n}", np.float64(dm.norm(x, "inf")), np.float64(g[f"{dt}_{n}_norminf"]))

    g = golden("rdim")
    shapes = sorted({k.rsplit("_", 1)[0] for k in g if k.count("_") == 2})
    for key in shapes:
        X = M(g[key])
        for op in ("sum", "min", "max", "mean"):
            for dim in (0, 1):
                same(f"{op}{dim}_{key}", dm.evaluate(getattr(dm, op)(X, dim)).to_numpy(), g[f"{key}_{op}{dim}"])

    g = golden("gemm")
    for dt in ("f32", "f64"):
        a, b, bt = M(g[f"{dt}_a"]), M(g[f"{dt}_b"]), M(g[f"{dt}_bt"])
        tol = 1e-5 if dt == "f32" else 1e-12
        check(f"gemm_ab_{dt}", rel(dm.evaluate(a @ b).to_numpy(), g[f"{dt}_ab"]) <= tol)
        check(f"gemm_abt_{dt}", rel(dm.evaluate(a @ bt.t()).to_numpy(), g[f"{dt}_abt"]) <= tol)

    # config 1 at its BASELINE shape through the reference's own planner
    # (fused_chain + reduce_accu: two launches on the B200)
    A, B, C, D = (M(x) for x in cfg1_inputs())
    before = rt.counters_snapshot()
    v = np.float32(dm.accu(2 * A + B * C - dm.exp(D)))
    launches = (rt.counters_snapshot() - before).launches
    gb = golden("baseline")
    check("cfg1_4096", rel(v, gb["cfg1_accu_exp"]) <= 1e-5)
    same("cfg1_4096_noexp", np.float32(dm.accu(2 * A + B * C - D)), gb["cfg1_accu_noexp"])
    res["cfg1_value"] = float(v)
    res["cfg1_reference_launches"] = int(launches)
    dm.synchronise()
    dm.shutdown()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
