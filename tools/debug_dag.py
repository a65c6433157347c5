"""Find the first sub-expression whose GPU value departs from the oracle
(random-DAG debugging on the GPU box)."""
import pathlib
import random
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle as O  # noqa: E402
from dag_gen import gen  # noqa: E402


def err(dm, node):
    want = O.tree_walk(node, lambda m: m.to_numpy())
    got = dm.evaluate(node).to_numpy()
    if node.elem_type in ("i32", "u64"):
        return 0.0 if np.array_equal(got, want) else 1.0
    e = float(np.max(np.abs(got.astype(np.float64) - want.astype(np.float64)))) if got.size else 0.0
    return e / max(float(np.max(np.abs(want))) if want.size else 0.0, 1.0)


def walk(dm, node, depth=0):
    bad = []
    if node.kind != "leaf":
        for c in node.operands:
            bad += walk(dm, c, depth + 1)
    tol = 1e-5 if node.elem_type == "f32" else 1e-12
    e = err(dm, node)
    if e > tol and not bad:
        print("  " * depth, "FIRST BAD:", node.kind, node.elem_type, dm.shape_of(node), node.aux, "err", e,
              "children:", [(c.kind, c.elem_type) for c in node.operands if hasattr(c, "kind")])
        p = dm.plan(node)
        for s in p.steps:
            print("    step", s.kernel, s.params, [(r[0], getattr(r[1], "elem_type", r[1])) for r in s.inputs])
        return [node]
    return bad


def main():
    import paper_2308_03120_b200 as dm
    dm.init("b200")
    elem = sys.argv[1] if len(sys.argv) > 1 else "f64"
    rng = random.Random({"f32": 1, "f64": 2, "i32": 3}[elem])
    for i in range(40):
        node = gen(dm, rng, 4, rng.randrange(1, 9), rng.randrange(1, 9), elem)
        e = err(dm, node)
        tol = 1e-5 if elem == "f32" else 1e-12
        if elem != "i32" and e > tol or elem == "i32" and e:
            print("DAG", i, "err", e)
            walk(dm, node)
    dm.shutdown()


if __name__ == "__main__":
    main()
