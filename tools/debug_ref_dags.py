"""Random DAGs of the REFERENCE's generator (baseline/_ref_tests/dag_util.py,
staged by tools/stage_reference_suite.py) through this package: print the first
sub-expression whose device value departs from the oracle, with its plan."""
import pathlib
import random
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
for p in (ROOT / "tests" / "dropin", ROOT, ROOT / "baseline" / "_ref_tests", ROOT / "tools"):
    sys.path.insert(0, str(p))

import devmat as dm  # noqa: E402  (the alias of this package)
from dag_util import gen_dag  # noqa: E402
from debug_dag import err, walk  # noqa: E402


def main():
    dm.init("reference")
    elem = sys.argv[1] if len(sys.argv) > 1 else "f64"
    rng = random.Random({"f32": 1, "f64": 2, "i32": 3}[elem])
    for i in range(60):
        node = gen_dag(rng, 4, rng.randrange(1, 9), rng.randrange(1, 9), elem)
        e = err(dm, node)
        if e > (1e-5 if elem == "f32" else 1e-12):
            print("DAG", i, "err", e, flush=True)
            walk(dm, node)
    dm.shutdown()


if __name__ == "__main__":
    main()
