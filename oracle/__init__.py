"""CPU oracle for the B200 hot path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's algorithms for the hot path
(reference/pkg/src/devmat/kernels.py, expr.py, ops.py, linalg.py), used as
the checker by tests/, by __graft_entry__.smoke() and by bench.py's
cpu_baseline leg.  The product package never imports this module.

Pinning: tests/test_oracle.py checks every function here against golden
vectors produced by running the unmodified reference package
(tools/make_golden.py -> tests/golden/*.npz).
"""
from .devmat_oracle import *  # noqa: F401,F403
