"""Matrix product and scalar-valued linear algebra on the B200 path.

``gemm``/``gemv`` and ``norm`` follow reference/pkg/src/devmat/linalg.py
(:111-117, :486-529).  ``norm`` never materialises its argument: the 2- and
Frobenius norms are one fused dot kernel over a single read of the data
(``sqrt`` of the element-type dot, in f64 on the host, exactly like
linalg.py:88-94), the inf/-inf vector norms are one fused abs+max/min kernel,
and p-norms are one fused abs+pow+accu kernel.
"""
from __future__ import annotations

import math

from . import expr as _expr
from . import ops as _ops
from . import runtime as _rt
from .errors import DimensionError, ElemTypeError
from .expr import as_expr, evaluate, shape_of
from .matrix import Matrix


def gemm(a, b) -> Matrix:
    """C = A @ B (tcgen05 3xTF32 for f32, DMMA for f64, exact for integers);
    transposed operands fold into the kernel (``gemm(A, B.t())`` is NT)."""
    return evaluate(as_expr(a) @ as_expr(b))


def gemv(a, x) -> Matrix:
    return gemm(a, x)


def _require_float(node, op: str) -> None:
    if node.elem_type not in ("f32", "f64"):
        raise ElemTypeError(f"{op} requires a float matrix, got {node.elem_type}")


def _fro(node) -> float:
    return math.sqrt(float(_expr.reduce_value("dot", node, node)))


def norm(x, kind=2) -> float:
    """Vector p-norms (p >= 1, "inf", "-inf", "fro") and matrix "fro"/"inf"/"-inf"."""
    node = as_expr(x)
    _require_float(node, "norm")
    s = shape_of(node)
    if s.n_elem == 0:
        return 0.0
    if s.rows == 1 or s.cols == 1:
        if kind == "fro" or kind == 2:
            return _fro(node)
        if kind in ("inf", "-inf"):
            return float(_expr.reduce_value("max" if kind == "inf" else "min", _ops.absolute(node)))
        if isinstance(kind, int) and kind >= 1:
            total = _expr.reduce_value("accu", _ops.power(_ops.absolute(node), kind))
            return float(total) ** (1.0 / kind)
        raise ValueError(f"bad vector norm kind {kind!r}")
    if kind == "fro":
        return _fro(node)
    if kind in ("inf", "-inf"):
        sums = evaluate(_ops.sum(_ops.absolute(node), dim=1))
        try:
            return float(_expr.reduce_value("max" if kind == "inf" else "min", sums))
        finally:
            sums._release_storage()
    raise ValueError(f"matrix norm kind {kind!r} not supported (use 'fro', 'inf', '-inf')")


def as_scalar(x):
    """Evaluate a 1x1 expression and return its element."""
    node = as_expr(x)
    s = shape_of(node)
    if (s.rows, s.cols) != (1, 1):
        raise DimensionError("as_scalar", (s.rows, s.cols))
    m = evaluate(node) if node.kind != "leaf" else node.operands[0]
    return _rt.get_runtime().read_scalar(m.mem, 0).item()


def trace(a) -> float:
    """Sum of the diagonal of a square matrix (one fused accu over the
    strided diagonal view)."""
    node = as_expr(a)
    s = shape_of(node)
    if s.rows != s.cols:
        raise DimensionError("trace", (s.rows, s.cols))
    if s.rows == 0:
        return 0
    m = node.operands[0] if node.kind == "leaf" else evaluate(node)
    return _ops.accu(m.diag(0))
