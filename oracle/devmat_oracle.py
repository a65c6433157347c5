"""Numpy restatement of the reference's hot-path algorithms (test oracle).

Each function cites the reference file:line it restates.  Everything is plain
numpy so the oracle runs anywhere the tests run; nothing here is imported by
the product package.
"""
from __future__ import annotations

import math

import numpy as np

# kernels.py:28-35
NP_DTYPE = {"f32": np.dtype(np.float32), "f64": np.dtype(np.float64), "i32": np.dtype(np.int32),
            "u64": np.dtype(np.uint64)}
ELEM_BLOCK = 1 << 16          # kernels.py:86
REDUCE_BLOCK = 1 << 13        # kernels.py:87
GEMM_PANEL = 64               # kernels.py:88
DIM_BLOCK = 64                # kernels.py:89

__all__ = ["NP_DTYPE", "REDUCE_BLOCK", "ELEM_BLOCK", "GEMM_PANEL", "cast_out", "stage_cast", "scalar_of",
           "int_div", "apply_unary", "apply_scalar", "apply_glue", "run_program", "combine_pairwise",
           "block_ranges", "reduce_accu", "reduce_min", "reduce_max", "reduce_dot", "numpy_pairwise_sum",
           "rdim", "gemm", "norm_vector", "norm_matrix", "uniform_stream", "normal_stream",
           "logistic_step", "tree_walk", "py_min", "py_max", "predicate_mask", "find_indices"]


# ---------------------------------------------------------------------------
# element-wise semantics (kernels.py:259-377)

def cast_out(values: np.ndarray, out_dtype) -> np.ndarray:
    """Write-time C-cast of a two-way kernel (kernels.py:259-267)."""
    out_dtype = np.dtype(out_dtype)
    if values.dtype == out_dtype:
        return values
    with np.errstate(invalid="ignore", over="ignore"):
        return values.astype(out_dtype)


def stage_cast(values: np.ndarray, dtype) -> np.ndarray:
    """Round every stage to the compute dtype (kernels.py:270-277)."""
    return cast_out(np.asarray(values), dtype)


def scalar_of(k, dtype):
    """Scalar argument in the compute dtype (kernels.py:280-283)."""
    dtype = np.dtype(dtype)
    return dtype.type(int(k)) if dtype.kind in "iu" else dtype.type(k)


def int_div(a, b, dtype):
    """i32: truncate through f64; u64: floor_divide (kernels.py:286-292)."""
    dtype = np.dtype(dtype)
    if dtype.kind == "u":
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.floor_divide(a, b)
    with np.errstate(divide="ignore", invalid="ignore"):
        return (np.asarray(a, dtype=np.float64) / np.asarray(b, dtype=np.float64)).astype(dtype)


_UNARY = {"eop_exp": np.exp, "eop_log": np.log, "eop_log10": np.log10, "eop_sqrt": np.sqrt,
          "eop_square": lambda x: x * x, "eop_abs": np.abs, "eop_cos": np.cos, "eop_sin": np.sin,
          "eop_tan": np.tan, "eop_acos": np.arccos, "eop_asin": np.arcsin, "eop_atan": np.arctan}


def apply_unary(op, x, k, dtype):
    """kernels.py:311-316"""
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        if op == "eop_pow":
            return stage_cast(np.power(x, scalar_of(k, dtype)), dtype)
        return stage_cast(_UNARY[op](x), dtype)


def apply_scalar(op, x, k, dtype):
    """kernels.py:319-336"""
    dtype = np.dtype(dtype)
    kv = scalar_of(k, dtype)
    isint = dtype.kind in "iu"
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        r = {"eop_scalar_plus": lambda: x + kv,
             "eop_scalar_minus_pre": lambda: kv - x,
             "eop_scalar_minus_post": lambda: x - kv,
             "eop_scalar_times": lambda: x * kv,
             "eop_scalar_div_pre": lambda: int_div(kv, x, dtype) if isint else kv / x,
             "eop_scalar_div_post": lambda: int_div(x, kv, dtype) if isint else x / kv}[op]()
    return stage_cast(r, dtype)


def apply_glue(op, a, b, dtype):
    """kernels.py:339-351"""
    dtype = np.dtype(dtype)
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        if op == "eglue_plus":
            r = a + b
        elif op == "eglue_minus":
            r = a - b
        elif op == "eglue_schur":
            r = a * b
        else:
            r = int_div(a, b, dtype) if dtype.kind in "iu" else a / b
    return stage_cast(r, dtype)


def run_program(program, ins, compute_dtype) -> np.ndarray:
    """Post-order stage program over equally sized inputs (kernels.py:354-377).
    Inputs whose dtype differs from the compute dtype are C-cast on load
    (the reference's mov_copy, kernels.py:580-581)."""
    compute_dtype = np.dtype(compute_dtype)
    stack: list = []
    for st in program:
        tag = st[0]
        if tag == "load":
            stack.append(cast_out(np.asarray(ins[st[1]]), compute_dtype))
        elif tag == "unary":
            stack.append(apply_unary(st[1], stack.pop(), st[2] if len(st) > 2 else None, compute_dtype))
        elif tag == "scalar":
            stack.append(apply_scalar(st[1], stack.pop(), st[2], compute_dtype))
        elif tag == "glue":
            b = stack.pop()
            a = stack.pop()
            stack.append(apply_glue(st[1], a, b, compute_dtype))
        else:
            raise KeyError(tag)
    return stack[0] if len(stack) == 1 else tuple(stack)


# ---------------------------------------------------------------------------
# scalar reductions (kernels.py:380-392, 459-472, 779-798; runtime.py:279-285)

def py_min(a, b):
    """Python's built-in min(a, b): keeps a unless b < a."""
    return b if b < a else a


def py_max(a, b):
    return b if b > a else a


def combine_pairwise(partials, op):
    """Fixed binary-tree fold in block order, odd element carried (kernels.py:380-392)."""
    vals = list(partials)
    if not vals:
        raise ValueError("no partials to combine")
    while len(vals) > 1:
        nxt = [op(vals[i], vals[i + 1]) for i in range(0, len(vals) - 1, 2)]
        if len(vals) % 2:
            nxt.append(vals[-1])
        vals = nxt
    return vals[0]


def block_ranges(total: int, block: int):
    """kernels.py:856-861"""
    if total == 0:
        return []
    return [(i * block, min((i + 1) * block, total)) for i in range((total + block - 1) // block)]


def reduce_accu(x: np.ndarray):
    """reduce_accu: per-block ndarray.sum in the element type, pairwise fold."""
    x = np.ascontiguousarray(x).reshape(-1)
    parts = [x[lo:hi].sum(dtype=x.dtype) for lo, hi in block_ranges(x.shape[0], REDUCE_BLOCK)]
    if not parts:
        return x.dtype.type(0)
    with np.errstate(over="ignore"):
        return combine_pairwise(parts, lambda a, b: a + b)


def reduce_min(x: np.ndarray):
    x = np.ascontiguousarray(x).reshape(-1)
    parts = [x[lo:hi].min() for lo, hi in block_ranges(x.shape[0], REDUCE_BLOCK)]
    if not parts:
        raise ValueError("reduce_min: reduction over an empty range")
    return combine_pairwise(parts, py_min)


def reduce_max(x: np.ndarray):
    x = np.ascontiguousarray(x).reshape(-1)
    parts = [x[lo:hi].max() for lo, hi in block_ranges(x.shape[0], REDUCE_BLOCK)]
    if not parts:
        raise ValueError("reduce_max: reduction over an empty range")
    return combine_pairwise(parts, py_max)


def reduce_dot(a: np.ndarray, b: np.ndarray):
    """reduce_dot: per-block np.dot (OpenBLAS sdot/ddot), pairwise fold."""
    a = np.ascontiguousarray(a).reshape(-1)
    b = np.ascontiguousarray(b).reshape(-1)
    parts = [np.dot(a[lo:hi], b[lo:hi]) for lo, hi in block_ranges(a.shape[0], REDUCE_BLOCK)]
    if not parts:
        return a.dtype.type(0)
    with np.errstate(over="ignore"):
        return combine_pairwise(parts, lambda u, v: u + v)


def numpy_pairwise_sum(a: np.ndarray):
    """numpy's pairwise summation as ndarray.sum performs it on a contiguous
    array: 8 interleaved accumulators for n <= 128, otherwise split at n/2
    rounded down to a multiple of 8; the reduction adds the result to 0.
    This is the order the device reproduces (bm_reduce.cuh); pinned against
    ndarray.sum in tests/test_oracle.py."""
    dt = a.dtype.type

    def rec(lo: int, n: int):
        if n < 8:
            r = dt(0)
            for i in range(n):
                r = dt(r + a[lo + i])
            return r
        if n <= 128:
            acc = [a[lo + j] for j in range(8)]
            i = 8
            body = n - n % 8
            while i < body:
                for j in range(8):
                    acc[j] = dt(acc[j] + a[lo + i + j])
                i += 8
            r = dt(dt(dt(acc[0] + acc[1]) + dt(acc[2] + acc[3])) + dt(dt(acc[4] + acc[5]) + dt(acc[6] + acc[7])))
            while i < n:
                r = dt(r + a[lo + i])
                i += 1
            return r
        n2 = n // 2
        n2 -= n2 % 8
        return dt(rec(lo, n2) + rec(lo + n2, n - n2))

    with np.errstate(over="ignore", invalid="ignore"):
        return dt(dt(0) + rec(0, a.shape[0]))


# ---------------------------------------------------------------------------
# per-dimension reductions (kernels.py:496-531)

def rdim(op: str, a: np.ndarray, dim: int) -> np.ndarray:
    """op in sum/min/max/mean/var over a (rows, cols) array; returns the
    reference's result shape (1 x cols for dim 0, rows x 1 for dim 1).
    Blocks of DIM_BLOCK outputs, as the reference executes them."""
    a = np.asfortranarray(a)
    rows, cols = a.shape
    axis = 0 if dim == 0 else 1
    total = cols if dim == 0 else rows
    out = np.empty(total, dtype=a.dtype)
    for lo, hi in block_ranges(total, DIM_BLOCK):
        seg = a[:, lo:hi] if dim == 0 else a[lo:hi, :]
        if op == "sum":
            r = seg.sum(axis=axis, dtype=a.dtype)
        elif op == "min":
            r = seg.min(axis=axis)
        elif op == "max":
            r = seg.max(axis=axis)
        elif op == "mean":
            r = apply_scalar("eop_scalar_div_post", seg.sum(axis=axis, dtype=a.dtype), seg.shape[axis], a.dtype)
        elif op == "var":
            extent = seg.shape[axis]
            if extent < 2:
                r = np.zeros(seg.shape[1 - axis], dtype=a.dtype)
            else:
                mean = np.expand_dims(seg.sum(axis=axis, dtype=np.float64) / extent, axis)
                d = seg.astype(np.float64) - mean
                r = stage_cast((d * d).sum(axis=axis) / (extent - 1), a.dtype)
        else:
            raise KeyError(op)
        out[lo:hi] = cast_out(np.ascontiguousarray(r), a.dtype)
    return out.reshape(1, -1) if dim == 0 else out.reshape(-1, 1)


# ---------------------------------------------------------------------------
# gemm (kernels.py:704-708): 64-row panels through np.dot

def gemm(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    m = a.shape[0]
    out = np.empty((m, b.shape[1]), dtype=a.dtype)
    for lo, hi in block_ranges(m, GEMM_PANEL):
        out[lo:hi, :] = np.dot(a[lo:hi, :], b)
    return out


# ---------------------------------------------------------------------------
# norms (linalg.py:88-94, 486-529)

def norm_vector(x: np.ndarray, kind=2) -> float:
    x = np.ascontiguousarray(x).reshape(-1)
    if x.size == 0:
        return 0.0
    if kind in (2, "fro"):
        return math.sqrt(float(reduce_dot(x, x)))
    if kind == "inf":
        return float(reduce_max(np.abs(x)))
    if kind == "-inf":
        return float(reduce_min(np.abs(x)))
    if isinstance(kind, int) and kind >= 1:
        p = apply_unary("eop_pow", np.abs(x), kind, x.dtype)
        return float(reduce_accu(p)) ** (1.0 / kind)
    raise ValueError(kind)


def norm_matrix(a: np.ndarray, kind="fro") -> float:
    if a.size == 0:
        return 0.0
    if kind == "fro":
        flat = np.asfortranarray(a).reshape(-1, order="F")
        return math.sqrt(float(reduce_dot(flat, flat)))
    sums = rdim("sum", np.abs(a), 1).reshape(-1)
    return float(reduce_max(sums) if kind == "inf" else reduce_min(sums))


# ---------------------------------------------------------------------------
# counter RNG (kernels.py:227-253)

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def _mix64(x):
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def uniform_stream(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    key = _mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ _mix64(np.uint64(stream)))
    return (_mix64(idx ^ key) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal_stream(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    u1 = uniform_stream(seed, stream, 2 * start, 2 * count)[0::2]
    u2 = uniform_stream(seed, stream, 2 * start + 1, 2 * count)[0::2]
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


# ---------------------------------------------------------------------------
# config 5: logistic-regression gradient step, as the reference plans it
# (z = X@w -> gemm; r = 1/(1+exp(0-z)) - y -> 5-stage fused chain;
#  g = X.t()@r -> transpose + gemm; s = accu(r))

LOGISTIC_PROGRAM = (("load", 0), ("scalar", "eop_scalar_minus_pre", 0), ("unary", "eop_exp", None),
                    ("scalar", "eop_scalar_plus", 1), ("scalar", "eop_scalar_div_pre", 1), ("load", 1),
                    ("glue", "eglue_minus"))


def logistic_step(X: np.ndarray, w: np.ndarray, y: np.ndarray):
    z = gemm(X, w)
    r = run_program(LOGISTIC_PROGRAM, [z.reshape(-1), y.reshape(-1)], X.dtype).reshape(-1, 1)
    g = gemm(np.ascontiguousarray(X.T), r)
    s = reduce_accu(r)
    return g, r, s


# ---------------------------------------------------------------------------
# tree-walk evaluator (expr.py:851-1028): per-node numpy, no fusion

def tree_walk(node, leaf_data):
    """Evaluate an expression tree node by node.  ``leaf_data(matrix)`` returns
    the host (rows, cols) array of a leaf.  Node kinds/aux follow the
    reference's ExprNode (expr.py:63-139)."""
    kind = node.kind
    dt = NP_DTYPE[node.elem_type]
    if kind == "leaf":
        return np.asarray(leaf_data(node.operands[0]))
    if kind == "subview":
        parent = tree_walk(node.operands[0], leaf_data)
        return _region(parent, node.aux[0]).astype(dt)
    if kind in ("gen_zeros", "gen_ones", "gen_fill", "gen_eye", "gen_linspace"):
        r, c = node.aux[0], node.aux[1]
        if kind == "gen_zeros":
            return np.zeros((r, c), dtype=dt)
        if kind == "gen_ones":
            return np.ones((r, c), dtype=dt)
        if kind == "gen_fill":
            return np.full((r, c), node.aux[2]).astype(dt)
        if kind == "gen_eye":
            return np.eye(r, c, dtype=dt)
        return np.linspace(node.aux[2], node.aux[3], r).astype(dt).reshape(r, 1)
    if kind in ("gen_randu", "gen_randn"):      # expr.py:875-877: a device RNG stream cannot be replayed
        raise ValueError(f"oracle cannot replay the device RNG stream of {kind}")
    if kind == "mtop_conv_to":
        return cast_out(tree_walk(node.operands[0], leaf_data), dt)
    a = tree_walk(node.operands[0], leaf_data)
    if kind.startswith("eop_scalar"):
        return apply_scalar(kind, a, node.aux[0], dt)
    if kind.startswith("eop_"):
        return apply_unary(kind, a, node.aux[0] if node.aux else None, dt)
    if kind.startswith("eglue_"):
        return apply_glue(kind, a, tree_walk(node.operands[1], leaf_data), dt)
    if kind == "op_htrans":
        return np.ascontiguousarray(a.T)
    if kind == "op_diagmat":
        return np.diag(a.reshape(-1, order="F")).astype(dt)
    if kind == "op_diagvec":
        return np.diagonal(a, offset=node.aux[0]).astype(dt).reshape(-1, 1)
    if kind == "op_vectorise":
        return a.reshape(-1, order="F").reshape(-1, 1)
    if kind == "op_reshape":
        r, c = node.aux
        flat = a.reshape(-1, order="F")
        out = np.zeros(r * c, dtype=dt)
        n = min(flat.shape[0], r * c)
        out[:n] = flat[:n]
        return out.reshape((r, c), order="F")
    if kind == "op_resize":
        r, c = node.aux
        out = np.zeros((r, c), dtype=dt)
        kr, kc = min(r, a.shape[0]), min(c, a.shape[1])
        out[:kr, :kc] = a[:kr, :kc]
        return out
    if kind == "op_repmat":
        return np.tile(a, (node.aux[0], node.aux[1]))
    if kind in ("op_sum_dim", "op_min_dim", "op_max_dim", "op_mean_dim", "op_var_dim", "op_stddev_dim"):
        op = kind[3:-4]
        if op == "stddev":
            v = rdim("var", a, node.aux[0])
            return stage_cast(np.sqrt(v), dt)
        return rdim(op, a, node.aux[0])
    if kind == "glue_times":
        return np.dot(a, tree_walk(node.operands[1], leaf_data))
    if kind == "glue_join_rows":
        return np.hstack([a, tree_walk(node.operands[1], leaf_data)])
    if kind == "glue_join_cols":
        return np.vstack([a, tree_walk(node.operands[1], leaf_data)])
    raise ValueError(f"oracle: unknown node kind {kind!r}")


def _region(parent: np.ndarray, region: tuple) -> np.ndarray:
    tag = region[0]
    if tag == "diag":
        return np.diagonal(parent, offset=region[1]).reshape(-1, 1)
    if tag == "row":
        return parent[region[1]:region[1] + 1, :]
    if tag == "col":
        return parent[:, region[1]:region[1] + 1]
    if tag == "rows":
        return parent[region[1]:region[2] + 1, :]
    if tag == "cols":
        return parent[:, region[1]:region[2] + 1]
    p, q, r, s = region[1:]
    return parent[p:r + 1, q:s + 1]


# -- predicates (kernels.py:643-699) -------------------------------------------------------------

def predicate_mask(x: np.ndarray, op: str, k) -> np.ndarray:
    """_predicate_mask (kernels.py:643-657): the threshold cast to the element
    type first (_scalar), then numpy's comparison (NaN compares false except !=)."""
    kv = scalar_of(k, x.dtype)
    return {">": np.greater, "<": np.less, ">=": np.greater_equal, "<=": np.less_equal,
            "==": np.equal, "!=": np.not_equal}[op](x, kv)


def find_indices(a: np.ndarray, op: str = "!=", k=0) -> np.ndarray:
    """find (ops.py:207-229, kernels.py:660-662): ascending column-major linear
    indices of the matches, as u64."""
    flat = np.asfortranarray(a).reshape(-1, order="F")
    return np.nonzero(predicate_mask(flat, op, k))[0].astype(np.uint64)
