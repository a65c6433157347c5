"""Delayed evaluation: immutable expression trees, shape inference,
construction-time rewrites, and the planner that lowers a tree onto device
invocations.

Semantics (node kinds, shape rules, error types and messages, the three
rewrites, plan/evaluate behaviour) are the reference's
(reference/pkg/src/devmat/expr.py).  The lowering is B200-first:

* an element-wise subtree becomes ONE fused kernel of any depth (the
  reference splits after 8 stages, expr.py:615-626; splitting never changes
  bits because every stage rounds, so the planner only splits when the device
  limits of 16 inputs / 64 program slots are reached);
* a type conversion of a materialised matrix inside a chain is folded into the
  chain's load (the reference emits a separate mov_copy, expr.py:512-518);
* ``op_htrans`` operands of ``glue_times`` become GEMM transpose flags, so
  ``A @ B.t()`` is one NT GEMM with no mov_transpose (expr.py:543-547);
* scalar reductions over an expression (``accu``, ``dot``, ``norm``) run the
  element-wise program and the reduction in the same kernel
  (:func:`plan_reduce`) instead of materialising the tree first
  (ops.py:153-177);
* evaluate / evaluate_many / scalar reductions keep a recipe per DAG shape:
  the plan and its device invocations are built once, and a later call with
  matrices of the same shapes and types only re-addresses buffers (the
  reference re-plans every call), which keeps the host out of the way of a
  step that ends in a scalar read.
"""
from __future__ import annotations

import collections
import os
import threading
from dataclasses import dataclass, field, replace
from typing import NamedTuple

import numpy as np

from . import kernels, runtime
from .errors import DimensionError, ElemTypeError
from .kernels import NP_DTYPE
from .runtime import BlockView, FlatView, KernelInvocation


class Shape(NamedTuple):
    rows: int
    cols: int

    @property
    def n_elem(self) -> int:
        return self.rows * self.cols


EOP_UNARY_KINDS = frozenset(kernels.EOP_UNARY)
EOP_SCALAR_KINDS = frozenset(kernels.EOP_SCALAR)
EGLUE_KINDS = frozenset(kernels.EGLUE)
ELEMENTWISE_KINDS = EOP_UNARY_KINDS | EOP_SCALAR_KINDS | EGLUE_KINDS
GEN_KINDS = frozenset({"gen_zeros", "gen_ones", "gen_fill", "gen_eye", "gen_linspace", "gen_randu", "gen_randn"})
UNARY_OP_KINDS = frozenset({"op_htrans", "op_diagmat", "op_diagvec", "op_vectorise", "op_resize", "op_reshape",
                            "op_repmat"})
REDUCE_DIM_KINDS = frozenset({"op_sum_dim", "op_min_dim", "op_max_dim", "op_mean_dim", "op_var_dim",
                              "op_stddev_dim"})
GLUE_KINDS = frozenset({"glue_times", "glue_join_rows", "glue_join_cols"})
# conv_to folds into the producing kernel for these (two-way kernels)
CONV_FUSABLE_KINDS = ELEMENTWISE_KINDS | GEN_KINDS | UNARY_OP_KINDS | frozenset({"subview"})


# ---------------------------------------------------------------------------
# nodes

def _is_scalar(x) -> bool:
    return isinstance(x, (int, float, np.integer, np.floating)) and not isinstance(x, bool)


def as_expr(x) -> "ExprNode":
    if isinstance(x, ExprNode):
        return x
    hook = getattr(x, "_as_expr_node", None)
    if hook is None:
        raise TypeError(f"not an expression or matrix: {x!r}")
    return hook()


def _binary(kind_scalar: str, kind_glue: str):
    def op(a, b):
        if _is_scalar(b):
            return build_node(kind_scalar, (as_expr(a),), (b,))
        return build_node(kind_glue, (as_expr(a), as_expr(b)))
    return op


_plus = _binary("eop_scalar_plus", "eglue_plus")
_minus = _binary("eop_scalar_minus_post", "eglue_minus")
_divide = _binary("eop_scalar_div_post", "eglue_div")


def _times(a, b):
    if _is_scalar(b):
        return scalar_times(as_expr(a), b)
    return build_node("eglue_schur", (as_expr(a), as_expr(b)))


def _schur(a, b):
    return build_node("eglue_schur", (as_expr(a), as_expr(b)))


class ExpressionOps:
    """Operator surface shared by expression nodes and containers.

    ``*`` is the element-wise (Schur) product or a scalar multiply and ``@``
    is the matrix product -- the reference's operator assignment
    (expr.py:93-106), which its own tests depend on.  ``%`` is provided as
    an explicit Schur-product alias (Armadillo spelling).
    """

    __slots__ = ()
    __array_ufunc__ = None

    def __add__(self, other):
        return _plus(self, other)

    def __radd__(self, other):
        return _plus(self, other)

    def __sub__(self, other):
        return _minus(self, other)

    def __rsub__(self, other):
        return build_node("eop_scalar_minus_pre", (as_expr(self),), (other,))

    def __mul__(self, other):
        return _times(self, other)

    def __rmul__(self, other):
        return _times(self, other)

    def __mod__(self, other):
        return _schur(self, other)

    def __truediv__(self, other):
        return _divide(self, other)

    def __rtruediv__(self, other):
        return build_node("eop_scalar_div_pre", (as_expr(self),), (other,))

    def __matmul__(self, other):
        return build_node("glue_times", (as_expr(self), as_expr(other)))

    def __neg__(self):
        return build_node("eop_scalar_minus_pre", (as_expr(self),), (0,))

    def __pos__(self):
        return as_expr(self)

    def __abs__(self):
        return build_node("eop_abs", (as_expr(self),))

    def __gt__(self, k):
        return Relational(">", self, k)

    def __lt__(self, k):
        return Relational("<", self, k)

    def __ge__(self, k):
        return Relational(">=", self, k)

    def __le__(self, k):
        return Relational("<=", self, k)


@dataclass(frozen=True, eq=False)
class ExprNode(ExpressionOps):
    """Immutable DAG node; leaves (kind "leaf") hold a device matrix."""
    kind: str
    operands: tuple = ()
    aux: tuple = ()
    elem_type: str = "f32"

    __array_ufunc__ = None

    def t(self) -> "ExprNode":
        return rewrite_trans(self)

    def eval(self, elem_type: str | None = None):
        return evaluate(self if elem_type is None else conv_node(self, elem_type))

    def __repr__(self):
        s = shape_of(self)
        return f"ExprNode({self.kind}, {s.rows}x{s.cols}, {self.elem_type})"

    __hash__ = object.__hash__


@dataclass(frozen=True)
class Relational:
    """Element-versus-scalar comparison (consumed by find/all/any)."""
    op: str
    operand: object
    threshold: float


# ---------------------------------------------------------------------------
# shape inference (no device work)

def _diag_length(rows: int, cols: int, k: int) -> int:
    return max(0, min(rows, cols - k)) if k >= 0 else max(0, min(rows + k, cols))


def _region_shape(parent: Shape, region: tuple) -> Shape:
    tag = region[0]
    if tag == "diag":
        return Shape(_diag_length(parent.rows, parent.cols, region[1]), 1)
    if tag == "row":
        return Shape(1, parent.cols)
    if tag == "col":
        return Shape(parent.rows, 1)
    if tag == "rows":
        return Shape(region[2] - region[1] + 1, parent.cols)
    if tag == "cols":
        return Shape(parent.rows, region[2] - region[1] + 1)
    if tag == "submat":
        p, q, r, s = region[1:]
        return Shape(r - p + 1, s - q + 1)
    raise ValueError(f"unknown region kind {tag!r}")


def shape_of(node: ExprNode) -> Shape:
    """Result shape of an expression (expr.py:253-297)."""
    k = node.kind
    if k == "leaf":
        m = node.operands[0]
        return Shape(m.n_rows, m.n_cols)
    if k == "subview":
        return _region_shape(shape_of(node.operands[0]), node.aux[0])
    if k in GEN_KINDS or k in ("op_resize", "op_reshape"):
        return Shape(node.aux[0], node.aux[1])
    if k in ELEMENTWISE_KINDS or k == "mtop_conv_to":
        return shape_of(node.operands[0])
    a = shape_of(node.operands[0])
    if k == "op_htrans":
        return Shape(a.cols, a.rows)
    if k == "op_diagmat":
        return Shape(a.n_elem, a.n_elem)
    if k == "op_diagvec":
        return Shape(_diag_length(a.rows, a.cols, node.aux[0]), 1)
    if k == "op_vectorise":
        return Shape(a.n_elem, 1)
    if k == "op_repmat":
        return Shape(a.rows * node.aux[0], a.cols * node.aux[1])
    if k in REDUCE_DIM_KINDS:
        return Shape(1, a.cols) if node.aux[0] == 0 else Shape(a.rows, 1)
    if k in GLUE_KINDS:
        b = shape_of(node.operands[1])
        if k == "glue_times":
            return Shape(a.rows, b.cols)
        if k == "glue_join_rows":
            return Shape(a.rows, a.cols + b.cols)
        return Shape(a.rows + b.rows, a.cols)
    raise ValueError(f"unknown node kind {k!r}")


# ---------------------------------------------------------------------------
# construction

def _same_type(kind: str, a: ExprNode, b: ExprNode) -> None:
    if a.elem_type != b.elem_type:
        raise ElemTypeError(f"{kind}: element types differ ({a.elem_type} vs {b.elem_type}); "
                            "insert an explicit conversion")


def build_node(kind: str, operands: tuple = (), aux: tuple = (), elem_type: str | None = None) -> ExprNode:
    """Validating constructor: shape/type checks, no rewrites, no device work."""
    operands = tuple(operands)
    if elem_type is None:
        elem_type = operands[0].elem_type if operands else "f32"
    if kind in EGLUE_KINDS or kind in GLUE_KINDS:
        a, b = operands
        sa, sb = shape_of(a), shape_of(b)
        bad = {
            "glue_times": sa.cols != sb.rows,
            "glue_join_rows": sa.rows != sb.rows,
            "glue_join_cols": sa.cols != sb.cols,
        }.get(kind, sa != sb)
        if bad:
            raise DimensionError(kind, sa, sb)
        _same_type(kind, a, b)
    elif kind == "op_diagmat":
        s = shape_of(operands[0])
        if s.rows != 1 and s.cols != 1:
            raise DimensionError(kind, s)
    elif kind in ("op_resize", "op_reshape") or kind in GEN_KINDS:
        if aux[0] < 0 or aux[1] < 0:
            raise DimensionError(kind, (aux[0], aux[1]))
    elif kind in REDUCE_DIM_KINDS:
        if aux[0] not in (0, 1):
            raise ValueError(f"{kind}: dim must be 0 or 1")
    return ExprNode(kind, operands, tuple(aux), elem_type)


def conv_node(x, elem_type: str) -> ExprNode:
    node = as_expr(x)
    if elem_type not in NP_DTYPE:
        raise ElemTypeError(f"unknown element type {elem_type!r}")
    if node.elem_type == elem_type:
        return node
    return build_node("mtop_conv_to", (node,), (), elem_type)


def rewrite_trans(x) -> ExprNode:
    """trans(diagmat(v)) -> diagmat(v); trans(trans(X)) -> X (expr.py:368-380)."""
    node = as_expr(x)
    if node.kind == "op_diagmat":
        return node
    if node.kind == "op_htrans":
        return node.operands[0]
    return build_node("op_htrans", (node,))


def scalar_times(x, k) -> ExprNode:
    """k1*(k2*A) -> (k1*k2)*A (expr.py:383-388)."""
    node = as_expr(x)
    if node.kind == "eop_scalar_times":
        return build_node("eop_scalar_times", node.operands, (node.aux[0] * k,))
    return build_node("eop_scalar_times", (node,), (k,))


def census(x) -> dict[str, int]:
    """Node-kind histogram, shared nodes counted once."""
    out: dict[str, int] = {}
    seen: set[int] = set()
    stack = [as_expr(x)]
    while stack:
        n = stack.pop()
        if id(n) in seen:
            continue
        seen.add(id(n))
        out[n.kind] = out.get(n.kind, 0) + 1
        if n.kind != "leaf":
            stack.extend(n.operands)
    return out


# ---------------------------------------------------------------------------
# planning

@dataclass(frozen=True)
class PlanStep:
    kernel: str
    inputs: tuple            # ("slot", i) | ("leaf", Matrix)
    in_modes: tuple          # "flat" | "2d" | ("flat-region" | "block-region", ...)
    out_slot: int
    out_mode: str
    scalars: tuple = ()
    params: dict = field(default_factory=dict)


@dataclass(frozen=True)
class SlotInfo:
    rows: int
    cols: int
    elem_type: str


@dataclass
class EvalPlan:
    """Ordered device schedule for one evaluation."""
    steps: list
    slots: list
    result: tuple
    absorbed: list
    reduce: PlanStep | None = None   # trailing fused reduction (plan_reduce)
    extra: tuple = ()                # further result refs (evaluate_many)
    sums: tuple = ()                 # (slot, sum slot): a step also left accu(slot) in the reference's
                                     # order in a 1-element slot (the fused logistic step's r)

    @property
    def n_invocations(self) -> int:
        return len(self.steps) + (1 if self.reduce is not None else 0)

    @property
    def temp_schedule(self) -> dict:
        """slot -> (producing step, last consuming step); the result slot has none."""
        final = self.final_slots
        span = {s.out_slot: [i, None] for i, s in enumerate(self.steps)}
        for i, st in enumerate(self.steps):    # side outputs written by the step (logistic_grad's r)
            for a in st.params.get("alloc_slots", ()):
                span[a] = [i, None]
        consumers = list(self.steps) + ([self.reduce] if self.reduce is not None else [])
        for i, s in enumerate(consumers):
            for ref in s.inputs:
                if ref[0] == "slot" and ref[1] not in final:
                    span[ref[1]][1] = i
        return {k: tuple(v) for k, v in span.items()}

    @property
    def final_slots(self) -> set:
        refs = ((self.result,) if self.result else ()) + tuple(self.extra)
        return {r[1] for r in refs if r and r[0] == "slot"}

    def leaf_buffer_ids(self) -> set[int]:
        ids = {ref[1].mem.buffer_id for s in self.steps for ref in s.inputs if ref[0] == "leaf"}
        if self.result and self.result[0] == "leaf":
            ids.add(self.result[1].mem.buffer_id)
        return ids


# bm_reduce.cuh LG_ACCU_MAX_BLOCKS: the fused logistic step's accu(r) side output covers
# up to this many 8192-element blocks (2^26 rows)
LGRAD_ACCU_MAX_BLOCKS = 8192

_GEN_KERNEL = {"gen_zeros": "gen_fill_const", "gen_ones": "gen_fill_const", "gen_fill": "gen_fill_const",
               "gen_eye": "gen_eye", "gen_linspace": "gen_linspace", "gen_randu": "gen_randu",
               "gen_randn": "gen_randn"}
_FUSED_RDIM = frozenset({"op_sum_dim", "op_mean_dim", "op_min_dim", "op_max_dim", "op_var_dim", "op_stddev_dim"})
_RDIM_KERNEL = {"op_sum_dim": "rdim_sum", "op_min_dim": "rdim_min", "op_max_dim": "rdim_max",
                "op_mean_dim": "rdim_mean", "op_var_dim": "rdim_var", "op_stddev_dim": "rdim_var"}


class _Program:
    """Post-order stage program being assembled for one fused kernel."""

    def __init__(self):
        self.stages: list[tuple] = []
        self.inputs: list[tuple] = []

    def load(self, ref: tuple) -> None:
        key = (ref[0], id(ref[1]) if ref[0] == "leaf" else ref[1])
        for i, r in enumerate(self.inputs):
            if (r[0], id(r[1]) if r[0] == "leaf" else r[1]) == key:
                self.stages.append(("load", i))
                return
        self.inputs.append(ref)
        self.stages.append(("load", len(self.inputs) - 1))

    @property
    def n_stages(self) -> int:
        return sum(1 for s in self.stages if s[0] != "load")


class _Lowerer:
    def __init__(self, fuse: bool, chain_max: int | None = None):
        self.fuse = fuse
        self.chain_max = kernels.FUSED_CHAIN_MAX if chain_max is None else chain_max
        self.steps: list[PlanStep] = []
        self.slots: list[SlotInfo] = []
        self.absorbed: list[tuple] = []
        self.memo: dict = {}          # (id(node), type) -> ref of a value a fused step already produced
        self.sums: list = []          # (slot, sum slot) side outputs (EvalPlan.sums)

    def emit(self, kernel, inputs, in_modes, shape, out_type, out_mode, scalars=(), params=None,
             absorbed_from=None) -> tuple:
        self.slots.append(SlotInfo(shape.rows, shape.cols, out_type))
        slot = len(self.slots) - 1
        self.steps.append(PlanStep(kernel, tuple(inputs), tuple(in_modes), slot, out_mode, tuple(scalars),
                                   params or {}))
        if absorbed_from is not None and absorbed_from != out_type:
            self.absorbed.append((len(self.steps) - 1, absorbed_from, out_type))
        return ("slot", slot)

    # -- recursion ------------------------------------------------------------------------
    def lower(self, node: ExprNode, want: str):
        hit = self.memo.get((id(node), want))
        if hit is not None:
            return hit
        k = node.kind
        if k == "leaf":
            m = node.operands[0]
            if want == m.elem_type:
                return ("leaf", m)
            return self.emit("mov_copy", [("leaf", m)], ["flat"], shape_of(node), want, "flat")
        if k == "mtop_conv_to":
            child = node.operands[0]
            if self.fuse and child.kind in CONV_FUSABLE_KINDS:
                return self.lower(child, want)
            src = self.lower(child, child.elem_type)
            return self.emit("mov_copy", [src], ["flat"], shape_of(node), want, "flat")
        if k in ELEMENTWISE_KINDS:
            return self._chain(node, want)
        if k in GEN_KINDS:
            return self._generator(node, want)
        if k == "subview":
            parent = node.operands[0].operands[0]
            mode = _region_view_mode(parent, node.aux[0])
            return self.emit("mov_extract_strided", [("leaf", parent)], [mode], shape_of(node), want, "flat",
                             absorbed_from=node.elem_type)
        if k in UNARY_OP_KINDS:
            child = node.operands[0]
            src = self.lower(child, child.elem_type)
            shape = shape_of(node)
            if k == "op_htrans":
                return self.emit("mov_transpose", [src], ["2d"], shape, want, "2d", absorbed_from=node.elem_type)
            if k == "op_diagmat":
                return self.emit("mov_diagmat_build", [src], ["flat"], shape, want, "2d",
                                 absorbed_from=node.elem_type)
            if k == "op_diagvec":
                return self.emit("mov_diagvec_extract", [src], ["2d"], shape, want, "flat",
                                 params={"k": node.aux[0]}, absorbed_from=node.elem_type)
            if k in ("op_vectorise", "op_reshape"):
                return self.emit("mov_reshape_copy", [src], ["flat"], shape, want, "flat",
                                 absorbed_from=node.elem_type)
            if k == "op_resize":
                return self.emit("mov_resize", [src], ["2d"], shape, want, "2d", absorbed_from=node.elem_type)
            return self.emit("gen_repmat", [src], ["2d"], shape, want, "flat", params={"rows_out": shape.rows},
                             absorbed_from=node.elem_type)
        if k in ("glue_join_rows", "glue_join_cols"):
            a = self.lower(node.operands[0], node.operands[0].elem_type)
            b = self.lower(node.operands[1], node.operands[1].elem_type)
            kern = "mov_join_rows" if k == "glue_join_rows" else "mov_join_cols"
            return self.emit(kern, [a, b], ["2d", "2d"], shape_of(node), want, "2d", absorbed_from=node.elem_type)
        if k in REDUCE_DIM_KINDS:
            child = node.operands[0]
            ref = self._fused_rdim(node, want)
            if ref is not None:
                return ref
            src = self.lower(child, child.elem_type)
            ref = self.emit(_RDIM_KERNEL[k], [src], ["2d"], shape_of(node), child.elem_type, "flat",
                            params={"dim": node.aux[0]})
            if k == "op_stddev_dim":
                ref = self.emit("eop_sqrt", [ref], ["flat"], shape_of(node), child.elem_type, "flat")
            if want != child.elem_type:
                ref = self.emit("mov_copy", [ref], ["flat"], shape_of(node), want, "flat")
            return ref
        if k == "glue_times":
            if self.fuse:
                ref = self._logistic(node, want)
                if ref is None:
                    ref = self._gemm_prologue(node, want)
                if ref is not None:
                    return ref
            a, b = node.operands
            ta = tb = 0
            if a.kind == "op_htrans":     # fold the transpose into the GEMM
                a, ta = a.operands[0], 1
            if b.kind == "op_htrans":
                b, tb = b.operands[0], 1
            ra = self.lower(a, a.elem_type)
            rb = self.lower(b, b.elem_type)
            ref = self.emit("gemm", [ra, rb], ["2d", "2d"], shape_of(node), node.operands[0].elem_type, "2d",
                            params={"trans_a": ta, "trans_b": tb})
            if want != node.operands[0].elem_type:
                ref = self.emit("mov_copy", [ref], ["flat"], shape_of(node), want, "flat")
            return ref
        raise ValueError(f"cannot lower node kind {k!r}")

    # -- fused single-pass logistic step ---------------------------------------
    def _logistic(self, node: ExprNode, want: str):
        """X.t() @ F(X @ w, leaves...) -> one logistic_grad step that reads X
        once and also produces F(...) (memoised, so evaluate_many can return
        it).  Only the config-5 shape class: f32, X a leaf with k <= 4096
        columns and m % 4 == 0 rows, F element-wise over the one product X @ w
        and m x 1 f32 leaves.  Anything else lowers as GEMV + chain + GEMV."""
        a, b = node.operands
        if a.kind != "op_htrans" or a.operands[0].kind != "leaf" or b.kind not in ELEMENTWISE_KINDS:
            return None
        X = a.operands[0].operands[0]
        m, k = X.n_rows, X.n_cols
        sb = shape_of(b)
        if X.elem_type != "f32" or b.elem_type != "f32" or sb.rows != m or sb.cols != 1:
            return None
        if not 1 <= k <= 4096 or m % 4 or m < 16:      # clusters of 2 / 4 / 8 CTAs x 512 columns
            return None
        found: list = []

        def scan(n: ExprNode) -> bool:
            if n.kind in ELEMENTWISE_KINDS:
                return all(scan(o) for o in n.operands)
            if n.kind == "glue_times" and n.operands[0].kind == "leaf" and n.operands[0].operands[0] is X:
                if found and found[0] is not n:
                    return False
                found[:] = [n]
                return True
            if n.kind == "leaf":
                s_ = shape_of(n)
                return n.elem_type == "f32" and s_.rows == m and s_.cols == 1
            return False

        ok = scan(b)
        scan = None  # noqa: F841  (break the closure's self-reference, as for walk below)
        if not ok or not found:
            return None
        gnode = found[0]
        w = gnode.operands[1]
        sw = shape_of(w)
        if w.elem_type != "f32" or sw.rows != k or sw.cols != 1:
            return None
        prog = _Program()
        prog.inputs.append(("z", None))       # program input 0: X @ w, computed in the kernel

        def walk(n: ExprNode) -> None:
            if n is gnode:
                prog.stages.append(("load", 0))
            elif n.kind == "leaf":
                prog.load(("leaf", n.operands[0]))
            elif n.kind in EGLUE_KINDS:
                walk(n.operands[0])
                walk(n.operands[1])
                prog.stages.append(("glue", n.kind))
            elif n.kind in EOP_SCALAR_KINDS:
                walk(n.operands[0])
                prog.stages.append(("scalar", n.kind, n.aux[0]))
            else:
                walk(n.operands[0])
                prog.stages.append(("unary", n.kind, n.aux[0] if n.aux else None))

        walk(b)
        walk = None  # noqa: F841  (break the closure's self-reference, see program())
        if len(prog.stages) > 64 or len(prog.inputs) + 2 > 16:
            return None
        wref = self.lower(w, "f32")
        self.slots.append(SlotInfo(m, 1, "f32"))
        r_slot = len(self.slots) - 1
        params = {"program": tuple(prog.stages), "compute_dtype": NP_DTYPE["f32"].str, "alloc_slots": (r_slot,)}
        if -(-m // kernels.REDUCE_BLOCK) <= LGRAD_ACCU_MAX_BLOCKS:
            # the kernel also leaves accu(r) (reference order) in a 1-element slot, so a
            # following accu(r) of the returned matrix is a 4-byte read (runtime sum cache)
            self.slots.append(SlotInfo(1, 1, "f32"))
            a_slot = len(self.slots) - 1
            params["alloc_slots"] = (r_slot, a_slot)
            params["accu_slot"] = a_slot
            self.sums.append((r_slot, a_slot))
        inputs = [("leaf", X), wref, ("slot", r_slot)] + list(prog.inputs[1:])
        modes = ["2d", "flat", "flat"] + ["flat"] * (len(prog.inputs) - 1)
        ref = self.emit("logistic_grad", inputs, modes, shape_of(node), "f32", "flat", params=params)
        self.memo[(id(b), "f32")] = ("slot", r_slot)
        if want != "f32":
            ref = self.emit("mov_copy", [ref], ["flat"], shape_of(node), want, "flat")
        return ref

    # -- GEMM prologue fusion ------------------------------------------------
    def _gemm_prologue(self, node: ExprNode, want: str):
        """glue_times with an element-wise operand on the tensor-core paths:
        f32 -- the operands' programs run inside the 3xTF32 split pre-pass;
        f64 -- inside the DMMA kernel's register-staged producer (gemm_fused),
        instead of materialising `2*A + 1` first (expr.py:596-605).  Vector
        and small shapes keep the reference's lowering (GEMV / SIMT)."""
        a, b = node.operands
        ta = tb = 0
        if a.kind == "op_htrans":
            a, ta = a.operands[0], 1
        if b.kind == "op_htrans":
            b, tb = b.operands[0], 1
        elem = node.elem_type
        if elem not in ("f32", "f64") or a.elem_type != elem or b.elem_type != elem:
            return None
        if elem == "f64" and not _F64_PROLOGUE:
            # the DMMA producer re-evaluates an operand program in every CTA that
            # reads the tile; the issue-bound loop measured 36.2 ms against 32.1 ms
            # for materialising (2A + 1), (B - 3) first at 8192^3 (bm_gemm_tc.cuh)
            return None
        if a.kind not in ELEMENTWISE_KINDS and b.kind not in ELEMENTWISE_KINDS:
            return None
        s = shape_of(node)
        sa, sb = shape_of(a), shape_of(b)
        k = sa.rows if ta else sa.cols
        if s.rows < 2 or s.cols < 2 or s.rows * s.cols * k < (1 << (21 if elem == "f32" else 18)):
            return None
        if elem == "f64" and -(-s.rows // 64) > 65535:
            return None
        mark = (len(self.steps), len(self.slots), len(self.absorbed))
        progs = []
        for x in (a, b):
            if x.kind in ELEMENTWISE_KINDS:
                pr = self._fit_program(x, elem)
            else:
                pr = _Program()
                pr.load(self.lower(x, elem))
            progs.append(pr)
        # f64 (DMMA): every input of an operand program is staged in shared memory
        # beside the others, so at most three f64 inputs in all (two CTAs per SM)
        limit = 16 if elem == "f32" else 3
        f64_ok = elem == "f32" or all(self._ref_elem(r) == "f64" for pr in progs for r in pr.inputs)
        if len(progs[0].inputs) + len(progs[1].inputs) > limit or len(progs[0].stages) + len(progs[1].stages) > 64 \
                or not f64_ok:
            del self.steps[mark[0]:]
            del self.slots[mark[1]:]
            del self.absorbed[mark[2]:]
            return None
        inputs = list(progs[0].inputs) + list(progs[1].inputs)
        ref = self.emit("gemm_fused", inputs, ["flat"] * len(inputs), s, elem, "2d",
                        params={"a_prog": tuple(progs[0].stages), "b_prog": tuple(progs[1].stages),
                                "na": len(progs[0].inputs), "trans_a": ta, "trans_b": tb,
                                "a_rows": sa.rows, "b_rows": sb.rows, "m": s.rows, "n": s.cols, "k": k})
        if want != elem:
            ref = self.emit("mov_copy", [ref], ["flat"], s, want, "flat")
        return ref

    # -- element-wise programs -----------------------------------------------------------------
    def program(self, root: ExprNode, elem: str, budget: int, pre=None) -> _Program:
        """Collect the fusable element-wise subtree under ``root`` into a stage
        program; everything else is lowered into slots and loaded.  ``pre`` =
        (node, ref): that node is program input 0 and loads ``ref`` instead of
        being lowered (a GEMM whose store runs the program, _gemm_epilogue)."""
        prog = _Program()
        if pre is not None:
            prog.inputs.append(pre[1])
        left = [budget if self.fuse else 1]

        def load(node: ExprNode) -> None:
            if pre is not None and node is pre[0]:
                prog.load(pre[1])
                return
            # a converted materialised matrix is read with a load-time cast
            if (self.fuse and node.kind == "mtop_conv_to" and node.elem_type == elem
                    and node.operands[0].kind == "leaf"):
                prog.load(("leaf", node.operands[0].operands[0]))
                return
            prog.load(self.lower(node, elem))

        def walk(node: ExprNode) -> None:
            if node.kind not in ELEMENTWISE_KINDS or left[0] <= 0:
                load(node)
                return
            left[0] -= 1
            if node.kind in EGLUE_KINDS:
                walk(node.operands[0])
                walk(node.operands[1])
                prog.stages.append(("glue", node.kind))
            elif node.kind in EOP_SCALAR_KINDS:
                walk(node.operands[0])
                prog.stages.append(("scalar", node.kind, node.aux[0]))
            else:
                walk(node.operands[0])
                prog.stages.append(("unary", node.kind, node.aux[0] if node.aux else None))

        walk(root)
        # `walk` refers to itself through its closure cell: clear the cell so
        # that the program's operands (device matrices) are released by
        # reference counting, not at the next garbage-collector pass
        walk = None  # noqa: F841
        return prog

    def _fit_program(self, root: ExprNode, elem: str, extra_slots: int = 0, pre=None) -> _Program:
        budget = self.chain_max
        while True:
            mark = (len(self.steps), len(self.slots), len(self.absorbed))
            prog = self.program(root, elem, budget, pre)
            fits = (len(prog.inputs) <= kernels.FUSED_INPUTS_MAX
                    and len(prog.stages) + extra_slots <= 64)
            if fits or budget <= 1:
                return prog
            # roll back and retry with a shallower fusion
            del self.steps[mark[0]:]
            del self.slots[mark[1]:]
            del self.absorbed[mark[2]:]
            budget = max(1, budget // 2)

    def _gemm_epilogue(self, root: ExprNode, want: str):
        """An element-wise function of one matrix product (f32 on the 3xTF32
        path, f64 on DMMA), e.g. ``exp(A @ B.t() / n)``: the tree becomes the
        GEMM's epilogue (gemm_epi), so the product is never materialised and
        C is written once.  The reference lowers the product and the chain
        separately (expr.py:596-605, 611-657).  GEMV, small shapes and trees
        that read other matrices keep that plan."""
        elem = root.elem_type
        if elem not in ("f32", "f64"):
            return None
        found: list = []

        def scan(n: ExprNode) -> None:
            if n.kind in ELEMENTWISE_KINDS:
                for o in n.operands:
                    scan(o)
            elif n.kind == "glue_times" and not any(f is n for f in found):
                found.append(n)

        scan(root)
        scan = None  # noqa: F841  (break the closure's self-reference)
        if len(found) != 1 or found[0].elem_type != elem:
            return None
        g = found[0]
        a, b = g.operands
        ta = tb = 0
        if a.kind == "op_htrans":
            a, ta = a.operands[0], 1
        if b.kind == "op_htrans":
            b, tb = b.operands[0], 1
        s = shape_of(g)
        sa = shape_of(a)
        k = sa.rows if ta else sa.cols
        if s.rows < 2 or s.cols < 2 or k < 1 or s.rows * s.cols * k < (1 << (21 if elem == "f32" else 18)):
            return None
        mark = (len(self.steps), len(self.slots), len(self.absorbed))
        ra = self.lower(a, elem)
        rb = self.lower(b, elem)
        prog = self._fit_program(root, elem, pre=(g, ("gemm", None)))
        # Programs of the product alone, or (f32) of the product and one f32 matrix
        # with 4 | rows, which the pair kernel stages through shared memory during the main loop
        # (8192^3: exp(AB^T/n) - C 4.53 ms fused vs 4.60 unfused, 2AB^T + 3C 4.45-4.58
        # vs 4.73-4.78; profiles/r02_gemm_persist.txt).  More inputs, f64 and odd row
        # counts read them with dependent loads after the drain: slower, the
        # reference's plan unless BM_GEMM_EPI_INPUTS=1.
        mem = prog.inputs[1:]
        mem_ok = not mem or _EPI_MEM_INPUTS or (
            _EPI_STAGE and elem == "f32" and len(mem) == 1 and self._ref_elem(mem[0]) == "f32" and s.rows % 4 == 0)
        if not mem_ok or len(prog.stages) > 64 or \
                prog.inputs[0] != ("gemm", None) or ("load", 0) not in prog.stages:
            del self.steps[mark[0]:]
            del self.slots[mark[1]:]
            del self.absorbed[mark[2]:]
            return None
        inputs = [ra, rb] + list(prog.inputs[1:])
        ref = self.emit("gemm_epi", inputs, ["2d", "2d"] + ["flat"] * (len(inputs) - 2), shape_of(root), elem, "flat",
                        params={"program": tuple(prog.stages), "compute_dtype": NP_DTYPE[elem].str,
                                "trans_a": ta, "trans_b": tb})
        if want != elem:
            ref = self.emit("mov_copy", [ref], ["flat"], shape_of(root), want, "flat")
        return ref

    def _chain(self, root: ExprNode, want: str):
        elem = root.elem_type
        if self.fuse:
            ref = self._gemm_epilogue(root, want)
            if ref is not None:
                return ref
        prog = self._fit_program(root, elem)
        shape = shape_of(root)
        if prog.n_stages == 1 and len(prog.stages) == len(prog.inputs) + 1 and \
                all(prog.stages[i] == ("load", i) for i in range(len(prog.inputs))) and \
                all(self._ref_elem(r) == elem for r in prog.inputs):
            # one stage over distinct inputs: the reference's dedicated kernel name
            st = prog.stages[-1]
            scal = (st[2],) if len(st) > 2 and st[2] is not None else ()
            return self.emit(st[1], prog.inputs, ["flat"] * len(prog.inputs), shape, want, "flat",
                             scalars=scal, absorbed_from=elem)
        return self.emit("fused_chain", prog.inputs, ["flat"] * len(prog.inputs), shape, want, "flat",
                         params={"program": tuple(prog.stages), "compute_dtype": NP_DTYPE[elem].str},
                         absorbed_from=elem)

    def _fused_rdim(self, node: ExprNode, want: str):
        """sum / mean / min / max over dim 0 of an element-wise tree: one
        ``fused_rdim`` step (b200mat.h BM_K_RDIM_FUSED) whose column reductions
        evaluate the tree's program instead of reading a materialised temporary
        (the reference lowers the child first, expr.py:583-594).  Same values,
        same reduction order: the same bits."""
        k, child = node.kind, node.operands[0]
        dim = node.aux[0]
        if not self.fuse or k not in _FUSED_RDIM or child.kind not in ELEMENTWISE_KINDS:
            return None
        shp = shape_of(child)
        if shp.rows == 0 or shp.cols == 0:
            return None
        elem = child.elem_type
        if dim == 1:
            # TMA-staged row folds (bm_rdim0.cuh rdim1_fused_body): rows must make
            # 16-B column strides, and numpy's lone-row block (rows % 64 == 1,
            # kernels.py:89) sums pairwise, so it keeps the two-step plan
            isz = NP_DTYPE[elem].itemsize
            if (shp.rows * isz) % 16 or shp.rows % 64 == 1:
                return None
        mark = (len(self.steps), len(self.slots), len(self.absorbed))
        prog = self._fit_program(child, elem)
        if dim == 1 and (len(prog.inputs) > 8 or any(self._ref_elem(r) != elem for r in prog.inputs)):
            del self.steps[mark[0]:]
            del self.slots[mark[1]:]
            del self.absorbed[mark[2]:]
            return None
        ref = self.emit("fused_rdim", prog.inputs, ["flat"] * len(prog.inputs), shape_of(node), elem, "flat",
                        params={"program": tuple(prog.stages), "compute_dtype": NP_DTYPE[elem].str,
                                "op": _RDIM_KERNEL[k], "rows": shp.rows, "cols": shp.cols, "dim": dim})
        if k == "op_stddev_dim":
            ref = self.emit("eop_sqrt", [ref], ["flat"], shape_of(node), elem, "flat")
        if want != elem:
            ref = self.emit("mov_copy", [ref], ["flat"], shape_of(node), want, "flat")
        return ref

    def _ref_elem(self, ref) -> str:
        return ref[1].elem_type if ref[0] == "leaf" else self.slots[ref[1]].elem_type

    def _generator(self, node: ExprNode, want: str):
        shape = shape_of(node)
        params: dict = {"gen_type": node.elem_type}
        scalars: tuple = ()
        k = node.kind
        if k == "gen_zeros":
            scalars = (0,)
        elif k == "gen_ones":
            scalars = (1,)
        elif k == "gen_fill":
            scalars = (node.aux[2],)
        elif k == "gen_eye":
            params["rows"] = shape.rows
        elif k == "gen_linspace":
            scalars = (node.aux[2], node.aux[3])
            params["n"] = shape.n_elem
        else:
            params["rng"] = True
        return self.emit(_GEN_KERNEL[k], [], [], shape, want, "flat", scalars=scalars, params=params,
                         absorbed_from=node.elem_type)


def _region_view_mode(parent, region: tuple):
    """A subview region as a concrete strided view descriptor (expr.py:682-703)."""
    n, tag = parent.n_rows, region[0]
    if tag == "diag":
        k = region[1]
        length = _diag_length(parent.n_rows, parent.n_cols, k)
        return ("flat-region", k * n if k >= 0 else -k, length, n + 1)
    if tag == "row":
        return ("flat-region", region[1], parent.n_cols, n)
    if tag == "col":
        return ("flat-region", region[1] * n, parent.n_rows, 1)
    if tag == "rows":
        a, b = region[1], region[2]
        return ("block-region", a, b - a + 1, parent.n_cols, n)
    if tag == "cols":
        c, d = region[1], region[2]
        return ("block-region", c * n, parent.n_rows, d - c + 1, n)
    if tag == "submat":
        p, q, r, s = region[1:]
        return ("block-region", p + q * n, r - p + 1, s - q + 1, n)
    raise ValueError(f"unknown region kind {tag!r}")


def plan(x, out_elem_type: str | None = None, fuse: bool = True, chain_max: int | None = None) -> EvalPlan:
    """Lower an expression to an ordered device schedule.  ``chain_max=8``
    reproduces the reference's chain splitting (kernels.py:91-92)."""
    node = as_expr(x)
    low = _Lowerer(fuse, chain_max)
    result = low.lower(node, out_elem_type or node.elem_type)
    return EvalPlan(low.steps, low.slots, result, low.absorbed, sums=tuple(low.sums))


def plan_reduce(op: str, *xs, fuse: bool = True) -> EvalPlan:
    """Plan a scalar reduction (``accu``/``min``/``max`` over one expression,
    ``dot`` over two) whose element-wise part runs inside the reduction kernel.
    The result is ``plan.reduce``, a ``fused_reduce`` step executed with
    Runtime.execute_reduce."""
    nodes = [as_expr(x) for x in xs]
    elem = nodes[0].elem_type
    low = _Lowerer(fuse)
    prog = _Program()
    for node in nodes:
        sub = low._fit_program(node, elem, extra_slots=len(prog.stages))
        remap = []
        for ref in sub.inputs:
            before = len(prog.inputs)
            prog.load(ref)
            remap.append(prog.stages.pop()[1])
            del before
        for st in sub.stages:
            prog.stages.append(("load", remap[st[1]]) if st[0] == "load" else st)
    red = PlanStep("fused_reduce", tuple(prog.inputs), ("flat",) * len(prog.inputs), -1, "none", (),
                   {"program": tuple(prog.stages), "compute_dtype": NP_DTYPE[elem].str, "op": op})
    return EvalPlan(low.steps, low.slots, None, low.absorbed, reduce=red, sums=tuple(low.sums))


# ---------------------------------------------------------------------------
# execution

def _make_view(buf, rows: int, cols: int, mode):
    if mode == "flat":
        return FlatView(buf, 0, rows * cols)
    if mode == "2d":
        return BlockView(buf, 0, rows, cols, rows)
    if mode[0] == "flat-region":
        return FlatView(buf, mode[1], mode[2], mode[3])
    if mode[0] == "block-region":
        return BlockView(buf, mode[1], mode[2], mode[3], mode[4])
    raise ValueError(f"unknown view mode {mode!r}")


def _step_views(plan_obj: EvalPlan, step: PlanStep, slot_bufs: dict, leaves=None) -> list:
    views = []
    for ref, mode in zip(step.inputs, step.in_modes):
        if ref[0] == "slot":
            info = plan_obj.slots[ref[1]]
            views.append(_make_view(slot_bufs[ref[1]], info.rows, info.cols, mode))
        else:
            m = ref[1] if ref[0] == "leaf" else leaves[ref[1]]
            views.append(_make_view(m.mem, m.n_rows, m.n_cols, mode))
    return views


# ---------------------------------------------------------------------------
# plan recipes
#
# A recipe is a plan lowered once for a DAG *shape* -- node kinds, scalars,
# element types, matrix shapes and which nodes / matrices are shared -- with
# its leaves replaced by positions ("leafpos", i), plus the device invocation
# of every step built on first use.  A later call with the same shape binds its
# own leaf matrices and only re-addresses the invocations (buffer pointers),
# skipping lowering, view construction and build_invocation.  Lowering depends
# on nothing but what the key holds (shapes, types, sharing), so a recipe is
# exactly the plan the call would have made.

_RECIPE_MAX = 256
_RECIPE_LOCK = threading.Lock()
_RECIPES_ON = os.environ.get("BM_PLAN_CACHE", "1") != "0"
_F64_PROLOGUE = os.environ.get("BM_F64_PROLOGUE", "0") == "1"   # f64 operand chains inside DMMA (off: slower)
_EPI_MEM_INPUTS = os.environ.get("BM_GEMM_EPI_INPUTS", "0") == "1"   # epilogues that read other matrices (off: slower)
_EPI_STAGE = os.environ.get("BM_GEMM_EPI_STAGE", "1") != "0"        # the kernel stages a one-matrix f32 input


class _NoRecipe(Exception):
    pass


def _dag_key(roots):
    """Structural key of the DAG under ``roots`` and its distinct leaf
    matrices in first-visit order (None when a node is not cacheable)."""
    ids: dict = {}
    lv: dict = {}
    leaves: list = []
    out: list = []
    stack = list(reversed(roots))
    while stack:
        n = stack.pop()
        i = ids.get(id(n))
        if i is not None:
            out.append(i)                       # a shared node: back-reference
            continue
        if not isinstance(n, ExprNode):
            return None, None
        ids[id(n)] = len(ids)
        if n.kind == "leaf":
            m = n.operands[0]
            j = lv.get(id(m))
            if j is None:
                j = lv[id(m)] = len(leaves)
                leaves.append(m)
            out.append((j, m.n_rows, m.n_cols, m.elem_type))
        else:
            out.append((n.kind, n.aux, n.elem_type, len(n.operands)))
            stack.extend(reversed(n.operands))
    return tuple(out), leaves


class _Recipe:
    __slots__ = ("plan", "protos", "reduce_proto", "out_refs", "finals", "release_after")

    def __init__(self, plan_obj: EvalPlan, out_refs=None):
        self.plan = plan_obj
        self.protos: list = [None] * len(plan_obj.steps)   # prebuilt invocation per step
        self.reduce_proto = None
        self.out_refs = out_refs
        self.finals = plan_obj.final_slots                  # the plan's schedule, computed once
        self.release_after = {s: span[1] for s, span in plan_obj.temp_schedule.items()}


def _templatise(plan_obj: EvalPlan, leaves: list) -> EvalPlan:
    pos = {id(m): i for i, m in enumerate(leaves)}

    def conv(ref):
        if ref is not None and ref[0] == "leaf":
            i = pos.get(id(ref[1]))
            if i is None:
                raise _NoRecipe
            return ("leafpos", i)
        return ref

    steps = [replace(st, inputs=tuple(conv(r) for r in st.inputs)) for st in plan_obj.steps]
    red = replace(plan_obj.reduce, inputs=tuple(conv(r) for r in plan_obj.reduce.inputs)) \
        if plan_obj.reduce is not None else None
    return EvalPlan(steps, plan_obj.slots, conv(plan_obj.result), [], reduce=red,
                    extra=tuple(conv(r) for r in plan_obj.extra), sums=plan_obj.sums)


def _recipe_for(key, leaves, make):
    """The recipe cached under ``key`` (per runtime, LRU), or a new one from
    ``make() -> (plan, out_refs)``; None when the plan cannot be one."""
    rt = runtime.get_runtime()
    cache = getattr(rt, "_recipes", None)
    if cache is None:
        cache = rt._recipes = collections.OrderedDict()
    with _RECIPE_LOCK:             # user threads evaluate concurrently (reference test_integration)
        rec = cache.get(key)
        if rec is not None:
            cache.move_to_end(key)
            return rec, None
    plan_obj, out_refs = make()
    if not plan_obj.steps and plan_obj.reduce is None:
        return None, plan_obj
    try:
        tmpl = _templatise(plan_obj, leaves)
        outs = None if out_refs is None else tuple(
            ("leafpos", leaves.index(r[1])) if r[0] == "leaf" else r for r in out_refs)
    except (_NoRecipe, ValueError):
        return None, plan_obj
    rec = _Recipe(tmpl, outs)
    with _RECIPE_LOCK:
        cache[key] = rec
        if len(cache) > _RECIPE_MAX:
            cache.popitem(last=False)
    return rec, None


def execute_plan(plan_obj: EvalPlan, target_buf=None, sums: dict | None = None, leaves=None, recipe=None):
    """Run the plan's steps; returns the result buffer (or the leaf matrix for
    an empty plan).  When the plan carries a fused reduction it is executed
    last and its value is returned instead.  ``sums`` (optional) receives
    {result slot: 1-element buffer} for the reference-order accu a step left
    beside a returned result (EvalPlan.sums); every other side output is
    released here.  A recipe's template plan names leaves by position
    (``leaves``); its invocations are built on the first run and re-addressed
    on later ones."""
    rt = runtime.get_runtime()
    if plan_obj.result is not None and plan_obj.result[0] == "leaf" and plan_obj.reduce is None and not plan_obj.extra:
        return plan_obj.result[1]
    final_slot = plan_obj.result[1] if plan_obj.result is not None else None
    if recipe is not None:
        finals, release_after = recipe.finals, recipe.release_after
    else:
        finals = plan_obj.final_slots
        release_after = {s: span[1] for s, span in plan_obj.temp_schedule.items()}
    slot_bufs: dict[int, object] = {}
    protos = recipe.protos if recipe is not None else None

    def ref_buf(ref):
        if ref[0] == "slot":
            return slot_bufs[ref[1]]
        return (ref[1] if ref[0] == "leaf" else leaves[ref[1]]).mem

    def step_bufs(refs):
        return [ref_buf(r) for r in refs]

    def release_inputs(step: PlanStep, i: int) -> None:
        done = set()
        for ref in step.inputs:
            s = ref[1]
            if ref[0] == "slot" and s not in finals and release_after.get(s) == i and s not in done:
                done.add(s)
                rt.release_deferred(slot_bufs.pop(s))

    def release_leftovers() -> None:
        # side outputs nobody consumed (the logistic step's r under evaluate(g), a sum slot
        # whose matrix is not returned): stream-ordered release
        if sums is not None:
            for r_slot, a_slot in plan_obj.sums:
                if r_slot in finals and a_slot in slot_bufs:
                    sums[r_slot] = slot_bufs.pop(a_slot)
        for s in [s for s in slot_bufs if s not in finals]:
            rt.release_deferred(slot_bufs.pop(s))

    for i, step in enumerate(plan_obj.steps):
        for a in step.params.get("alloc_slots", ()):     # side outputs the step writes
            ai = plan_obj.slots[a]
            slot_bufs[a] = rt.acquire_memory(ai.rows * ai.cols, ai.elem_type)
        info = plan_obj.slots[step.out_slot]
        if step.out_slot == final_slot and target_buf is not None:
            out_buf = target_buf
        else:
            out_buf = rt.acquire_memory(info.rows * info.cols, info.elem_type)
        slot_bufs[step.out_slot] = out_buf
        proto = protos[i] if protos is not None else None
        if proto is not None:
            a = step.params.get("accu_slot")
            rt.enqueue_prebuilt(proto, step.kernel, step_bufs(step.inputs), out_buf,
                                slot_bufs[a].ptr if a is not None else 0)
        else:
            views = _step_views(plan_obj, step, slot_bufs, leaves)
            params = dict(step.params)
            rng = params.pop("rng", None)
            if rng:
                params["seed"] = rt.seed
                params["stream"] = rt.next_stream_id()
            if "accu_slot" in params:
                params["accu_ptr"] = slot_bufs[params["accu_slot"]].ptr
            inv = KernelInvocation(step.kernel, tuple(views), _make_view(out_buf, info.rows, info.cols,
                                                                         step.out_mode), step.scalars, params)
            if protos is None or rng:
                rt.enqueue(inv)
            else:                                        # first run of a recipe: keep the invocation
                protos[i] = rt.prebuild(inv)
                rt.enqueue_prebuilt(protos[i], step.kernel, [v.buf for v in views], out_buf,
                                    params.get("accu_ptr", 0))
        release_inputs(step, i)
    if plan_obj.reduce is not None:
        step = plan_obj.reduce
        try:
            proto = recipe.reduce_proto if recipe is not None else None
            if proto is not None:
                value = rt.execute_reduce_prebuilt(proto, "fused_reduce", step_bufs(step.inputs))
            else:
                views = _step_views(plan_obj, step, slot_bufs, leaves)
                inv = KernelInvocation("fused_reduce", tuple(views), None, (), dict(step.params))
                if recipe is None:
                    value = rt.execute_reduce(inv)
                else:
                    recipe.reduce_proto = rt.prebuild(inv)
                    value = rt.execute_reduce_prebuilt(recipe.reduce_proto, "fused_reduce", [v.buf for v in views])
        finally:
            release_inputs(step, len(plan_obj.steps))
            release_leftovers()
        return value
    release_leftovers()
    if plan_obj.extra:
        return [slot_bufs[r[1]] if r[0] == "slot" else (r[1] if r[0] == "leaf" else leaves[r[1]])
                for r in (plan_obj.result,) + tuple(plan_obj.extra)]
    return slot_bufs[final_slot]


def evaluate(x, out=None, fuse: bool = True):
    """Evaluate into ``out`` (or a fresh matrix); expr.py:792-835 semantics:
    a bare leaf is a device-to-device copy, an output that aliases an operand
    adopts a fresh result buffer."""
    from .matrix import Matrix

    node = as_expr(x)
    rt = runtime.get_runtime()
    if out is not None and out.elem_type != node.elem_type:
        raise ElemTypeError(f"cannot assign {node.elem_type} expression to {out.elem_type} matrix; "
                            "convert explicitly")
    rec = leaves = None
    p = None
    if _RECIPES_ON:
        key, leaves = _dag_key((node,))
        if key is not None:
            rec, p = _recipe_for(("eval", fuse, node.elem_type, key), leaves,
                                 lambda: (plan(node, node.elem_type, fuse=fuse), None))
    if rec is not None:
        p = rec.plan
        leaf_ids = {m.mem.buffer_id for m in leaves}
    else:
        if p is None:
            p = plan(node, node.elem_type, fuse=fuse)
        leaves = None
        leaf_ids = None
    if p.result[0] == "slot":               # the plan knows the result's shape (no tree walk)
        si = p.slots[p.result[1]]
        shape = Shape(si.rows, si.cols)
    else:
        shape = shape_of(node)
    if p.result[0] == "leaf":
        src = p.result[1]
        if out is None:
            out = Matrix._uninitialised(shape.rows, shape.cols, node.elem_type)
        elif out is src:
            return out
        else:
            out._reshape_storage(shape.rows, shape.cols)
        rt.copy_d2d(src.mem, out.mem, shape.n_elem)
        return out
    if leaf_ids is None:
        leaf_ids = p.leaf_buffer_ids()
    aliased = out is not None and out.mem.buffer_id in leaf_ids
    if out is None or aliased:
        buf = execute_plan(p, leaves=leaves, recipe=rec)
        if out is None:
            return Matrix._adopt(buf, shape.rows, shape.cols, node.elem_type)
        out._adopt_buffer(buf, shape.rows, shape.cols)
        return out
    out._reshape_storage(shape.rows, shape.cols)
    execute_plan(p, target_buf=out.mem, leaves=leaves, recipe=rec)
    return out


def _lower_many(nodes, fuse: bool):
    low = _Lowerer(fuse)
    # products first, so that side outputs of fused steps are memoised
    # before the expressions that name them are lowered
    order = sorted(range(len(nodes)), key=lambda i: 0 if nodes[i].kind == "glue_times" else 1)
    refs: list = [None] * len(nodes)
    for i in order:
        refs[i] = low.lower(nodes[i], nodes[i].elem_type)
    seen: set = set()
    out_refs = []
    for r in refs:                 # a value asked for twice is copied for the second matrix
        if r[0] == "slot" and r[1] in seen:
            r = ("dup", r[1])
        elif r[0] == "slot":
            seen.add(r[1])
        out_refs.append(r)
    slot_refs = [r if r[0] != "dup" else ("slot", r[1]) for r in out_refs]
    p = EvalPlan(low.steps, low.slots, slot_refs[0], low.absorbed, extra=tuple(slot_refs[1:]),
                 sums=tuple(low.sums))
    return p, out_refs


def evaluate_many(*xs, fuse: bool = True) -> list:
    """Evaluate several expressions in one plan and return one fresh matrix
    per expression (an extension of the reference's evaluate).  Values a
    fused step produces on the way are shared: with r = F(X @ w, y) and
    g = X.t() @ r, ``r, g = evaluate_many(r, g)`` reads X once (the fused
    logistic step) instead of twice."""
    from .matrix import Matrix
    nodes = [as_expr(x) for x in xs]
    if not nodes:
        return []
    rec = leaves = None
    if _RECIPES_ON:
        key, leaves = _dag_key(nodes)
        if key is not None:
            rec, _ = _recipe_for(("many", fuse, key), leaves, lambda: _lower_many(nodes, fuse))
    if rec is not None:
        p, out_refs = rec.plan, rec.out_refs
    else:
        p, out_refs = _lower_many(nodes, fuse)
        leaves = None
    rt = runtime.get_runtime()
    sums: dict = {}
    if not p.steps:
        bufs = [(r[1] if r[0] == "leaf" else leaves[r[1]]) if r[0] != "slot" else None
                for r in ((p.result,) + tuple(p.extra))]
    else:
        bufs = execute_plan(p, sums=sums, leaves=leaves, recipe=rec)
    result = []
    for node, r, b in zip(nodes, out_refs, bufs):
        if r[0] == "slot":
            si = p.slots[r[1]]
            shape = Shape(si.rows, si.cols)
        else:
            shape = shape_of(node)
        if r[0] == "slot":
            result.append(Matrix._adopt(b, shape.rows, shape.cols, node.elem_type))
            if r[1] in sums:          # accu of this matrix already on the device (runtime sum cache)
                rt.remember_sum(b, sums.pop(r[1]))
        else:   # a leaf or a duplicate: a copy, like evaluate(leaf)
            src = b if r[0] == "dup" else b.mem
            m = Matrix._uninitialised(shape.rows, shape.cols, node.elem_type)
            rt.copy_d2d(src, m.mem, shape.n_elem)
            result.append(m)
    for buf in sums.values():
        rt.release_deferred(buf)
    return result


def reduce_value(op: str, *xs):
    """Run a fused scalar reduction and return the numpy scalar."""
    if _RECIPES_ON:
        nodes = [as_expr(x) for x in xs]
        key, leaves = _dag_key(nodes)
        if key is not None:
            rec, p = _recipe_for(("reduce", op, key), leaves, lambda: (plan_reduce(op, *nodes), None))
            if rec is not None:
                return execute_plan(rec.plan, leaves=leaves, recipe=rec)
            return execute_plan(p)
    return execute_plan(plan_reduce(op, *xs))
