"""Host-side planner behaviour (no device): plan shapes, fusion, transpose
folding, fused reductions, and NVRTC compilation of the emitted programs."""
import ctypes
import itertools

import numpy as np
import pytest

import paper_2308_03120_b200 as dm
from paper_2308_03120_b200 import _clib, expr, kernels
from paper_2308_03120_b200.runtime import DeviceBuffer, FlatView, KernelInvocation, build_invocation

_ids = itertools.count(1)


class FakeMatrix:
    """Stands in for a device matrix: planning never touches memory."""

    def __init__(self, rows, cols, elem="f32"):
        self.n_rows, self.n_cols, self.elem_type = rows, cols, elem
        bid = next(_ids)
        self.mem = DeviceBuffer(0, bid, rows * cols, elem, 0x7f0000000000 + bid * 0x10000000)

    @property
    def n_elem(self):
        return self.n_rows * self.n_cols

    def _as_expr_node(self):
        return expr.ExprNode("leaf", (self,), (), self.elem_type)


def leaf(r, c, elem="f32"):
    return FakeMatrix(r, c, elem)._as_expr_node()


def test_config1_tree_is_one_fused_kernel():
    A, B, C, D = (leaf(64, 64) for _ in range(4))
    node = 2 * A + B % C - dm.exp(D)
    p = dm.plan(node)
    assert p.n_invocations == 1
    assert p.steps[0].kernel == "fused_chain"
    assert p.steps[0].params["program"] == (
        ("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1), ("load", 2), ("glue", "eglue_schur"),
        ("glue", "eglue_plus"), ("load", 3), ("unary", "eop_exp", None), ("glue", "eglue_minus"))


def test_percent_and_star_are_schur():
    A, B = leaf(3, 3), leaf(3, 3)
    assert (A % B).kind == "eglue_schur"
    assert (A * B).kind == "eglue_schur"
    assert (A @ B).kind == "glue_times"


def test_deep_chains_fuse_beyond_reference_cap():
    node = leaf(4, 4)
    for i in range(20):
        node = dm.build_node("eop_scalar_plus", (node,), (i,))
    assert dm.plan(node).n_invocations == 1
    # reference plan shape on request (tests/test_integration.py:83-88: 8 + 8 + 4)
    assert dm.plan(node, chain_max=kernels.REFERENCE_CHAIN_MAX).n_invocations == 3


def test_input_limit_splits_wide_trees():
    leaves = [leaf(8, 8) for _ in range(40)]
    node = leaves[0]
    for x in leaves[1:]:
        node = node + x
    p = dm.plan(node)
    for s in p.steps:
        assert len(s.inputs) <= kernels.FUSED_INPUTS_MAX
        if s.kernel == "fused_chain":
            assert len(s.params["program"]) <= 64


def test_nt_gemm_has_no_transpose_pass():
    A, B = leaf(32, 16), leaf(24, 16)
    p = dm.plan(A @ B.t())
    assert [s.kernel for s in p.steps] == ["gemm"]
    assert p.steps[0].params == {"trans_a": 0, "trans_b": 1}
    p = dm.plan(A.t() @ leaf(32, 5))
    assert p.steps[0].params["trans_a"] == 1


def test_gemm_with_elementwise_operands_takes_three():
    a, b = leaf(4, 4), leaf(4, 4)
    assert dm.plan((2 * a + 1) @ (b - 3)).n_invocations == 3


def test_conv_over_product_stays_standalone():
    a = leaf(4, 4)
    p = dm.plan(dm.conv_to(a @ a, "f64"))
    assert [s.kernel for s in p.steps] == ["gemm", "mov_copy"]


def test_conv_of_leaf_folds_into_chain_load():
    ints = leaf(2, 2, "i32")
    p = dm.plan(dm.exp(dm.conv_to(ints, "f32")) + 1)
    assert p.n_invocations == 1
    assert p.steps[0].inputs[0][1].elem_type == "i32"


def test_shared_leaf_loaded_once():
    a = leaf(6, 6)
    shared = 2 * a + 1
    p = dm.plan((shared + shared) - shared)
    assert len(p.steps[0].inputs) == 1


def test_fused_reduction_plans():
    A, B, C, D = (leaf(64, 64) for _ in range(4))
    p = dm.plan_reduce("accu", 2 * A + B % C - dm.exp(D))
    assert p.steps == [] and p.reduce.kernel == "fused_reduce"
    assert len(p.reduce.inputs) == 4
    x = leaf(100, 1)
    p = dm.plan_reduce("dot", x, x)
    assert len(p.reduce.inputs) == 1
    assert p.reduce.params["program"] == (("load", 0), ("load", 0))
    p = dm.plan_reduce("accu", leaf(3, 3) @ leaf(3, 3))
    assert [s.kernel for s in p.steps] == ["gemm"] and p.n_invocations == 2


def test_temp_schedule_releases_after_last_use():
    a, b = leaf(4, 4), leaf(4, 4)
    p = dm.plan((2 * a + 1) @ (b - 3))
    final = p.result[1]
    for slot, (born, dies) in p.temp_schedule.items():
        if slot != final:
            assert dies is not None and dies > born
        else:
            assert dies is None


def test_shape_and_type_errors():
    with pytest.raises(dm.DimensionError) as e:
        dm.build_node("eglue_plus", (leaf(2, 3), leaf(3, 2)))
    assert "eglue_plus" in str(e.value) and "2x3" in str(e.value) and "3x2" in str(e.value)
    with pytest.raises(dm.DimensionError):
        dm.build_node("glue_times", (leaf(2, 3), leaf(2, 5)))
    with pytest.raises(dm.ElemTypeError):
        dm.build_node("eglue_plus", (leaf(2, 2, "f32"), leaf(2, 2, "i32")))
    with pytest.raises(ValueError):
        dm.build_node("op_sum_dim", (leaf(2, 2),), (2,))


def test_rewrites():
    a = leaf(3, 4)
    assert dm.trans(dm.trans(a)) is a
    v = leaf(5, 1)
    d = dm.diagmat(v)
    assert dm.trans(d) is d
    n = 2 * (3 * a)
    assert n.kind == "eop_scalar_times" and n.aux[0] == 6 and n.operands[0] is a


# ---- NVRTC compilation of emitted programs (no GPU needed) ---------------------------------------

def _compile(kind, views, out, params, scalars=()):
    inv = build_invocation(KernelInvocation(kind, tuple(views), out, scalars, params))
    rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
    assert rc == 0, _clib.last_error()


def _flat(m, count=None, stride=1, offset=0):
    return FlatView(m.mem, offset, m.n_elem if count is None else count, stride)


@pytest.mark.parametrize("elem", ["f32", "f64", "i32", "u64"])
def test_programs_compile_for_every_type(elem):
    A, B = FakeMatrix(16, 16, elem), FakeMatrix(16, 16, elem)
    out = FakeMatrix(16, 16, elem)
    prog = (("load", 0), ("scalar", "eop_scalar_times", 3), ("load", 1), ("glue", "eglue_div"),
            ("unary", "eop_abs", None), ("unary", "eop_sqrt", None), ("scalar", "eop_scalar_div_pre", 2))
    params = {"program": prog, "compute_dtype": kernels.NP_DTYPE[elem].str}
    _compile("fused_chain", [_flat(A), _flat(B)], _flat(out), params)
    for op in ("accu", "min", "max"):
        _compile("fused_reduce", [_flat(A), _flat(B)], None, dict(params, op=op))
    dot = {"program": (("load", 0), ("load", 1)), "compute_dtype": kernels.NP_DTYPE[elem].str, "op": "dot"}
    _compile("fused_reduce", [_flat(A), _flat(B)], None, dot)


def test_all_unary_ops_compile():
    A, out = FakeMatrix(8, 8), FakeMatrix(8, 8, "f64")
    prog = [("load", 0)] + [("unary", op, 2 if op == "eop_pow" else None) for op in kernels.EOP_UNARY]
    _compile("fused_chain", [_flat(A)], _flat(out), {"program": tuple(prog), "compute_dtype": "<f4"})


def test_strided_and_converted_inputs_compile():
    A, Bi, out = FakeMatrix(10, 10), FakeMatrix(10, 10, "i32"), FakeMatrix(50, 1, "u64")
    prog = (("load", 0), ("load", 1), ("glue", "eglue_plus"))
    _compile("fused_chain", [_flat(A, 50, 2), _flat(Bi, 50, 2, 1)], _flat(out, 50), {"program": prog,
                                                                                      "compute_dtype": "<f4"})



def test_planning_leaves_no_reference_cycles():
    """Plans must not keep operands alive until a GC pass: device matrices
    are released by reference counting (a cycle here made every e2e step
    allocate fresh pool memory)."""
    import gc
    gc.collect()
    gc.set_debug(gc.DEBUG_SAVEALL)
    try:
        e = 2 * leaf(64, 64) + leaf(64, 64) % leaf(64, 64) - dm.exp(leaf(64, 64))
        p = expr.plan_reduce("accu", e)
        del p
        p = expr.plan(e)
        del p, e
        g = leaf(64, 64) @ leaf(64, 64).t()
        p = expr.plan(g)
        del p, g
        # the fused paths' pattern matchers (logistic step, GEMM prologue, dim reductions)
        X, w, y = leaf(4096, 1024), leaf(1024, 1), leaf(4096, 1)
        r = 1 / (1 + dm.exp(0 - X @ w)) - y
        p = expr.plan(X.t() @ r)
        del p, r, X, w, y
        a, b = leaf(256, 256), leaf(256, 256)
        p = expr.plan((2 * a + 1) @ (b - 3).t())
        q = expr.plan(dm.sum(2 * a + b, 1))
        del p, q, a, b
        assert gc.collect() == 0, [type(o).__name__ for o in gc.garbage][:20]
    finally:
        gc.set_debug(0)
        gc.garbage.clear()


# ---- fused single-pass logistic step ------------------------------------------

def _logistic_parts(m=4096, k=1024):
    X, w, y = FakeMatrix(m, k), FakeMatrix(k, 1), FakeMatrix(m, 1)
    xn, wn, yn = X._as_expr_node(), w._as_expr_node(), y._as_expr_node()
    r = 1 / (1 + dm.exp(0 - xn @ wn)) - yn
    return X, w, y, xn, r


def test_logistic_gradient_is_one_fused_step():
    X, w, y, xn, r = _logistic_parts()
    p = expr.plan(xn.t() @ r)
    assert [s.kernel for s in p.steps] == ["logistic_grad"]
    st = p.steps[0]
    assert st.inputs[0] == ("leaf", X) and st.inputs[1] == ("leaf", w) and st.inputs[3] == ("leaf", y)
    assert st.params["program"][0] == ("load", 0)            # X @ w is program input 0
    r_slot = st.inputs[2][1]
    a_slot = st.params["accu_slot"]                            # accu(r) side output (1 x 1 f32)
    assert st.params["alloc_slots"] == (r_slot, a_slot)
    assert p.sums == ((r_slot, a_slot),)
    assert (p.slots[a_slot].rows, p.slots[a_slot].cols, p.slots[a_slot].elem_type) == (1, 1, "f32")
    assert p.temp_schedule[r_slot] == (0, 0)                   # r is released after the step
    # beyond 2^26 rows (8192 blocks of 8192) the kernel has no room to fold accu(r)
    X, w, y, xn, r = _logistic_parts(m=(1 << 26) + 8)
    st = expr.plan(xn.t() @ r).steps[0]
    assert st.kernel == "logistic_grad" and "accu_slot" not in st.params and len(st.params["alloc_slots"]) == 1


def test_logistic_fusion_declines_other_shapes():
    X, w, y, xn, r = _logistic_parts(m=4098)                   # rows not a multiple of 4
    assert [s.kernel for s in expr.plan(xn.t() @ r).steps] != ["logistic_grad"]
    X, w, y, xn, r = _logistic_parts(k=4100)                   # too many columns (clusters of 8 x 512)
    assert "logistic_grad" not in [s.kernel for s in expr.plan(xn.t() @ r).steps]
    X2 = FakeMatrix(4096, 1024)._as_expr_node()                # a different X in the product
    w = FakeMatrix(1024, 1)._as_expr_node()
    r2 = 1 / (1 + dm.exp(0 - X2 @ w))
    assert "logistic_grad" not in [s.kernel for s in expr.plan(xn.t() @ r2).steps]


@pytest.mark.parametrize("k", [1024, 2000, 4096])
def test_logistic_kernel_compiles(k):
    X, w, y, xn, r = _logistic_parts(k=k)                      # CTA pairs; clusters of 4 and 8 past 1024
    p = expr.plan(xn.t() @ r)
    st = p.steps[0]
    assert st.kernel == "logistic_grad"
    fake_r = FakeMatrix(4096, 1)
    views = [expr._make_view(X.mem, 4096, k, "2d"), expr._make_view(w.mem, k, 1, "flat"),
             expr._make_view(fake_r.mem, 4096, 1, "flat"), expr._make_view(y.mem, 4096, 1, "flat")]
    g = FakeMatrix(k, 1)
    inv = build_invocation(KernelInvocation("logistic_grad", tuple(views), _flat(g), (), st.params))
    rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
    assert rc == 0, _clib.last_error()


def test_f64_operand_chains_fuse_into_the_dmma_producer(monkeypatch):
    a, b, c = leaf(256, 256, "f64"), leaf(256, 256, "f64"), leaf(256, 256, "f64")
    assert "gemm_fused" not in [s.kernel for s in dm.plan((2 * a + 1) @ (b - 3).t()).steps]   # off by default
    monkeypatch.setattr(expr, "_F64_PROLOGUE", True)
    p = dm.plan((2 * a + 1) @ (b - 3).t())
    assert [s.kernel for s in p.steps] == ["gemm_fused"]
    st = p.steps[0]
    assert st.params["na"] == 1 and st.params["trans_b"] == 1
    out = FakeMatrix(256, 256, "f64")
    views = [_flat(a.operands[0]), _flat(b.operands[0])]
    inv = build_invocation(KernelInvocation("gemm_fused", tuple(views), _flat(out), (), st.params))
    assert inv.compute_dtype == _clib.BM_F64
    rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
    assert rc == 0, _clib.last_error()
    # more than three program inputs in all: the operands are materialised (register budget)
    assert "gemm_fused" not in [s.kernel for s in dm.plan((a % c + a) @ (b % c - b)).steps]


# ---- GEMM epilogue fusion ------------------------------------------------------

@pytest.mark.parametrize("elem", ["f32", "f64"])
def test_gemm_epilogue_fuses_the_consuming_chain(elem):
    a, b, c = leaf(256, 256, elem), leaf(256, 256, elem), leaf(256, 256, elem)
    prod = a @ b.t()
    e = dm.exp(2 * prod) - prod % prod / 3
    p = dm.plan(e)
    assert [s.kernel for s in p.steps] == ["gemm_epi"]
    st = p.steps[0]
    assert st.inputs[0] == ("leaf", a.operands[0]) and st.inputs[1] == ("leaf", b.operands[0])
    assert len(st.inputs) == 2
    assert st.params["trans_a"] == 0 and st.params["trans_b"] == 1
    assert st.params["program"][:2] == (("load", 0), ("scalar", "eop_scalar_times", 2))
    # a tree that also reads one m x n matrix fuses for f32 (staged through shared memory),
    # keeps the reference's plan for f64 and for two extra matrices (measured slower fused)
    kinds = [s.kernel for s in dm.plan(dm.exp(2 * prod) + c).steps]
    assert kinds == (["gemm_epi"] if elem == "f32" else ["gemm", "fused_chain"])
    d = leaf(256, 256, elem)
    assert "gemm_epi" not in [s.kernel for s in dm.plan(prod + c + d).steps]
    # the kernel compiles (NVRTC, sm_100a): 3xTF32 pair kernel / DMMA with the program in the store
    views = [expr._make_view(x.operands[0].mem, 256, 256, "2d") for x in (a, b)]
    out = FakeMatrix(256, 256, elem)
    inv = build_invocation(KernelInvocation("gemm_epi", tuple(views), _flat(out), (), st.params))
    rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
    assert rc == 0, _clib.last_error()


def test_gemm_epilogue_declines():
    a, b = leaf(256, 256), leaf(256, 256)
    assert "gemm_epi" not in [s.kernel for s in dm.plan(2 * (leaf(8, 8) @ leaf(8, 8))).steps]   # small: SIMT + chain
    v = leaf(256, 1)
    assert "gemm_epi" not in [s.kernel for s in dm.plan(2 * (a @ v)).steps]                    # GEMV
    assert "gemm_epi" not in [s.kernel for s in dm.plan((a @ b) + (b @ a)).steps]               # two products
    ai = leaf(256, 256, "i32")
    assert "gemm_epi" not in [s.kernel for s in dm.plan(2 * (ai @ ai)).steps]                   # integer GEMM
    assert "gemm_epi" not in [s.kernel for s in dm.plan(2 * (a @ b), fuse=False).steps]


# ---- GEMM prologue fusion ------------------------------------------------------

def test_gemm_operand_chains_fuse_into_the_split_pass():
    a, b = leaf(256, 256), leaf(256, 256)
    p = dm.plan((2 * a + 1) @ (b - 3).t())
    assert [s.kernel for s in p.steps] == ["gemm_fused"]
    st = p.steps[0]
    assert st.params["na"] == 1 and st.params["trans_b"] == 1
    assert st.params["a_prog"][0] == ("load", 0) and st.params["b_prog"][0] == ("load", 0)
    # one chained operand and one plain leaf
    p = dm.plan((2 * a + 1) @ b)
    assert [s.kernel for s in p.steps] == ["gemm_fused"]
    # small and vector shapes keep the reference's lowering
    assert dm.plan((2 * leaf(4, 4) + 1) @ (leaf(4, 4) - 3)).n_invocations == 3
    v = leaf(256, 1)
    assert "gemm_fused" not in [s.kernel for s in dm.plan((2 * a + 1) @ v).steps]


def test_gemm_split_kernel_compiles():
    A, B, C = FakeMatrix(256, 256), FakeMatrix(256, 256), FakeMatrix(256, 256)
    an, bn = A._as_expr_node(), B._as_expr_node()
    p = dm.plan(dm.exp(an) * 0.5 @ (bn - 3))
    st = p.steps[0]
    views = [expr._make_view(A.mem, 256, 256, "flat"), expr._make_view(B.mem, 256, 256, "flat")]
    inv = build_invocation(KernelInvocation("gemm_fused", tuple(views), expr._make_view(C.mem, 256, 256, "2d"), (),
                                            st.params))
    assert inv.kind == _clib.BM_K_GEMM_FUSED and inv.iparams[0] == 1


# ---- dim-0 reductions over element-wise trees ----------------------------------

def test_dim0_reduction_of_a_tree_is_one_fused_step():
    a, b = leaf(512, 40), leaf(512, 40)
    for op, kern in (("sum", "rdim_sum"), ("mean", "rdim_mean"), ("min", "rdim_min"), ("max", "rdim_max")):
        p = dm.plan(getattr(dm, op)(2 * a + b, 0))
        assert [s.kernel for s in p.steps] == ["fused_rdim"], op
        st = p.steps[0]
        assert st.params["op"] == kern and st.params["rows"] == 512
        assert st.params["program"] == (("load", 0), ("scalar", "eop_scalar_times", 2), ("load", 1),
                                        ("glue", "eglue_plus"))
    # dim 1 too, with TMA-compatible rows; a leaf, numpy's lone-row block, var/stddev and
    # empty shapes keep the reference's lowering
    p1 = dm.plan(dm.sum(2 * a + b, 1))
    assert [s.kernel for s in p1.steps] == ["fused_rdim"] and p1.steps[0].params["dim"] == 1
    assert p1.steps[0].params["cols"] == 40
    assert [s.kernel for s in dm.plan(dm.sum(a, 0)).steps] == ["rdim_sum"]
    lone = leaf(65, 8)
    assert [s.kernel for s in dm.plan(dm.sum(2 * lone + 1, 1)).steps] == ["fused_chain", "rdim_sum"]
    odd = leaf(6, 8)                                            # 24-B columns: no TMA
    assert [s.kernel for s in dm.plan(dm.sum(2 * odd + 1, 1)).steps] == ["fused_chain", "rdim_sum"]
    assert [s.kernel for s in dm.plan(dm.var(2 * a + b, 0)).steps] == ["fused_rdim"]
    assert [s.kernel for s in dm.plan(dm.stddev(2 * a + b, 1)).steps] == ["fused_rdim", "eop_sqrt"]
    assert [s.kernel for s in dm.plan(dm.sum(2 * leaf(0, 5) + 1, 0)).steps] != ["fused_rdim"]


@pytest.mark.parametrize("dim", [0, 1])
def test_fused_dim_kernels_compile(dim):
    for elem in ("f32", "f64", "i32"):
        a, b = leaf(512, 40, elem), leaf(512, 40, elem)
        for op in ("sum", "mean", "min", "max", "var"):
            p = dm.plan(getattr(dm, op)(a * b + 3, dim))
            st = p.steps[0]
            views = [expr._make_view(r[1].mem, 512, 40, "flat") for r in st.inputs]
            out = FakeMatrix(1, 40, elem) if dim == 0 else FakeMatrix(512, 1, elem)
            inv = build_invocation(KernelInvocation("fused_rdim", tuple(views), _flat(out), (), st.params))
            rc = _clib.lib().bm_jit_compile_only(ctypes.byref(inv))
            assert rc == 0, _clib.last_error()
