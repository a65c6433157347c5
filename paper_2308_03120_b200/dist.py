"""Column-block sharding over the GPUs of one box.

One process per GPU (torchrun); torch.distributed over NCCL is plumbing
only: it carries one partial per rank.  Element-wise work on a column block
needs no communication.  A scalar reduction is computed per shard to one
partial (the fused kernel writes it straight into a device slot), the
partials are all-gathered in rank order and folded on the device with the
reference's combine_pairwise (kernels.py:380-392).  When every shard is an
aligned power-of-two run of REDUCE_BLOCK-element blocks (e.g. 4096x4096 f32
per GPU), the result is bit-identical to the single-device reduction of the
concatenated matrix; otherwise it is still deterministic for a given world
size.  No float atomics, no NCCL sum whose order NCCL chooses.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _clib, kernels
from . import expr as _expr
from . import runtime as _rt

_TORCH_DTYPE = {"f32": "float32", "f64": "float64", "i32": "int32", "u64": "uint64"}


def column_block(total_cols: int, rank: int, world: int) -> tuple[int, int]:
    """[start, start+count) of the columns rank `rank` owns: contiguous,
    balanced, in rank order (column-major => each block is contiguous)."""
    base, extra = divmod(total_cols, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def bind_torch_stream():
    """Make one CUDA stream current for both torch and the device library, so
    NCCL collectives issued by torch.distributed and torch.cuda.Event timing
    are stream-ordered with the library's kernels.  Returns the stream."""
    import torch
    rt = _rt.get_runtime()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    _clib.check(rt._lib.bm_set_stream(ctypes.c_void_p(s.cuda_stream)), "bind stream")
    return s


def partial_dtype(op: str, elem: str) -> str:
    """Element type of one rank's partial (dot partials of floats are f64)."""
    return "f64" if op == "dot" and elem in ("f32", "f64") else elem


class ShardedReduction:
    """A scalar reduction over column-block shards, reusable across steps.

    ``prepare`` plans the fused kernel once; ``launch`` enqueues this rank's
    partial, the all-gather and the device-side fold without any host
    synchronisation; ``value`` reads the folded result back.
    """

    def __init__(self, op: str, *local_exprs, group=None):
        import torch
        import torch.distributed as dist
        self.op = op
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.plan = _expr.plan_reduce(op, *local_exprs)
        if self.plan.steps:
            raise ValueError("sharded reduction expects a purely element-wise local program")
        node = _expr.as_expr(local_exprs[0])
        self.elem = node.elem_type
        self.pdt = partial_dtype(op, self.elem)
        tdt = getattr(torch, _TORCH_DTYPE[self.pdt])
        self.partial = torch.zeros(1, dtype=tdt, device="cuda")
        self.gathered = torch.zeros(self.world, dtype=tdt, device="cuda")
        self.result = torch.zeros(1, dtype=tdt, device="cuda")
        views = _expr._step_views(self.plan, self.plan.reduce, {})
        self.inv = _rt.build_invocation(_rt.KernelInvocation("fused_reduce", tuple(views), None, (),
                                                             dict(self.plan.reduce.params)))
        self._lib = _clib.lib()
        self._op_code = {"accu": _clib.BM_R_ACCU, "min": _clib.BM_R_MIN, "max": _clib.BM_R_MAX,
                         "dot": _clib.BM_R_DOT}[op]

    def launch(self) -> None:
        _clib.check(self._lib.bm_reduce_to_device(ctypes.byref(self.inv), ctypes.c_void_p(self.partial.data_ptr())),
                    "sharded reduce")
        if self.world == 1:
            return
        self.dist.all_gather_into_tensor(self.gathered, self.partial, group=self.group)
        _clib.check(self._lib.bm_combine_partials_to_device(
            ctypes.c_void_p(self.gathered.data_ptr()), self.world, _clib.DTYPE_CODE[self.elem], self._op_code,
            ctypes.c_void_p(self.result.data_ptr())), "combine partials")

    def value(self):
        import torch
        torch.cuda.synchronize()
        src = self.partial if self.world == 1 else self.result
        v = src.cpu().numpy()[0]
        dt = kernels.NP_DTYPE[self.elem]
        if self.op == "dot" and dt.kind == "f":
            return dt.type(v)
        return np.asarray(v).astype(dt)[()]


def sharded_accu(local_expr, group=None):
    """accu over a column-block-sharded expression (all ranks call)."""
    r = ShardedReduction("accu", local_expr, group=group)
    r.launch()
    return r.value().item()


def sharded_dot(a_local, b_local, group=None):
    r = ShardedReduction("dot", a_local, b_local, group=group)
    r.launch()
    return r.value().item()


# ---------------------------------------------------------------------------
# device buffers as torch tensors (zero copy), for the collectives only

class _CudaArray:
    """__cuda_array_interface__ over a device buffer (column-major flat)."""

    def __init__(self, ptr: int, count: int, elem: str):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": kernels.NP_DTYPE[elem].str, "data": (ptr, False),
            "version": 3, "strides": None, "stream": None}


def torch_view(m):
    """The column-major storage of a device matrix as a flat torch tensor
    sharing its memory (no copy): what NCCL reads and writes."""
    import torch
    return torch.as_tensor(_CudaArray(m.mem.ptr, m.n_elem, m.elem_type), device="cuda")


def _world(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def broadcast_matrix(m, src: int = 0, group=None):
    """Replicate a device matrix from rank `src` (config 4: A of A*B^T)."""
    import torch.distributed as dist
    if _world(group)[1] > 1:
        dist.broadcast(torch_view(m), src, group=group)
    return m


def gather_columns(local, group=None):
    """All-gather one rows x 1 partial per rank into a rows x world matrix,
    column r = rank r's partial (column-major: a column is contiguous, so the
    NCCL all-gather writes each rank's block in place)."""
    import torch.distributed as dist
    from .matrix import Matrix
    rank, world = _world(group)
    if world == 1:
        return local
    out = Matrix(local.n_elem, world, elem_type=local.elem_type)
    dist.all_gather_into_tensor(torch_view(out), torch_view(local), group=group)
    return out


def sharded_reduce_dim(op: str, local_expr, dim: int, group=None):
    """sum/min/max along `dim` of a column-block-sharded matrix.

    dim 0 (one value per column): every rank owns its columns' results, no
    communication.  dim 1 (one value per row): each rank reduces its columns
    to a rows x 1 partial, the partials are all-gathered in rank order and
    folded with the same device reduction along dim 1 -- a left-to-right fold
    0 + p_0 + p_1 + ..., deterministic for a given world size (min/max are
    exact).  Returns the local dim-0 block or the full dim-1 column."""
    from . import ops
    fn = {"sum": ops.sum, "min": ops.min, "max": ops.max}[op]
    local = _expr.evaluate(fn(local_expr, dim))
    if dim == 0 or _world(group)[1] == 1:
        return local
    return _expr.evaluate(fn(gather_columns(local, group), 1))


def sharded_gemm_nt(a, b_local):
    """C = A * B^T sharded over the rows of B (= the columns of C): rank r
    holds B's row block r and A replicated (broadcast_matrix), and computes
    its column block of C with no communication."""
    return _expr.evaluate(a @ b_local.t())


def sharded_logistic_step(x_local, w, y_local, group=None):
    """One logistic-regression gradient step sharded by samples (row blocks
    of X): z = X_r w, r = 1/(1+exp(-z)) - y_r,
    g = sum_r X_r^T r_r (one all-gather of a 1024-vector, folded in rank
    order) and s = accu(r) over all ranks.  Returns (g, s)."""
    from . import ops
    z = _expr.evaluate(x_local @ w)
    r = _expr.evaluate(1 / (1 + ops.exp(0 - z)) - y_local)
    g_local = _expr.evaluate(x_local.t() @ r)
    if _world(group)[1] == 1:
        return g_local, ops.accu(r)
    g = _expr.evaluate(ops.sum(gather_columns(g_local, group), 1))
    s = ShardedReduction("accu", r, group=group)
    s.launch()
    return g, s.value().item()
