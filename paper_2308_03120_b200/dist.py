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
import os

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


class PeerExchange:
    """Exchange buffers of every rank mapped into this process (CUDA IPC): the
    peer-memory replacement of the all-gather + fold in ShardedReduction
    (b200mat.h bm_exchange_*).  One kernel writes this rank's partial into
    every rank's buffer over NVLink, publishes a step epoch with release
    semantics, waits for all epochs and folds in rank order."""

    def __init__(self, group=None, nvals=None):
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nvals = nvals                  # None: one value per rank; else the slot capacity in 4-byte units
        self._lib = _clib.lib()
        self._own = None
        self._opened = []
        self.epoch = 0

        def agree(ok: bool) -> bool:          # every rank learns whether every rank succeeded
            t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            return bool(t.item())

        handle = ctypes.create_string_buffer(64)
        ok = True
        try:
            own = ctypes.c_void_p()
            if nvals is None:
                _clib.check(self._lib.bm_exchange_alloc(self.world, ctypes.byref(own), handle), "exchange alloc")
            else:
                _clib.check(self._lib.bm_exchange_alloc_vec(self.world, nvals, ctypes.byref(own), handle),
                            "exchange alloc")
            self._own = own.value
        except Exception:  # noqa: BLE001 - reported collectively below
            ok = False
        if not agree(ok):
            self.close()
            raise RuntimeError("peer exchange: buffer allocation failed on some rank")
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        ptrs = []
        ok = True
        try:
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self._own)
                    continue
                p = ctypes.c_void_p()
                _clib.check(self._lib.bm_exchange_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)),
                            "exchange open")
                ptrs.append(p.value)
                self._opened.append(p.value)
        except Exception:  # noqa: BLE001
            ok = False
        if not agree(ok):                   # every rank mapped every buffer, or nobody uses them
            self.close()
            raise RuntimeError("peer exchange: mapping a peer buffer failed on some rank")
        self._ptrs = (ctypes.c_void_p * self.world)(*ptrs)
        self.dev_ptrs = torch.tensor(ptrs, dtype=torch.int64, device="cuda")   # for the fused kernel
        # the fused kernel reads dev_ptrs on the library's stream, which need not be
        # torch's current stream: finish the host-to-device copy first
        torch.cuda.current_stream().synchronize()
        self.broken = False

    def combine(self, partial, elem: str, op_code: int, result) -> None:
        self.epoch += 1
        _clib.check(self._lib.bm_exchange_combine(
            ctypes.c_void_p(partial.data_ptr()), self._ptrs, self.world, self.rank, self.epoch,
            _clib.DTYPE_CODE[elem], op_code, ctypes.c_void_p(result.data_ptr())), "exchange combine")

    def gsum(self, g_ptr: int, n: int, s_ptr: int, g_out_ptr: int, s_out_ptr: int) -> None:
        """Vector buffers only: g_out = sum over ranks of g (n f32, rank order) and
        s_out = combine_pairwise of the ranks' s, in one kernel (bm_exchange_gsum)."""
        if self.nvals is None or n > self.nvals:
            raise ValueError("gsum needs a vector exchange of at least n values")
        self.epoch += 1
        _clib.check(self._lib.bm_exchange_gsum(
            ctypes.c_void_p(g_ptr), n, ctypes.c_void_p(s_ptr), self._ptrs, self.world, self.rank, self.epoch,
            self.nvals, ctypes.c_void_p(g_out_ptr), ctypes.c_void_p(s_out_ptr)), "exchange gsum")

    def rows(self, x_ptr: int, n: int, elem: str, op_code: int, out_ptr: int) -> None:
        """Vector buffers only: out = the rank-order fold (sum / min / max) of every
        rank's n-vector, in one kernel (bm_exchange_rows)."""
        if self.nvals is None or n * kernels.itemsize(elem) > 4 * self.nvals:
            raise ValueError("rows needs a vector exchange with room for n values")
        self.epoch += 1
        _clib.check(self._lib.bm_exchange_rows(
            ctypes.c_void_p(x_ptr), n, _clib.DTYPE_CODE[elem], op_code, self._ptrs, self.world, self.rank,
            self.epoch, self.nvals, ctypes.c_void_p(out_ptr)), "exchange rows")

    def reduce(self, inv, result) -> None:
        """The shard reduction and the exchange in one kernel
        (bm_reduce_to_device_exchange): the folded world value lands in result."""
        self.epoch += 1
        _clib.check(self._lib.bm_reduce_to_device_exchange(
            ctypes.byref(inv), ctypes.c_void_p(result.data_ptr()), ctypes.c_void_p(self.dev_ptrs.data_ptr()),
            self.world, self.rank, self.epoch), "fused reduce + exchange")

    def close(self) -> None:
        for p in self._opened:
            self._lib.bm_exchange_close(ctypes.c_void_p(p), 1)
        self._opened = []
        if self._own:
            self._lib.bm_exchange_close(ctypes.c_void_p(self._own), 0)
            self._own = None


# group -> PeerExchange (or None when peer mapping failed somewhere).  Entries
# hold the group object itself, so an id() is never reused for another group;
# runtime.shutdown() forgets them (their pointers die with the library state).
_SHARED_EXCHANGES: dict = {}


def shared_exchange(group=None):
    """The process's PeerExchange for `group`, created once (collectively) and
    reused by every sharded reduction that exchanges over peer memory, whose
    epochs then advance in the same order on every rank; None when peer
    mapping is unavailable anywhere (then the NCCL all-gather serves) or the
    exchange timed out earlier (BM_ERR_PEER: it is no longer in step)."""
    key = id(group)
    ent = _SHARED_EXCHANGES.get(key)
    if ent is None or ent[0] is not group:
        try:
            ex = PeerExchange(group)
        except RuntimeError:
            ex = None
        ent = (group, ex)
        _SHARED_EXCHANGES[key] = ent
    ex = ent[1]
    return None if ex is None or ex.broken else ex


def shared_vec_exchange(nvals: int, group=None):
    """The process's vector PeerExchange for `group` with room for `nvals` values
    (created once, collectively; None when peer mapping is unavailable anywhere
    or an exchange timed out).  Shares the registry (and its teardown) with
    shared_exchange."""
    key = (id(group), "vec", nvals)
    ent = _SHARED_EXCHANGES.get(key)
    if ent is None or ent[0] is not group:
        try:
            ex = PeerExchange(group, nvals=nvals)
        except RuntimeError:
            ex = None
        ent = (group, ex)
        _SHARED_EXCHANGES[key] = ent
    ex = ent[1]
    return None if ex is None or ex.broken else ex


def close_exchanges() -> None:
    """Collective: unmap every peer buffer, wait for all ranks, free the own
    buffers.  Call on every rank before destroying the process group."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    ents = list(_SHARED_EXCHANGES.values())
    _SHARED_EXCHANGES.clear()
    for group, ex in ents:
        if ex is not None:
            for q in ex._opened:
                ex._lib.bm_exchange_close(ctypes.c_void_p(q), 1)
            ex._opened = []
    for group, ex in ents:
        if ex is not None:
            dist.barrier(group=group)      # no peer maps this rank's buffer any more
            ex.close()


def _forget_exchanges() -> None:
    """runtime.shutdown hook (not collective): unmap peer buffers and drop
    every entry, so no stale device pointer is reused after a re-init.  The
    own buffers are left to the process (a peer may still map them)."""
    for _, ex in list(_SHARED_EXCHANGES.values()):
        if ex is not None:
            for q in ex._opened:
                ex._lib.bm_exchange_close(ctypes.c_void_p(q), 1)
            ex._opened = []
            ex._own = None
    _SHARED_EXCHANGES.clear()


_rt._shutdown_hooks.append(_forget_exchanges)


def _agree_all(group, flag: bool) -> bool:
    """Collective AND of a per-rank flag."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


class ShardedReduction:
    """A scalar reduction over column-block shards, reusable across steps.

    The constructor plans the fused kernel once; ``launch`` enqueues this
    rank's partial, the all-gather and the device-side fold without any host
    synchronisation; ``value`` reads the folded result back.

    With more than one rank, consecutive steps are software-pipelined: the
    partial of step k goes to a side stream that runs the all-gather and the
    fold, while the compute stream goes on with step k + 1.  Partials,
    gathered vectors and results are double-buffered by step parity, and step
    k + 2 waits for the gather that read its partial buffer, so a step costs
    max(kernel, collective) instead of their sum.  ``join`` orders the current
    stream after every collective issued so far (timing, value).
    ``collective="allreduce"`` gathers by summing rank-slotted vectors (for
    backends without all-gather of device tensors, e.g. gloo in tests);
    ``collective="p2p"`` replaces the all-gather and the fold with one kernel
    over peer memory (PeerExchange); ``"p2p_fused"`` moves that exchange into
    the reduction kernel itself (its last CTA publishes, waits and folds).
    """

    def __init__(self, op: str, *local_exprs, group=None, pipeline=None, collective=None):
        import torch
        import torch.distributed as dist
        self.op = op
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = _expr.plan_reduce(op, *local_exprs)
        if self.plan.steps:
            raise ValueError("sharded reduction expects a purely element-wise local program")
        if collective is None:
            collective = os.environ.get("BM_SHARD_COLLECTIVE", "p2p_fused")
        if collective not in ("all_gather", "allreduce", "p2p", "p2p_fused"):
            raise ValueError(f"unknown collective {collective!r}")
        node = _expr.as_expr(local_exprs[0])
        # Shard sizes, once: an empty shard of a min / max has no partial, so
        # the fold skips it (the peer-memory paths cannot: they fall back to
        # the gather); every shard empty is the reference's empty-range error.
        shp = _expr.shape_of(node)
        n_local = int(shp.rows) * int(shp.cols)
        self.counts = [n_local]
        self._fold_ranks = None
        if self.world > 1:
            counts = [None] * self.world
            dist.all_gather_object(counts, n_local, group=group)
            self.counts = counts
            if op in ("min", "max") and 0 in counts:
                self._fold_ranks = [r for r, c in enumerate(counts) if c > 0]
                if collective in ("p2p", "p2p_fused"):
                    collective = "all_gather" if dist.get_backend(group) == "nccl" else "allreduce"
        if op in ("min", "max") and sum(self.counts) == 0:
            raise ValueError(f"{op}: reduction over an empty range")
        ex = None
        if collective in ("p2p", "p2p_fused") and self.world > 1:
            # every rank must take the same path, or a peer waits for nothing
            ex = shared_exchange(group)
            if not _agree_all(group, ex is not None):
                ex = None
            if ex is None:
                collective = "all_gather" if dist.get_backend(group) == "nccl" else "allreduce"
        self.collective = collective
        self.elem = node.elem_type
        self.pdt = partial_dtype(op, self.elem)
        tdt = getattr(torch, _TORCH_DTYPE[self.pdt])
        if pipeline is None:
            pipeline = os.environ.get("BM_SHARD_PIPELINE", "1") != "0"
        # p2p_fused: the collective runs inside the reduction kernel, which already
        # overlaps the next step (programmatic dependent launch); no side stream
        self.pipeline = bool(pipeline) and self.world > 1 and collective != "p2p_fused"
        nbuf = 2 if self.pipeline else 1
        self.partials = [torch.zeros(1, dtype=tdt, device="cuda") for _ in range(nbuf)]
        self.gathered = [torch.zeros(self.world, dtype=tdt, device="cuda") for _ in range(nbuf)]
        self.results = [torch.zeros(1, dtype=tdt, device="cuda") for _ in range(nbuf)]
        self.partial = self.partials[0]
        self.result = self.results[0]
        views = _expr._step_views(self.plan, self.plan.reduce, {})
        self.inv = _rt.build_invocation(_rt.KernelInvocation("fused_reduce", tuple(views), None, (),
                                                             dict(self.plan.reduce.params)))
        self._lib = _clib.lib()
        self._op_code = {"accu": _clib.BM_R_ACCU, "min": _clib.BM_R_MIN, "max": _clib.BM_R_MAX,
                         "dot": _clib.BM_R_DOT}[op]
        self._step = 0
        self._last = 0
        self._exchange = ex if collective in ("p2p", "p2p_fused") else None
        if self.pipeline:
            self._comm = torch.cuda.Stream()
            self._reduced = [torch.cuda.Event() for _ in range(nbuf)]
            self._gathered = [None] * nbuf    # event after the gather + fold of the buffer's last step

    def _gather_and_fold(self, slot: int) -> None:
        part, gath = self.partials[slot], self.gathered[slot]
        if self._exchange is not None:     # one kernel over peer memory
            self._exchange.combine(part, self.elem, self._op_code, self.results[slot])
            return
        if self.collective == "all_gather":
            self.dist.all_gather_into_tensor(gath, part, group=self.group)
        else:
            gath.zero_()
            gath[self.rank:self.rank + 1].copy_(part)
            self.dist.all_reduce(gath, group=self.group)
        if self._fold_ranks is not None:        # min / max with empty shards: fold the others
            gath = gath[self._fold_ranks].contiguous()
        _clib.check(self._lib.bm_combine_partials_to_device(
            ctypes.c_void_p(gath.data_ptr()), gath.numel(), _clib.DTYPE_CODE[self.elem], self._op_code,
            ctypes.c_void_p(self.results[slot].data_ptr())), "combine partials")

    def launch(self) -> None:
        import torch
        slot = self._step % len(self.partials)
        self._step += 1
        self._last = slot
        compute = torch.cuda.current_stream()
        if self._exchange is not None and self.collective == "p2p_fused":
            self._exchange.reduce(self.inv, self.results[slot])
            return
        if self.pipeline and self._gathered[slot] is not None:
            compute.wait_event(self._gathered[slot])   # the gather that read this partial is done
        if self.counts[self.rank] > 0 or self.op not in ("min", "max"):
            _clib.check(self._lib.bm_reduce_to_device(ctypes.byref(self.inv),
                                                      ctypes.c_void_p(self.partials[slot].data_ptr())),
                        "sharded reduce")
        if self.world == 1:
            return
        if not self.pipeline:
            self._gather_and_fold(slot)
            return
        self._reduced[slot].record(compute)
        lib_stream = self._lib.bm_get_stream()
        with torch.cuda.stream(self._comm):
            self._comm.wait_event(self._reduced[slot])
            _clib.check(self._lib.bm_set_stream(ctypes.c_void_p(self._comm.cuda_stream)), "comm stream")
            try:
                self._gather_and_fold(slot)
            finally:
                _clib.check(self._lib.bm_set_stream(ctypes.c_void_p(lib_stream)), "compute stream")
            ev = torch.cuda.Event()
            ev.record(self._comm)
            self._gathered[slot] = ev

    def check(self) -> None:
        """After the caller synchronised: raise if an exchange timed out."""
        _check_exchange_error(self._exchange)

    def join(self) -> None:
        """Order the current stream after every collective issued so far."""
        import torch
        if self.pipeline:
            torch.cuda.current_stream().wait_stream(self._comm)

    def value(self):
        """The folded result of the last step.  Raises PeerTimeoutError when a
        peer never published into the exchange (the async-error contract of
        the reference: device errors surface at synchronisation)."""
        import torch
        self.join()
        torch.cuda.synchronize()
        self.check()
        src = self.partials[self._last] if self.world == 1 else self.results[self._last]
        v = src.cpu().numpy()[0]
        dt = kernels.NP_DTYPE[self.elem]
        if self.op == "dot" and dt.kind == "f":
            return dt.type(v)
        return np.asarray(v).astype(dt)[()]


def _check_exchange_error(ex) -> None:
    rc = _clib.lib().bm_poll_device_error()
    if rc != _clib.BM_OK:
        if ex is not None:
            ex.broken = True          # out of step with the peers: never used again
        _clib.check(rc, "sharded reduction")


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

    def __init__(self, ptr: int, count: int, elem: str, owner=None):
        self.owner = owner           # torch holds this object for the tensor's lifetime
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": kernels.NP_DTYPE[elem].str, "data": (ptr, False),
            "version": 3, "strides": None, "stream": None}


def torch_view(m):
    """The column-major storage of a device matrix as a flat torch tensor
    sharing its memory (no copy): what NCCL reads and writes.  The tensor
    keeps ``m`` alive (a view of a temporary stays valid); resizing ``m``
    (set_size / reset) leaves the view on the old storage."""
    import torch
    _rt.get_runtime().forget_sum(m.mem.buffer_id)   # the view can write: drop a cached accu
    return torch.as_tensor(_CudaArray(m.mem.ptr, m.n_elem, m.elem_type, owner=m), device="cuda")


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
    ov, lv = torch_view(out), torch_view(local)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(ov, lv, group=group)
    else:                                   # gloo (ranks sharing one GPU in tests): list all-gather
        dist.all_gather(list(ov.view(world, -1).unbind(0)), lv, group=group)
    return out


_LAST: dict = {}   # the path the last sharded call took ("peer" / "gather"; tests and bench)


def sharded_reduce_dim(op: str, local_expr, dim: int, group=None, collective=None):
    """sum/min/max along `dim` of a column-block-sharded matrix.

    dim 0 (one value per column): every rank owns its columns' results, no
    communication.  dim 1 (one value per row): each rank reduces its columns
    to a rows x 1 partial, the partials are all-gathered in rank order and
    folded with the same device reduction along dim 1 -- a left-to-right fold
    0 + p_0 + p_1 + ..., deterministic for a given world size (min/max are
    exact).  Returns the local dim-0 block or the full dim-1 column.  With
    peer memory (collective "p2p"/"p2p_fused", the default) the all-gather
    and the fold are one kernel (bm_exchange_rows), with the same bits."""
    from . import ops
    fn = {"sum": ops.sum, "min": ops.min, "max": ops.max}[op]
    local = _expr.evaluate(fn(local_expr, dim))
    if dim == 0 or _world(group)[1] == 1:
        return local
    if collective is None:
        collective = os.environ.get("BM_SHARD_COLLECTIVE", "p2p_fused")
    if collective in ("p2p", "p2p_fused"):
        # one kernel: every rank's partial over peer memory, folded in rank order
        cap = (local.n_elem * kernels.itemsize(local.elem_type) + 3) // 4
        ex = shared_vec_exchange(cap, group)
        if ex is not None:
            from .matrix import Matrix
            out = Matrix._uninitialised(local.n_rows, local.n_cols, local.elem_type)
            ex.rows(local.mem.ptr, local.n_elem, local.elem_type,
                    {"sum": _clib.BM_R_ACCU, "min": _clib.BM_R_MIN, "max": _clib.BM_R_MAX}[op], out.mem.ptr)
            _check_exchange_error(ex)
            _LAST["rows_collective"] = "peer"
            return out
    _LAST["rows_collective"] = "gather"
    return _expr.evaluate(fn(gather_columns(local, group), 1))


def sharded_gemm_nt(a, b_local):
    """C = A * B^T sharded over the rows of B (= the columns of C): rank r
    holds B's row block r and A replicated (broadcast_matrix), and computes
    its column block of C with no communication."""
    return _expr.evaluate(a @ b_local.t())


def sharded_logistic_step(x_local, w, y_local, group=None, collective=None):
    """One logistic-regression gradient step sharded by samples (row blocks
    of X): z = X_r w, r = 1/(1+exp(-z)) - y_r,
    g = sum_r X_r^T r_r (one all-gather of a 1024-vector, folded in rank
    order) and s = accu(r) over all ranks.  Returns (g, s).  Each rank runs
    the single-pass fused step on its shard (evaluate_many: X_r read once,
    bm_lgrad) wherever the planner can fuse it, the two-pass plan otherwise.
    With peer memory (collective "p2p"/"p2p_fused", the default) g and the
    folded accu(r) the fused step left in the sum cache cross the ranks in ONE
    kernel (bm_exchange_gsum); otherwise an NCCL all-gather of g, its dim-1
    sum and a ShardedReduction of r -- the same bits either way."""
    from . import ops
    r_e = 1 / (1 + ops.exp(0 - x_local @ w)) - y_local
    r, g_local = _expr.evaluate_many(r_e, x_local.t() @ r_e)
    if _world(group)[1] == 1:
        return g_local, ops.accu(r)
    if collective is None:
        collective = os.environ.get("BM_SHARD_COLLECTIVE", "p2p_fused")
    rt = _rt.get_runtime()
    slot = rt.sum_slot(r.mem)
    use_peer = collective in ("p2p", "p2p_fused") and g_local.elem_type == "f32" and \
        _agree_all(group, slot is not None)
    ex = shared_vec_exchange(g_local.n_elem, group) if use_peer else None
    if ex is not None:
        # one kernel: g and accu(r) of every rank over peer memory, folded in rank order
        from .matrix import Matrix
        g = Matrix._uninitialised(g_local.n_rows, g_local.n_cols, "f32")
        s_out = rt.acquire_memory(1, "f32")
        try:
            ex.gsum(g_local.mem.ptr, g_local.n_elem, slot.ptr, g.mem.ptr, s_out.ptr)
            s = float(rt.copy_d2h(s_out, 0, 1)[0])
        finally:
            rt.release_deferred(s_out)
        _check_exchange_error(ex)
        _LAST["logistic_collective"] = "peer"
        return g, s
    _LAST["logistic_collective"] = "gather"
    g = _expr.evaluate(ops.sum(gather_columns(g_local, group), 1))
    s = ShardedReduction("accu", r, group=group, collective=collective)
    s.launch()
    return g, s.value().item()
