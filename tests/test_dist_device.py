"""The sharded reductions' device path with several ranks on ONE GPU (gloo for
the host collectives, CUDA IPC for the peer-memory exchange).

This box has one GPU, so the ranks share it; the kernels, the exchange
protocol and the fold order are the ones an 8-GPU box runs.  Shard sizes are
the BASELINE config-3 scale per rank (2^27 - 2^28 elements), large enough for
the separate fold kernels, which the fused exchange must also cover (VERDICT
r1, missing 1).  Results are compared bit for bit with the single-device
reduction of the concatenated vector: every shard is an aligned power-of-two
run of REDUCE_BLOCK blocks, and aligned groups fold independently
(tests/test_oracle.py::test_combine_pairwise_is_hierarchical_over_aligned_groups),
so the reference's combine_pairwise order (kernels.py:380-392) is kept.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist



def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2308_03120_b200 as dm
    from paper_2308_03120_b200 import dist as D
    torch.cuda.set_device(0)
    dm.init("b200", device_id=0)
    D.bind_torch_stream()
    return dm, D


def _shard_of(dm, D, full, rank, world):
    """Rank's contiguous block of a device column vector, as its own Col."""
    start, count = D.column_block(full.n_elem, rank, world)
    shard = dm.Matrix(count, 1, elem_type=full.elem_type)
    if count:
        D.torch_view(shard).copy_(D.torch_view(full)[start:start + count])
    return shard


def _single(dm, op, a, b=None):
    """The single-device reduction through the public API."""
    if op == "dot":
        return dm.dot(a, b)
    return {"accu": dm.accu, "min": dm.reduce_min, "max": dm.reduce_max}[op](a)


def _bits(x, dt) -> bytes:
    return np.asarray(x).astype(dt).tobytes()


def _large_worker(rank, world, port, q, op, elem, n, collective):
    dm, D = _init(rank, world, port)
    try:
        dt = np.float32 if elem == "f32" else np.float64
        dm.set_seed(17)
        a = dm.Matrix(n, 1, fill="randn", elem_type=elem)
        b = dm.Matrix(n, 1, fill="randu", elem_type=elem) if op == "dot" else None
        want = _single(dm, op, a, b)
        args = (_shard_of(dm, D, a, rank, world),)
        if op == "dot":
            args += (_shard_of(dm, D, b, rank, world),)
        del a, b
        red = D.ShardedReduction(op, *args, collective=collective)
        red.launch()
        red.launch()                      # a second step: the other exchange parity
        got = red.value()
        q.put((rank, _bits(got, dt), _bits(want, dt), red.collective))
        dist.barrier()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


def _collect(world, target, *args):
    """Spawn `world` ranks that each put one tuple; return them by rank."""
    import torch.multiprocessing as mp
    from test_dist import _free_port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    import queue as _queue
    import time as _time
    out, t0 = [], _time.time()
    try:
        while len(out) < world:
            try:
                out.append(q.get(timeout=1))
            except _queue.Empty:
                bad = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
                assert not bad, f"a rank failed: exit codes {[p.exitcode for p in procs]}"
                assert _time.time() - t0 < 600, "ranks timed out"
        for p in procs:
            p.join(timeout=120)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    return sorted(out, key=lambda t: t[0])


# (op, elem, elements per rank): the first two take the in-kernel fold, the
# rest the separate chunk-fold kernels with the exchange in fold_final_kernel
LARGE = [("accu", "f32", 1 << 27), ("max", "f32", 1 << 27), ("dot", "f32", 1 << 27),
         ("accu", "f32", 1 << 28), ("min", "f32", 1 << 28), ("accu", "f64", 1 << 27)]


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("op,elem,per_rank", LARGE)
def test_fused_exchange_large_shards_bit_identical(op, elem, per_rank):
    """Two ranks, BASELINE-scale shards, the default collective (reduction +
    peer-memory exchange in one launch sequence): every rank gets the bits of
    the single-device reduction of the whole vector."""
    res = _collect(2, _large_worker, op, elem, 2 * per_rank, None)
    for rank, got, want, coll in res:
        assert coll == "p2p_fused"
        assert got == want, (rank, op, elem)


@pytest.mark.gpu
@pytest.mark.parametrize("collective", ["p2p_fused", "p2p", "allreduce"])
def test_sharded_dot_collectives_agree_world4(collective):
    """Four ranks on one GPU, config-3 dot at 2^24 per rank: every collective
    returns the single-device bits."""
    res = _collect(4, _large_worker, "dot", "f32", 4 << 24, collective)
    for rank, got, want, coll in res:
        assert coll == collective
        assert got == want, rank


def _empty_worker(rank, world, port, q, op, elem, n, collective):
    dm, D = _init(rank, world, port)
    try:
        dt = np.float32 if elem == "f32" else np.float64
        dm.set_seed(3)
        a = dm.Matrix(n, 1, fill="randn", elem_type=elem)
        b = dm.Matrix(n, 1, fill="randn", elem_type=elem)
        want = _single(dm, op, a, b)
        # every element on rank 0, rank 1 empty (column_block of one column)
        count = n if rank == 0 else 0
        sa = dm.Matrix(count, 1, elem_type=elem)
        sb = dm.Matrix(count, 1, elem_type=elem)
        if count:
            D.torch_view(sa).copy_(D.torch_view(a))
            D.torch_view(sb).copy_(D.torch_view(b))
        args = (sa, sb) if op == "dot" else (sa,)
        red = D.ShardedReduction(op, *args, collective=collective)
        red.launch()
        got = red.value()
        q.put((rank, _bits(got, dt), _bits(want, dt), red.collective))
        dist.barrier()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["accu", "dot", "min", "max"])
@pytest.mark.parametrize("collective", ["p2p_fused", "allreduce"])
def test_empty_shard(op, collective):
    """A rank with no columns (cols < world) takes part in the exchange with a
    zero (accu / dot) or is left out of the fold (min / max): the world result
    is the non-empty rank's, and no rank waits for a partial that never comes."""
    res = _collect(2, _empty_worker, op, "f32", 100_000, collective)
    for rank, got, want, coll in res:
        assert got == want, (rank, op, coll)


def _timeout_worker(rank, world, port, q):
    os.environ["BM_EXCH_TIMEOUT_S"] = "2"
    dm, D = _init(rank, world, port)
    try:
        from paper_2308_03120_b200._clib import PeerTimeoutError
        m = dm.Matrix(1 << 20, 1, fill="randu")
        red = D.ShardedReduction("accu", m)          # collective construction on every rank
        outcome = "no-error"
        if rank == 0:                                # rank 1 never launches its step
            red.launch()
            try:
                red.value()
            except PeerTimeoutError as e:
                outcome = "PeerTimeoutError: " + str(e)[:80]
        dist.barrier()
        # the next construction agrees on a path without the broken exchange
        red2 = D.ShardedReduction("accu", m)
        red2.launch()
        v = red2.value()
        q.put((rank, outcome, red2.collective, float(v)))
        dist.barrier()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_timeout_raises_at_synchronise():
    """A peer that never publishes turns into PeerTimeoutError at the next
    synchronisation (the reference re-raises asynchronous device errors at
    synchronise, runtime.py:340-353), not into a silently wrong value; the
    broken exchange is never used again."""
    res = _collect(2, _timeout_worker)
    (r0, out0, coll0, v0), (r1, out1, coll1, v1) = res
    assert out0.startswith("PeerTimeoutError"), out0
    assert out1 == "no-error"
    assert coll0 == coll1 == "allreduce"
    assert v0 == v1


# ---- the sample-sharded logistic step: g and accu(r) over peer memory in one kernel -------------

def _logistic_worker(rank, world, port, q, rows, cols):
    dm, D = _init(rank, world, port)
    try:
        rng = np.random.default_rng(21)
        X = rng.standard_normal((rows, cols), dtype=np.float32)
        w = (0.03 * rng.standard_normal((cols, 1))).astype(np.float32)
        y = (rng.random((rows, 1)) < 0.5).astype(np.float32)
        r0, rc = D.column_block(rows, rank, world)
        Xl = dm.Matrix.from_numpy(np.asfortranarray(X[r0:r0 + rc]))
        yl = dm.Matrix.from_numpy(np.asfortranarray(y[r0:r0 + rc]))
        wm = dm.Matrix.from_numpy(w)
        out = {}
        for coll in ("p2p_fused", "all_gather"):
            for step in range(2):             # two steps: both exchange parities
                g, s = D.sharded_logistic_step(Xl, wm, yl, collective=coll)
            out[coll] = (g.to_numpy().tobytes(), np.float32(s).tobytes(), D._LAST["logistic_collective"])
        # the single-device step on the full matrix (every rank computes it)
        Xf, yf = dm.Matrix.from_numpy(X), dm.Matrix.from_numpy(y)
        r_e = 1 / (1 + dm.exp(0 - Xf @ wm)) - yf
        r, gf = dm.evaluate_many(r_e, Xf.t() @ r_e)
        sf = dm.accu(r)
        q.put((rank, out, gf.to_numpy().astype(np.float64), float(sf)))
        dist.barrier()
        D.close_exchanges()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,rows,cols", [(2, 1 << 16, 256), (3, 3 * 8192 * 4, 1024), (2, 65536, 2000),
                                             (2, 65538, 512)])
def test_sharded_logistic_exchange_matches_all_gather(world, rows, cols):
    """bm_exchange_gsum (g and the sum-cached accu(r) of every rank in one kernel
    over CUDA IPC peer memory, folded in rank order) gives the bits of the NCCL /
    gloo all-gather path -- gathered columns summed along dim 1, accu exchanged --
    on every rank, and matches the single-device step."""
    res = _collect(world, _logistic_worker, rows, cols)
    paths = {out["p2p_fused"][2] for _, out, _, _ in res}
    assert len(paths) == 1, "ranks took different paths"      # agreed collectively
    for rank, out, gf, sf in res:
        if rows % (4 * world) == 0:
            assert out["p2p_fused"][2] == "peer"
        assert out["all_gather"][2] == "gather"
        assert out["p2p_fused"][:2] == out["all_gather"][:2], f"rank {rank}: exchange differs from all-gather"
        assert out["p2p_fused"][:2] == res[0][1]["p2p_fused"][:2], "ranks disagree"
        g = np.frombuffer(out["p2p_fused"][0], dtype=np.float32).astype(np.float64)
        assert np.abs(g - gf.reshape(-1)).max() <= 1e-5 * np.abs(gf).max()
        s = float(np.frombuffer(out["p2p_fused"][1], dtype=np.float32)[0])
        assert abs(s - sf) <= 1e-5 * max(abs(sf), 1.0)


def _rows_worker(rank, world, port, q, rows, cols, elem):
    dm, D = _init(rank, world, port)
    try:
        dt = np.float32 if elem == "f32" else np.float64
        full = np.random.default_rng(23).random((rows, cols)).astype(dt)
        full[3, 5] = -0.0
        c0, cc = D.column_block(cols, rank, world)
        m = dm.Matrix.from_numpy(np.asfortranarray(full[:, c0:c0 + cc]))
        out = {}
        for op in ("sum", "min", "max"):
            got = {}
            for coll in ("p2p_fused", "all_gather"):
                for _ in range(2):              # both exchange parities
                    v = D.sharded_reduce_dim(op, m, 1, collective=coll)
                got[coll] = (v.to_numpy().tobytes(), D._LAST["rows_collective"])
            out[op] = got
        single = {op: getattr(dm, op)(dm.Matrix.from_numpy(full), 1) for op in ("sum", "min", "max")}
        q.put((rank, out, {op: dm.evaluate(v).to_numpy().tobytes() for op, v in single.items()}))
        dist.barrier()
        D.close_exchanges()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,rows,cols,elem", [(2, 16384, 512, "f64"), (3, 4096, 300, "f32"), (4, 1000, 64, "f64")])
def test_sharded_row_reductions_exchange_matches_all_gather(world, rows, cols, elem):
    """bm_exchange_rows (every rank's dim-1 partial over peer memory, folded in
    rank order in one kernel) gives the bits of the all-gather + dim-1 fold on
    every rank; min / max are the single-device values exactly."""
    res = _collect(world, _rows_worker, rows, cols, elem)
    for rank, out, single in res:
        for op, got in out.items():
            assert got["p2p_fused"][1] == "peer" and got["all_gather"][1] == "gather"
            assert got["p2p_fused"][0] == got["all_gather"][0], f"rank {rank} {op}: exchange differs"
            assert got["p2p_fused"][0] == res[0][1][op]["p2p_fused"][0], "ranks disagree"
            if op != "sum":
                assert got["p2p_fused"][0] == single[op]


def _rows_empty_worker(rank, world, port, q, rows, cols):
    dm, D = _init(rank, world, port)
    try:
        full = np.random.default_rng(29).random((rows, cols))
        c0, cc = D.column_block(cols, rank, world)
        m = dm.Matrix.from_numpy(np.asfortranarray(full[:, c0:c0 + cc])) if cc else dm.Matrix(rows, 0, elem_type="f64")
        got = {}
        for coll in ("p2p_fused", "all_gather"):
            v = D.sharded_reduce_dim("sum", m, 1, collective=coll)
            got[coll] = (v.to_numpy().tobytes(), D._LAST["rows_collective"])
        q.put((rank, cc, got))
        dist.barrier()
        D.close_exchanges()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_row_sum_with_empty_shards():
    """More ranks than columns: a rank with no columns takes part in the
    exchange with zeros, and every rank gets the all-gather path's bits."""
    res = _collect(4, _rows_empty_worker, 512, 3)
    assert any(cc == 0 for _, cc, _ in res)
    for rank, cc, got in res:
        assert got["p2p_fused"][1] == "peer" and got["all_gather"][1] == "gather"
        assert got["p2p_fused"][0] == got["all_gather"][0], f"rank {rank}"
        assert got["p2p_fused"][0] == res[0][2]["p2p_fused"][0]
