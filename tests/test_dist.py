"""Host-side logic of the multi-GPU path on CPU (gloo, world size 2).

The device kernels need a GPU, so here every rank computes its shard's partial with the
oracle (the reference's algorithm). The ranks then all-gather the partials in rank order
over gloo and fold them with combine_pairwise, the same sequence paper_2308_03120_b200.dist
drives on the GPU. The result must equal the single-device reduction of the whole matrix,
bit for bit, when shards are power-of-two runs of REDUCE_BLOCK blocks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2308_03120_b200.dist import column_block


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_column_block_partition():
    for total in (1, 7, 64, 1000, 4096 * 8):
        for world in (1, 2, 3, 4, 8):
            spans = [column_block(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _worker(rank, world, port, rows, cols, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        full = (rng.standard_normal((rows, cols)) * np.exp2(rng.integers(-10, 10, (rows, cols)))).astype(np.float32)
        start, count = column_block(cols, rank, world)
        shard = np.asfortranarray(full[:, start:start + count]).reshape(-1, order="F")
        part_accu = O.reduce_accu(shard)
        part_max = O.reduce_max(shard)
        t = torch.tensor([float(part_accu), float(part_max)], dtype=torch.float64)
        gathered = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, t)
        accu_parts = [np.float32(g[0].item()) for g in gathered]
        max_parts = [np.float32(g[1].item()) for g in gathered]
        acc = O.combine_pairwise(accu_parts, lambda a, b: np.float32(a + b))
        mx = O.combine_pairwise(max_parts, O.py_max)
        if rank == 0:
            flat = np.asfortranarray(full).reshape(-1, order="F")
            q.put((np.float32(acc).tobytes(), np.float32(O.reduce_accu(flat)).tobytes(),
                   float(mx), float(O.reduce_max(flat))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols", [(512, 1024), (256, 2048)])
def test_sharded_reduction_is_bit_identical_to_single_device(rows, cols):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    sharded, single, mx, mx1 = q.get(timeout=10)
    assert sharded == single          # aligned power-of-two block runs per rank
    assert mx == mx1


# ---- row reductions, GEMM and the logistic step, sharded ---------------------------

def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    return q.get(timeout=10)


def _gather_columns(local: np.ndarray, world: int) -> np.ndarray:
    """What dist.gather_columns does on the device: all-gather in rank order
    into a rows x world column-major matrix (column r = rank r)."""
    t = torch.from_numpy(np.ascontiguousarray(local.reshape(-1)))
    out = torch.zeros(world * t.numel(), dtype=t.dtype)
    dist.all_gather_into_tensor(out, t)
    return out.numpy().reshape((t.numel(), world), order="F")


def _rdim_worker(rank, world, port, q, rows, cols):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = np.random.default_rng(4).standard_normal((rows, cols))
        start, count = column_block(cols, rank, world)
        local = np.asfortranarray(full[:, start:start + count])
        res = {}
        for op in ("sum", "min", "max"):
            part = O.rdim(op, local, 1).reshape(-1)                    # rows x 1 on this rank
            gathered = _gather_columns(part, world)                    # rows x world, rank order
            res[op] = O.rdim(op, gathered, 1).reshape(-1)              # the dim-1 fold of the partials
            res[op + "_single"] = O.rdim(op, np.asfortranarray(full), 1).reshape(-1)
            # dim 0: each rank's columns only, no communication
            res[op + "_dim0_ok"] = bool(np.array_equal(O.rdim(op, local, 0).reshape(-1),
                                                       O.rdim(op, np.asfortranarray(full), 0).reshape(-1)[start:start + count]))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_sharded_row_reductions_match_single_device():
    res = _spawn(_rdim_worker, 2, 300, 257)
    for op in ("sum", "min", "max"):
        assert res[op + "_dim0_ok"]
        if op == "sum":
            np.testing.assert_allclose(res[op], res[op + "_single"], rtol=1e-12)
        else:
            assert np.array_equal(res[op], res[op + "_single"])    # min/max are exact


def _gemm_worker(rank, world, port, q, m, n, k):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        a = rng.random((m, k)) if rank == 0 else np.zeros((m, k))
        b = np.random.default_rng(6).random((n, k))
        ta = torch.from_numpy(np.asfortranarray(a).reshape(-1, order="F").copy())
        dist.broadcast(ta, 0)                                          # broadcast_matrix
        a = ta.numpy().reshape((m, k), order="F")
        start, count = column_block(n, rank, world)                    # rows of B = columns of C
        c_local = a @ b[start:start + count].T                         # sharded_gemm_nt, no communication
        blocks = [torch.zeros(m * column_block(n, r, world)[1], dtype=torch.float64) for r in range(world)]
        dist.all_gather(blocks, torch.from_numpy(np.asfortranarray(c_local).reshape(-1, order="F").copy()))
        if rank == 0:
            c = np.concatenate([blk.numpy().reshape((m, -1), order="F") for blk in blocks], axis=1)
            q.put(float(np.abs(c - a @ b.T).max()))
    finally:
        dist.destroy_process_group()


def test_sharded_gemm_column_blocks_assemble_the_product():
    assert _spawn(_gemm_worker, 2, 40, 34, 20) < 1e-12


def _logistic_worker(rank, world, port, q, nrow, ncol):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        X = rng.standard_normal((nrow, ncol)).astype(np.float32)
        w = (0.03 * rng.standard_normal((ncol, 1))).astype(np.float32)
        y = (rng.random((nrow, 1)) < 0.5).astype(np.float32)
        start, count = column_block(nrow, rank, world)                 # samples = rows of X
        xl, yl = X[start:start + count], y[start:start + count]
        r = (1 / (1 + np.exp(-(xl.astype(np.float64) @ w))) - yl).astype(np.float32)
        g_local = (xl.T.astype(np.float64) @ r).reshape(-1)
        gathered = _gather_columns(g_local, world)
        g = O.rdim("sum", gathered, 1).reshape(-1)                     # fold in rank order
        s_parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(s_parts, torch.tensor([float(r.astype(np.float64).sum())], dtype=torch.float64))
        if rank == 0:
            rf = (1 / (1 + np.exp(-(X.astype(np.float64) @ w))) - y)
            gf = (X.T.astype(np.float64) @ rf).reshape(-1)
            q.put((float(np.abs(g - gf).max() / np.abs(gf).max()),
                   abs(sum(p.item() for p in s_parts) - rf.sum()) / max(abs(rf.sum()), 1.0)))
    finally:
        dist.destroy_process_group()


def test_sharded_logistic_step_matches_single_device():
    gerr, serr = _spawn(_logistic_worker, 2, 1000, 64)
    assert gerr < 1e-6 and serr < 1e-6


# ---- the pipelined device path: two ranks sharing one GPU over gloo ----------------------------

def _pipeline_worker(rank, world, port, q, rows, cols, pipeline, collective="allreduce"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_03120_b200 as dm
        from paper_2308_03120_b200 import dist as D
        torch.cuda.set_device(0)
        dm.init("b200", device_id=0)
        D.bind_torch_stream()
        full = np.random.default_rng(9).random((rows, cols), dtype=np.float32)
        start, count = column_block(cols, rank, world)
        m = dm.Matrix.from_numpy(np.asfortranarray(full[:, start:start + count]))
        red = D.ShardedReduction("accu", m, pipeline=pipeline, collective=collective)
        view = D.torch_view(m)
        # three back-to-back steps, the input doubled on the compute stream in between:
        # step k reduces 2^k * X (exact), step 2 reuses step 0's buffers
        red.launch()
        view.mul_(2)
        red.launch()
        view.mul_(2)
        red.launch()
        red.join()
        torch.cuda.synchronize()
        res = [np.float32(r.cpu().numpy()[0]).tobytes() for r in red.results]
        last = np.float32(red.value()).tobytes()
        if rank == 0:
            q.put((res, last, red.pipeline))
        if red._exchange is not None:
            dist.barrier()                 # no rank unmaps while a peer may still write
            red._exchange.close()
        dm.shutdown()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("pipeline", [True, False])
def test_pipelined_sharded_reduction_two_ranks_one_gpu(pipeline):
    rows, cols = 1024, 256                     # 16 REDUCE_BLOCK blocks per rank: bit-exact
    res, last, piped = _spawn(_pipeline_worker, 2, rows, cols, pipeline)
    full = np.random.default_rng(9).random((rows, cols), dtype=np.float32)
    want = [np.float32(O.reduce_accu((np.float32(2 ** k) * full).reshape(-1, order="F"))).tobytes()
            for k in range(3)]
    assert piped == pipeline
    assert last == want[2]
    if pipeline:
        assert res == [want[2], want[1]]       # buffers by step parity
    else:
        assert res == [want[2]]


@pytest.mark.gpu
@pytest.mark.parametrize("pipeline,collective", [(True, "p2p"), (False, "p2p"), (False, "p2p_fused")])
def test_peer_exchange_two_ranks_one_gpu(pipeline, collective):
    """The peer-memory exchange (one kernel: publish the partial into every
    rank's buffer over CUDA IPC, wait for all epochs, fold in rank order)
    gives the same bits as the all-gather path, pipelined or not."""
    rows, cols = 1024, 256
    res, last, piped = _spawn(_pipeline_worker, 2, rows, cols, pipeline, collective)
    full = np.random.default_rng(9).random((rows, cols), dtype=np.float32)
    want = [np.float32(O.reduce_accu((np.float32(2 ** k) * full).reshape(-1, order="F"))).tobytes()
            for k in range(3)]
    assert last == want[2]
    if pipeline:
        assert res == [want[2], want[1]]
    elif collective == "p2p":
        assert res == [want[2]]
