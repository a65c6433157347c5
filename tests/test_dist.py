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
