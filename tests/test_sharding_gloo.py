"""Multi-rank slot sharding on CPU with torch.distributed gloo, world_size 2: each rank
runs its contiguous slot range through the oracle forward, rank 0 gathers; the result equals the
unsharded forward bit-for-bit (no data-path collective, only the final LLR gather)."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import oracle
    from paper_2510_12739_b200 import graph as G, shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = G.CONFIGS["cfg1"].graph(seed=3)
    x = np.random.default_rng(5).standard_normal((B, 14, 72, 6)).astype(np.float32)
    b0, b1 = shard.slot_range(B, world, rank)
    local = oracle.forward(g, x[b0:b1]) if b1 > b0 else np.zeros((0, 14, 72, 2), np.float32)
    full = shard.gather_llr(local, B, world, rank)
    if rank == 0:
        q.put(np.array_equal(full, oracle.forward(g, x)))
    dist.barrier()
    dist.destroy_process_group()


def _gather_worker(rank, world, port, B, q):
    """bench.py's multi-GPU e2e gather at the cfg2 LLR shape [B, 14, 612, 4] (ragged split)."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2510_12739_b200 import shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full_ref = torch.arange(B * 14 * 612 * 4, dtype=torch.float32).reshape(B, 14, 612, 4)
    b0, b1 = shard.slot_range(B, world, rank)
    got = shard.gather_llr_tensor(full_ref[b0:b1].clone(), B, world, rank)
    if rank == 0:
        q.put(bool(torch.equal(got, full_ref)) and tuple(got.shape) == (B, 14, 612, 4))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)


@pytest.mark.parametrize("B", [3, 8])
def test_two_rank_llr_gather_cfg2_shape(B):
    _spawn(_gather_worker, 2, B)


@pytest.mark.parametrize("B", [5, 6])
def test_two_rank_sharded_forward_equals_full(B):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)


def test_slot_ranges_cover_batch():
    from paper_2510_12739_b200 import shard
    for B in (1, 7, 256, 8192):
        for w in (1, 2, 3, 8):
            r = [shard.slot_range(B, w, k) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
