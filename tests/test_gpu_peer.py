"""Peer-memory LLR gather (include/conetrx_cuda.h cnrx_ipc_*, shard.PeerLLR): a second process maps the
first process's batch buffer (CUDA IPC) and its plan's LLR head stores its slots straight into it --
the final gather fused into the last kernel.  On a one-GPU box both processes use cuda:0 (same-device
IPC); on an NVSwitch box the stores go over NVLink, same code.  The written slots must equal the
second process's own receive() bit for bit, and the first process's slots must be untouched."""
import dataclasses
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _writer(handle, b0, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2510_12739_b200 import graph as G, plan as P, slots
    try:
        link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=40)
        b = slots.generate(link, 3, 21)
        p = P.Plan(G.CONFIGS["cfg2"].graph(seed=6), "bf16")
        p.set_pilots(b.pilots, b.pilot_mask)
        base = P.ipc_open(0, handle)
        slot_bytes = 4 * link.T * link.F * 4
        y = torch.from_numpy(b.y).cuda()
        p.receive_device_ptr(y, base + b0 * slot_bytes, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        P.ipc_close(0, base)
        q.put(p.receive(b.y))
    except Exception as e:  # reported to the parent
        q.put(repr(e))


def test_peer_llr_stores_land_in_the_owner_buffer():
    import torch
    from paper_2510_12739_b200 import graph as G, plan as P, slots
    link = dataclasses.replace(G.CONFIGS["cfg2"].link, F=40)
    slot_bytes = 4 * link.T * link.F * 4
    B, b0 = 5, 2  # the owner's slots [0, 2), the writer's [2, 5)
    ptr, handle = P.ipc_alloc(0, B * slot_bytes)
    own = slots.generate(link, b0, 22)
    p = P.Plan(G.CONFIGS["cfg2"].graph(seed=6), "bf16")
    p.set_pilots(own.pilots, own.pilot_mask)
    p.receive_device_ptr(torch.from_numpy(own.y).cuda(), ptr, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_writer, args=(handle, b0, q))
    pr.start()
    res = q.get(timeout=300)
    pr.join(timeout=60)
    assert not isinstance(res, str), res
    out = torch.empty((B, link.T, link.F, 4), dtype=torch.float32).pin_memory()
    P.ipc_read(0, ptr, out.data_ptr(), B * slot_bytes)
    assert np.array_equal(out.numpy()[b0:], res)            # the writer's head stores, bit for bit
    assert np.array_equal(out.numpy()[:b0], p.receive(own.y))  # the owner's slots untouched
    # the stream-ordered read (bench.py's rank 0 reads step k on a side stream while step k + 1 computes)
    out2 = torch.zeros((B, link.T, link.F, 4), dtype=torch.float32).pin_memory()
    side = torch.cuda.Stream()
    P.ipc_read_async(0, ptr, out2.data_ptr(), B * slot_bytes, side.cuda_stream)
    side.synchronize()
    assert torch.equal(out2, out)
    P.ipc_free(0, ptr)
