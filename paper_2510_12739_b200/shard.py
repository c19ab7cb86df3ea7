"""Slot sharding across GPUs: every op of the CoNet-Rx forward is per slot and eval BN
uses running statistics (norms.hpp:65-74), so a slot batch splits into contiguous ranges with no
data-path collective.  The only exchange is the final LLR gather.

`slot_range` is the partition both bench.py (one process per GPU under torchrun) and
cnrx_receive_sharded (one process, several GPUs; api.cpp) use.  `gather_llr` collects per-rank LLR
slices on rank 0 over torch.distributed (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def slot_range(B: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous slot range [b0, b1) of `rank` out of `world` (ceil split, like api.cpp)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    per = (B + world - 1) // world
    b0 = min(B, rank * per)
    return b0, min(B, b0 + per)


def gather_llr_tensor(local, B: int, world: int, rank: int):
    """Tensor form of the final LLR gather (bench.py's multi-GPU e2e leg): `local` is this rank's LLR
    slice [b1-b0, T, F, bits] as a torch tensor on the backend's device (CUDA for NCCL, CPU for gloo),
    padded here to the ceil-split slice size; rank 0 returns the full [B, T, F, bits] tensor on that
    device, other ranks None.  One collective (gather), nothing else on the data path."""
    import torch
    import torch.distributed as dist

    per = (B + world - 1) // world
    if local.shape[0] != per:
        pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
        local = pad
    parts = [torch.empty_like(local) for _ in range(world)] if rank == 0 else None
    dist.gather(local.contiguous(), parts, dst=0)
    if rank != 0:
        return None
    return torch.cat(parts, 0)[:B]


def gather_llr(local: np.ndarray, B: int, world: int, rank: int):
    """All ranks pass their LLR slice [b1-b0, T, F, bits]; rank 0 returns the full [B, T, F, bits]."""
    import torch
    import torch.distributed as dist

    shape = local.shape[1:]
    per = (B + world - 1) // world
    buf = np.zeros((per,) + shape, np.float32)
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    parts = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, parts, dst=0)
    if rank != 0:
        return None
    full = np.concatenate([p.cpu().numpy() for p in parts], 0)
    return full[:B]
