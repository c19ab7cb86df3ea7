"""Slot sharding across GPUs: every op of the CoNet-Rx forward is per slot and eval BN
uses running statistics (norms.hpp:65-74), so a slot batch splits into contiguous ranges with no
data-path collective.  The only exchange is the final LLR gather.

`slot_range` is the partition both bench.py (one process per GPU under torchrun) and
cnrx_receive_sharded (one process, several GPUs; api.cpp) use.  `gather_llr` collects per-rank LLR
slices on rank 0 over torch.distributed (NCCL on the GPU box, gloo in the CPU tests).  `PeerLLR` fuses
the gather into the last kernel instead: rank 0's LLR buffer is mapped into every rank (CUDA IPC), and
each rank's LLR head stores its slots straight into it over NVLink.
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


class PeerLLR:
    """The whole batch's LLR buffer on rank 0's GPU, mapped into every rank (cnrx_ipc_alloc / _open):
    rank r passes `dst(b0)` (its first slot) as the LLR destination of receive_device_ptr, so the head
    kernel's stores land in rank 0's HBM over NVLink -- the final gather fused into the last kernel, no
    collective on the data path.  Completion protocol: every rank synchronizes its stream, then a
    host barrier (torch.distributed); rank 0 then reads the full batch (`to_host`).  The 64-byte handle
    travels once, at setup, with broadcast_object_list."""

    def __init__(self, B: int, row_shape, rank: int, device: int):
        import torch.distributed as dist
        from paper_2510_12739_b200 import plan as P
        self.rank, self.device = rank, device
        self.slot_bytes = 4 * int(np.prod(row_shape))
        self.B = B
        obj = [None]
        if rank == 0:
            self.ptr, handle = P.ipc_alloc(device, B * self.slot_bytes)
            obj = [handle]
        dist.broadcast_object_list(obj, src=0)
        err = None
        if rank != 0:
            try:
                self.ptr = P.ipc_open(device, obj[0])
            except Exception as e:  # e.g. no peer access between these GPUs
                self.ptr, err = None, e
        # every rank learns whether all mappings succeeded (so a failure cannot leave ranks in different code paths)
        ok = [err is None]
        allok = [None] * dist.get_world_size()
        dist.all_gather_object(allok, ok[0])
        if not all(allok):
            if rank == 0:
                P.ipc_free(device, self.ptr)
            elif self.ptr is not None:
                P.ipc_close(device, self.ptr)
            raise RuntimeError(f"peer mapping of rank 0's LLR buffer failed on some rank ({err!r})")

    def dst(self, b0: int) -> int:
        return self.ptr + b0 * self.slot_bytes

    def to_host(self, out) -> None:
        """rank 0: copy the full batch into `out` (a pinned torch tensor of B * slot_bytes bytes)."""
        from paper_2510_12739_b200 import plan as P
        P.ipc_read(self.device, self.ptr, out.data_ptr(), self.B * self.slot_bytes)

    def to_host_async(self, out, stream: int) -> None:
        """rank 0: the same copy enqueued on `stream` (a cudaStream_t handle), not waited for."""
        from paper_2510_12739_b200 import plan as P
        P.ipc_read_async(self.device, self.ptr, out.data_ptr(), self.B * self.slot_bytes, stream)

    def close(self) -> None:
        from paper_2510_12739_b200 import plan as P
        if self.rank == 0:
            P.ipc_free(self.device, self.ptr)
        else:
            P.ipc_close(self.device, self.ptr)
