"""Multi-process EP launch helpers (one process per GPU, torch.distributed).

Used by bench.py --ep and covered on CPU by tests/test_ep.py with gloo.
torch.distributed is plumbing only: it hands the per-link ncclUniqueIds from
rank 0 to every rank and reduces timings; the data path (ENCODE / embeddings /
residuals / logits) runs over the native NCCL transport (csrc/ep_transport.cu).
"""
from __future__ import annotations

from typing import Tuple

from . import api

# World size -> (prefill stages, encoder ranks): the paper's 1+1 / 2+2 / 4+4.
EP_LAYOUTS = {2: (1, 1), 4: (2, 2), 8: (4, 4)}


def topology_for(world: int) -> Tuple[int, int]:
    if world not in EP_LAYOUTS:
        raise api.N.ConfigError(f"EP needs 2, 4 or 8 ranks (E+P = 1+1, 2+2, 4+4); got {world}")
    return EP_LAYOUTS[world]


def share_link_ids(stages: int, encoders: int, device=None) -> bytes:
    """Rank 0 draws one ncclUniqueId per EP link; every rank returns all of
    them (links order). `device`: where the broadcast tensor lives (a CUDA
    device for an NCCL process group, None/CPU for gloo)."""
    import torch
    import torch.distributed as dist
    n = len(api.ep_links(stages, encoders))
    buf = torch.zeros(n * 128, dtype=torch.uint8)
    if dist.get_rank() == 0:
        ids = b"".join(api.nccl_unique_id() for _ in range(n))
        buf = torch.frombuffer(bytearray(ids), dtype=torch.uint8).clone()
    if device is not None:
        buf = buf.to(device)
    dist.broadcast(buf, src=0)
    return bytes(buf.cpu().numpy().tobytes())


def connect_ipc(group: "api.EpGroup") -> None:
    """Exchange the CUDA-IPC export blobs of all ranks and connect."""
    import torch.distributed as dist
    blobs = [None] * dist.get_world_size()
    dist.all_gather_object(blobs, group.export())
    group.connect(blobs)
    dist.barrier()


def shm_name_for_group() -> str:
    """One POSIX shm name per EP group, drawn on rank 0."""
    import os
    import torch.distributed as dist
    name = [f"/rserve_ep_{os.getpid()}_{os.urandom(4).hex()}" if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(name, src=0)
    return name[0]


def max_over_ranks(value: float, device=None) -> float:
    """Job time = the slowest rank's device time."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64)
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
