"""Process-group plumbing for the one-process-per-GPU comm (host side only).

The IPC handle exchange is the single synchronisation the C ABI needs before connect
(include/tl_api.h "comm lifecycle").  Written against torch.distributed so it runs under
both NCCL (GPU box) and gloo (CPU tests).
"""
from __future__ import annotations


def exchange_handles(my_handle: bytes, group=None) -> bytes:
    """All-gather fixed-size handle blobs; returns world * len(my_handle) bytes in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = len(my_handle)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.frombuffer(bytearray(my_handle), dtype=torch.uint8).to(dev)
    out = torch.empty(world * n, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, mine, group=group)
    blob = bytes(out.cpu().numpy().tobytes())
    assert blob[dist.get_rank(group) * n:(dist.get_rank(group) + 1) * n] == my_handle
    return blob


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank scalar (timing rule: report the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
