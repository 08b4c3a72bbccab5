"""world_size-2 gloo tests of the host-side multi-process plumbing (handle exchange, max-over-ranks
timing) that the NCCL path uses on the GPU box."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_20313_b200.bootstrap import exchange_handles, max_over_ranks
        mine = bytes([rank * 16 + i for i in range(40)])
        blob = exchange_handles(mine)
        expect = b"".join(bytes([r * 16 + i for i in range(40)]) for r in range(world))
        m = max_over_ranks(1.5 + rank)
        q.put((rank, blob == expect, m))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_handle_exchange_and_max(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, m in res:
        assert ok, f"rank {rank} got a wrong handle blob"
        assert m == 1.5 + world - 1
