"""The one-process-per-GPU path (tl_comm_create -> handle all-gather -> tl_comm_connect ->
cudaIpcOpenMemHandle) exercised with 2 processes sharing the single test GPU.

Bootstrap runs over gloo (the NCCL path uses the same exchange code).  Each process drives one
rank with half the SMs (num_ctas = 74), so the two persistent kernels can be co-resident when the
GPU runs both contexts concurrently (MPS); without MPS the contexts time-slice, which is slower but
still completes because every flag wait is bounded only by the 10 s timeout.  Either way the
results must match the fp64 oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2503_20313_b200 as tl
        import tl_inputs as TI
        M, H, I = 256, 128, 512
        X, G, U, W2 = TI.mlp_full(M, H, I, seed=4)
        Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, world, TI.ACT_SILU_MUL)
        comm = tl.Comm.from_process_group(None, 0, max_M=M, max_H=H)
        comm.set_option("num_ctas", 148 // world // 2 * 2)
        comm.set_option("timeout_ms", 60000)
        out = torch.empty(M // world, H, device="cuda", dtype=torch.bfloat16)
        res = []
        for _ in range(3):  # epochs / banks cycle across calls
            comm.mlp_forward(Xs[rank].cuda(), W1s[rank].cuda(), W2s[rank].cuda(), out, act=tl.ACT_SILU_MUL)
            st, diag = comm.check()
            res.append((st, out.float().cpu().numpy().copy()))
            dist.barrier()
        q.put((rank, [r[0] for r in res], [r[1] for r in res]))
        comm.close()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_mlp():
    import torch.multiprocessing as mp
    import tl_inputs as TI
    from oracle import tl_oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, sts, outs = q.get(timeout=600)
        assert sts != "error", outs
        got[rank] = (sts, outs)
    for p in procs:
        p.join(timeout=60)
    M, H, I = 256, 128, 512
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=4)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, world, TI.ACT_SILU_MUL)
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = O.mlp_forward(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL)
    for r in range(world):
        sts, outs = got[r]
        assert all(s == 0 for s in sts), sts
        for o in outs:
            assert O.rel_frobenius(o.astype(np.float64), ref[r]) < 5e-3
        assert all(np.array_equal(outs[0], o) for o in outs[1:])
