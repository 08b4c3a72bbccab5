"""The one-process-per-GPU path (tl_comm_create -> handle all-gather -> tl_comm_connect ->
cudaIpcOpenMemHandle) exercised with real processes: one device per rank when the box has enough GPUs
(the cross-device data plane over NVLink: tools/two_gpu_check.sh), else all ranks sharing cuda:0.

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

from parity import assert_parity

pytestmark = pytest.mark.gpu


def _device(rank, world):
    """One GPU per rank when the box has enough (real NVLink peers: the cross-device data plane),
    else every rank on cuda:0 (CUDA IPC within one device, half the SMs each)."""
    n = torch.cuda.device_count()
    return (rank, False) if n >= world else (0, True)


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
        dev, shared = _device(rank, world)
        torch.cuda.set_device(dev)
        import paper_2503_20313_b200 as tl
        import tl_inputs as TI
        M, H, I = 256, 128, 512
        X, G, U, W2 = TI.mlp_full(M, H, I, seed=4)
        Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, world, TI.ACT_SILU_MUL)
        comm = tl.Comm.from_process_group(None, dev, max_M=M, max_H=H)
        if shared:
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
            assert_parity(o.astype(np.float64), ref[r])
        assert all(np.array_equal(outs[0], o) for o in outs[1:])


def _worker_all(rank, world, port, q, mode="sm"):
    """One rank per process: the MLP layer, the MoE layer and SP attention through the
    process-group comm (IPC-mapped peers), results sent back for the oracle check."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev, shared = _device(rank, world)
        torch.cuda.set_device(dev)
        import paper_2503_20313_b200 as tl
        import tl_inputs as TI
        res = {}
        # MLP
        M, H, I = 128 * world, 128, 128 * world
        X, G, U, W2 = TI.mlp_full(M, H, I, seed=6)
        Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, world, TI.ACT_SILU_MUL)
        comm = tl.Comm.from_process_group(None, dev, max_M=max(M, 512 * world), max_H=512, max_topk=2)
        if shared:
            comm.set_option("num_ctas", max(2, 148 // world // 2 * 2))
        comm.set_option("timeout_ms", 120000)
        if mode == "dma":   # both exchanges on the copy engines (cross-process IPC copies + stream flags)
            comm.set_option("ag_binding", 1)
            comm.set_option("rs_binding", 1)
        if mode == "pull":  # AllGathers in pull mode: each rank reads the peers' tiles from their buffers
            comm.set_option("ag_mode", 1)
        out = torch.empty(M // world, H, device="cuda", dtype=torch.bfloat16)
        comm.mlp_forward(Xs[rank].cuda(), W1s[rank].cuda(), W2s[rank].cuda(), out, act=tl.ACT_SILU_MUL)
        res["mlp"] = out.float().cpu().numpy()
        # MoE (both halves)
        E, topk, Hm, Im = 4, 2, 128, 128 * world
        Xm = TI._randn((M, Hm), 7, 0)
        W1m = TI.moe_weights(E, 2 * (Im // world), Hm, world, seed=8)
        W2m = TI.moe_down_weights(E, Hm, Im // world, world, seed=9)
        ids = TI.moe_routing(M, E, topk, seed=10)
        wts = TI.moe_topk_weights(M, topk, seed=11)
        R = tl.moe_capacity(comm, M, topk, E)
        Y = torch.empty(R, Im // world, device="cuda", dtype=torch.bfloat16)
        rows = torch.empty(R, device="cuda", dtype=torch.int32)
        offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
        mo = torch.empty(M // world, Hm, device="cuda", dtype=torch.bfloat16)
        xm = TI.shard_rows(Xm, world)[rank].cuda()
        tl.moe_ag_gemm(comm, xm, ids.cuda(), W1m[rank].cuda(), Y, rows, offs, act=tl.ACT_SILU_MUL)
        tl.moe_gemm_rs(comm, Y, rows, offs, wts.cuda(), W2m[rank].cuda(), mo)
        res["moe"] = mo.float().cpu().numpy()
        # SP attention
        S, heads = 256 * world, 2
        Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, world, seed=12)
        ao = torch.empty(S // world, heads, 128, device="cuda", dtype=torch.bfloat16)
        tl.sp_attention(comm, Qs[rank].cuda(), Ks[rank].cuda(), Vs[rank].cuda(), ao)
        res["attn"] = ao.float().cpu().numpy()
        st, diag = comm.check()
        q.put((rank, st, res))
        dist.barrier()
        comm.close()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "sm"), (4, "sm"), (2, "dma"), (2, "pull"), (4, "pull"), (8, "sm"),
                                        (8, "pull"), (8, "dma")])
def test_processes_ipc_all_ops(world, mode):
    """Every fused op over real processes (one rank each, CUDA IPC peers): one GPU per rank when the box
    has them (NVLink peer stores / loads, TMA tensor stores into peer-mapped staging, sys-scope flags
    across devices), else the one GPU time-shared (world 8 only runs with 8 devices)."""
    if world > 4 and torch.cuda.device_count() < world:
        pytest.skip(f"world {world} needs {world} devices (cross-device data-plane check)")
    import torch.multiprocessing as mp
    import tl_inputs as TI
    from oracle import tl_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_all, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, st, res = q.get(timeout=900)
        assert st != "error", res
        assert st == 0
        got[rank] = res
    for p in procs:
        p.join(timeout=120)
    f = lambda L: [TI.to_f64(t) for t in L]
    M, H, I = 128 * world, 128, 128 * world
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=6)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, world, TI.ACT_SILU_MUL)
    ref = O.mlp_forward(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL)
    E, topk, Hm, Im = 4, 2, 128, 128 * world
    Xm = TI._randn((M, Hm), 7, 0)
    W1m = TI.moe_weights(E, 2 * (Im // world), Hm, world, seed=8)
    W2m = TI.moe_down_weights(E, Hm, Im // world, world, seed=9)
    ids = TI.moe_routing(M, E, topk, seed=10)
    wts = TI.moe_topk_weights(M, topk, seed=11)
    ref_moe = O.moe_forward(f(TI.shard_rows(Xm, world)), ids.numpy(), wts.double().numpy(), f(W1m), f(W2m),
                            TI.ACT_SILU_MUL)
    S, heads = 256 * world, 2
    Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, world, seed=12)
    ref_att = O.sp_attention(f(Qs), f(Ks), f(Vs), 128 ** -0.5)
    for r in range(world):
        assert_parity(got[r]["mlp"].astype(np.float64), ref[r])
        assert_parity(got[r]["moe"].astype(np.float64), ref_moe[r])
        assert_parity(got[r]["attn"].astype(np.float64), ref_att[r])
