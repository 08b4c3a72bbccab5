"""AllGather pull mode (option ag_mode = 1; tile_pull_data, "two modes for data
transfer -- pull and push"): every rank's copy role reads each source's producer tiles from that
source's gathered buffer (after the source's own copy of the tile is released) into its own.

SURVEY §8(c) pin 8: push and pull are pure data movement, so the gathered tensor and every output
must be bit-identical between the two modes (and the gathered tensor bit-identical to torch.cat).
World sizes > 1 run as loopback comms (all ranks on the one GPU); the cross-process variant is in
test_gpu_multiproc.py."""
import numpy as np
import pytest
import torch

import tl_inputs as TI
from oracle import tl_oracle as O
from parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tl():
    import paper_2503_20313_b200 as m
    m.lib()
    return m


def _cuda(L):
    return [t.cuda().contiguous() for t in L]


def _ag(tl, c, As, Bs, M, N, K, act, mode):
    c.set_option("ag_mode", mode)
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in As]
    Ag = [torch.zeros(M, K, device="cuda", dtype=torch.bfloat16) for _ in As]
    c.ag_gemm_lb(As, Bs, Cs, Ag, act=act)
    st, diag = c.check()
    assert st == 0, diag
    return Cs, Ag


@pytest.mark.parametrize("W", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
def test_pull_equals_push_bitwise(tl, W, act):
    M, K, N = 256 * W, 320, 192
    As, Bs = TI.ag_gemm_inputs(M, (2 if act else 1) * N, K, W, seed=20 + W)
    As, Bs = _cuda(As), _cuda(Bs)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    push, agp = _ag(tl, c, As, Bs, M, N, K, act, 0)
    pull, agl = _ag(tl, c, As, Bs, M, N, K, act, 1)
    full = torch.cat(As, 0)
    for r in range(W):
        assert torch.equal(agl[r].view(torch.int16), full.view(torch.int16)), f"rank {r}: gathered X (pull)"
        assert torch.equal(pull[r], push[r]), f"rank {r}: C differs between pull and push"
    _, Y = O.ag_gemm([TI.to_f64(a.cpu()) for a in As], [TI.to_f64(b.cpu()) for b in Bs])
    for r in range(W):
        assert_parity(pull[r].double().cpu().numpy(), O.activation(Y[r], act))


@pytest.mark.parametrize("W", [2, 4, 8])
def test_pull_placement_bit_exact(tl, W):
    """The integer placement fixture (SURVEY §8(c) pin 7) in pull mode: exact products."""
    M, K, N = 128 * W * 2, 64, 256
    Xs, Bs = TI.ag_placement_inputs(M, K, N, W)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    Cs, Ag = _ag(tl, c, _cuda(Xs), _cuda(Bs), M, N, K, TI.ACT_NONE, 1)
    _, ref = O.ag_gemm([TI.to_f64(x) for x in Xs], [TI.to_f64(b) for b in Bs])
    for r in range(W):
        assert np.array_equal(Cs[r].double().cpu().numpy(), ref[r])


@pytest.mark.parametrize("tm,ch,cc", [(16, 0, 0), (64, 2, 0), (48, 0, 3), (256, 1, 1)])
def test_pull_decoupling_and_ragged(tl, tm, ch, cc):
    """Communication tile / channels / copy CTAs never change output bits in pull mode either, also with
    producer tiles that do not divide the rank's rows (M/W = 200)."""
    W, M, K, N = 3, 600, 128, 256
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=9)
    As, Bs = _cuda(As), _cuda(Bs)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    ref, _ = _ag(tl, c, As, Bs, M, N, K, TI.ACT_NONE, 0)
    c.set_option("comm_tile_rows", tm)
    c.set_option("channels_per_rank", ch)
    c.set_option("copy_ctas", cc)
    got, _ = _ag(tl, c, As, Bs, M, N, K, TI.ACT_NONE, 1)
    for r in range(W):
        assert torch.equal(got[r], ref[r])


@pytest.mark.parametrize("W", [2, 4, 8])
def test_mlp_pull_equals_push_over_epochs(tl, W):
    """Whole layer, alternating modes and two input sets over 8 calls (bank reuse in pull mode)."""
    M, H, I = 256 * W, 256, 128 * W
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=2)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    x0, w1, w2 = _cuda(Xs), _cuda(W1s), _cuda(W2s)
    x1 = [(-t.float()).bfloat16() for t in x0]
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    outs = {}
    for call in range(8):
        mode, xi = call % 2, (x0, x1)[(call // 2) % 2]
        c.set_option("ag_mode", mode)
        o = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        c.mlp_forward_lb(xi, w1, w2, o, act=TI.ACT_SILU_MUL)
        assert c.check()[0] == 0
        key = (call // 2) % 2
        if key in outs:
            assert all(torch.equal(a, b) for a, b in zip(o, outs[key])), f"call {call}"
        else:
            outs[key] = o
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = np.concatenate(O.mlp_forward(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL), 0)
    assert_parity(torch.cat(outs[0]).double().cpu().numpy(), ref)


def test_pull_dropped_notify_times_out(tl):
    """Fault injection in pull mode: source rank 0 withholds its own notify of tile 1; every waiter on
    it (the puller on rank 1, rank 0's own consumers) gives up with a diagnostic instead of hanging."""
    W, M, K, N = 2, 512, 64, 128
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=1)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("ag_mode", 1)
    c.set_option("timeout_ms", 200)
    c.set_option("debug_drop_rank", 0)
    c.set_option("debug_drop_notify", 1)
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.ag_gemm_lb(_cuda(As), _cuda(Bs), Cs)
    st, diag = c.check()
    assert st == 4
    _, rank, kind, src, index, observed, expected, epoch = diag
    assert rank in (0, 1) and (kind, src, index) == (1, 0, 1) and observed < expected
    c.set_option("debug_drop_notify", -1)
    c.set_option("timeout_ms", 10000)
    c.ag_gemm_lb(_cuda(As), _cuda(Bs), Cs)
    assert c.check()[0] == 0


def test_pull_with_copy_engine_binding_rejected(tl):
    c = tl.Comm.loopback(2, 0, max_M=512, max_H=64)
    c.set_option("ag_mode", 1)
    c.set_option("ag_binding", 1)
    As, Bs = TI.ag_gemm_inputs(512, 128, 64, 2, seed=1)
    Cs = [torch.empty(512, 128, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    with pytest.raises(tl.TLError, match="UNSUPPORTED"):
        c.ag_gemm_lb(_cuda(As), _cuda(Bs), Cs)


@pytest.mark.parametrize("W", [2, 4])
def test_pull_bitwise_under_perturbed_schedules(tl, W):
    """Race detection: random delays before every pull wait / notify / consumer wait."""
    M, N, K = 1024, 256, 512
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=4)
    As, Bs = _cuda(As), _cuda(Bs)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("comm_tile_rows", 16)
    ref, _ = _ag(tl, c, As, Bs, M, N, K, TI.ACT_NONE, 0)
    full = torch.cat(As, 0)
    for d in (2000, 20000):
        c.set_option("debug_delay_ns", d)
        got, ag = _ag(tl, c, As, Bs, M, N, K, TI.ACT_NONE, 1)
        for r in range(W):
            assert torch.equal(ag[r], full) and torch.equal(got[r], ref[r]), f"delay {d} rank {r}"


@pytest.mark.parametrize("W", [2, 4])
def test_attention_pull_equals_push(tl, W):
    S, heads = 256 * W, 2
    Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, W, seed=3)
    qd, kd, vd = _cuda(Qs), _cuda(Ks), _cuda(Vs)
    c = tl.Comm.loopback(W, 0, max_M=max(128, 2 * S * heads * 128 // 4096), max_H=4096)
    res = []
    for mode in (0, 1):
        c.set_option("ag_mode", mode)
        o = [torch.empty_like(q) for q in qd]
        tl.sp_attention_lb(c, qd, kd, vd, o)
        assert c.check()[0] == 0
        res.append(o)
    for r in range(W):
        assert torch.equal(res[0][r], res[1][r])


@pytest.mark.parametrize("W", [2, 4])
def test_moe_pull_equals_push(tl, W):
    M, H, E, topk, N_out = 256 * W, 192, 8, 2, 320
    X = TI._randn((M, H), 5, 0)
    Xs = _cuda(TI.shard_rows(X, W))
    Ws = _cuda(TI.moe_weights(E, 2 * N_out, H, W, seed=6))
    ids = TI.moe_routing(M, E, topk, seed=7)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    R = tl.moe_capacity(c, M, topk, E)
    res = []
    for mode in (0, 1):
        c.set_option("ag_mode", mode)
        Ys = [torch.empty(R, N_out, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        rows = [torch.empty(R, device="cuda", dtype=torch.int32) for _ in range(W)]
        offs = [torch.empty(E + 1, device="cuda", dtype=torch.int32) for _ in range(W)]
        tl.moe_ag_gemm_lb(c, Xs, [ids.cuda() for _ in range(W)], Ws, Ys, rows, offs, act=TI.ACT_SILU_MUL)
        assert c.check()[0] == 0
        res.append((Ys, rows, offs))
    for r in range(W):
        n = int(res[0][2][r][-1])           # grouped rows written (padded groups); the rest is untouched
        assert n > 0 and torch.equal(res[0][2][r], res[1][2][r])
        assert torch.equal(res[0][1][r][:n], res[1][1][r][:n])
        assert torch.equal(res[0][0][r][:n], res[1][0][r][:n])
