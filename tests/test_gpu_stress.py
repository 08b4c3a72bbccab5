"""Race detection by schedule perturbation (SURVEY §4 test_stress / §5; SPEC S:207 release/acquire
stress): with the debug option "debug_delay_ns" every producer notify, consumer wait and
partial-tile push of every rank sleeps a pseudo-random time keyed by (call, rank, tile), so the
ranks' copy roles, GEMM consumers and reduce-scatter owners interleave differently on every call.
The fused protocol is correct only if no such schedule changes a single output bit: each perturbed
call is compared bitwise with the unperturbed result (the arithmetic and its order are fixed, so any
difference is a read of data that had not arrived, or a lost or stale partial)."""
import pytest
import torch

import tl_inputs as TI

pytestmark = pytest.mark.gpu
DELAYS = (3000, 20000, 100000)   # ns: up to a few tile times, up to many


@pytest.fixture(scope="module")
def tl():
    import paper_2503_20313_b200 as m
    m.lib()
    return m


def _cuda(L):
    return [t.cuda().contiguous() for t in L]


def _ms(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def test_perturbation_is_active(tl):
    """The injected sleeps really happen (a 100 us bound slows a small fused MLP call down)."""
    W, M, H, I = 4, 1024, 512, 2048
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=12)
    Xs, W1s, W2s = (_cuda(L) for L in TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    run = lambda: c.mlp_forward_lb(Xs, W1s, W2s, outs, act=TI.ACT_SILU_MUL)
    run()
    base = min(_ms(run) for _ in range(3))
    c.set_option("debug_delay_ns", 100000)
    slow = min(_ms(run) for _ in range(3))
    assert c.check()[0] == 0
    assert slow > base + 0.05, (base, slow)


@pytest.mark.parametrize("W,ring", [(2, 0), (4, 0), (8, 0), (4, 1), (8, 1), (4, "dma"), (8, "dma")])
def test_mlp_bitwise_under_perturbed_schedules(tl, W, ring):
    M, H, I = 1024, 512, 2048
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=11)
    Xs, W1s, W2s = (_cuda(L) for L in TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    if ring == "dma":                               # both exchanges on the copy engines
        c.set_option("ag_binding", 1)
        c.set_option("rs_binding", 1)
        c.set_option("rs_dma_rows", 128)
    else:
        c.set_option("rs_order", ring)
    c.set_option("comm_tile_rows", 32)            # many small producer tiles: many flags to race on
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.mlp_forward_lb(Xs, W1s, W2s, outs, act=TI.ACT_SILU_MUL)
    assert c.check()[0] == 0
    ref = [o.clone() for o in outs]
    for d in DELAYS:
        c.set_option("debug_delay_ns", d)
        for call in range(3):
            for o in outs:
                o.fill_(float("nan"))
            c.mlp_forward_lb(Xs, W1s, W2s, outs, act=TI.ACT_SILU_MUL)
            st, diag = c.check()
            assert st == 0, diag
            for r in range(W):
                assert torch.equal(outs[r], ref[r]), f"delay {d} call {call} rank {r}"


def test_perturbation_catches_a_missing_acquire(tl):
    """Negative control: with the consumers' flag waits removed (debug_mode 3) the same perturbed
    schedules make the GEMM read X_full rows that have not arrived yet (the bank still holds an older
    call's shards), so the check above has teeth."""
    W, M, N, K = 4, 1024, 256, 512
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("comm_tile_rows", 16)
    sets = []
    for seed in (21, 22):
        As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=seed)
        sets.append((_cuda(As), _cuda(Bs)))
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.ag_gemm_lb(*sets[1], Cs)
    ref = [x.clone() for x in Cs]
    c.ag_gemm_lb(*sets[0], Cs)        # both banks now hold set-0 shards
    c.ag_gemm_lb(*sets[0], Cs)
    c.set_option("debug_mode", 3)
    c.set_option("debug_delay_ns", 100000)
    c.ag_gemm_lb(*sets[1], Cs)        # set 1 without acquires: reads stale set-0 rows
    assert c.check()[0] == 0
    assert any(not torch.equal(Cs[r], ref[r]) for r in range(W))


@pytest.mark.parametrize("W", [4, 8])
def test_ag_gathered_tensor_bitwise_under_perturbed_schedules(tl, W):
    """The gathered X must equal torch.cat of the shards bit for bit whatever the copy schedule."""
    M, N, K = 1024, 256, 512
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=4)
    As, Bs = _cuda(As), _cuda(Bs)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("comm_tile_rows", 16)
    full = torch.cat(As, 0)
    Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    gath = [torch.empty(M, K, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.ag_gemm_lb(As, Bs, Cs, A_gathered=gath)
    ref = [x.clone() for x in Cs]
    for d in DELAYS:
        c.set_option("debug_delay_ns", d)
        for g in gath:
            g.zero_()
        c.ag_gemm_lb(As, Bs, Cs, A_gathered=gath)
        assert c.check()[0] == 0
        for r in range(W):
            assert torch.equal(gath[r], full), f"delay {d} rank {r}: gathered X"
            assert torch.equal(Cs[r], ref[r]), f"delay {d} rank {r}: C"


@pytest.mark.parametrize("W", [2, 4])
def test_moe_layer_bitwise_under_perturbed_schedules(tl, W):
    M, H, I, E, topk = 1024, 512, 1024, 8, 2
    il = I // W
    X = TI._randn((M, H), 3, 0)
    Xs = _cuda(TI.shard_rows(X, W))
    W1s, W2s = _cuda(TI.moe_weights(E, 2 * il, H, W, seed=4)), _cuda(TI.moe_down_weights(E, H, il, W, seed=5))
    ids = TI.moe_routing(M, E, topk, seed=6, skew=1.0)
    wts = TI.moe_topk_weights(M, topk, seed=7)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H, max_topk=topk)
    R = tl.moe_capacity(c, M, topk, E)
    Zg = [torch.empty(R, il, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    rows = [torch.empty(R, device="cuda", dtype=torch.int32) for _ in range(W)]
    offs = [torch.empty(E + 1, device="cuda", dtype=torch.int32) for _ in range(W)]
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    idd, wtd = [ids.cuda() for _ in range(W)], [wts.cuda() for _ in range(W)]

    def run():
        tl.moe_ag_gemm_lb(c, Xs, idd, W1s, Zg, rows, offs, act=TI.ACT_SILU_MUL)
        tl.moe_gemm_rs_lb(c, Zg, rows, offs, wtd, W2s, outs)
        st, diag = c.check()
        assert st == 0, diag
        return [o.clone() for o in outs]
    ref = run()
    for d in DELAYS:
        c.set_option("debug_delay_ns", d)
        for call in range(2):
            got = run()
            for r in range(W):
                assert torch.equal(got[r], ref[r]), f"delay {d} call {call} rank {r}"


@pytest.mark.parametrize("W,s_r", [(2, 512), (4, 512), (4, 200)])
def test_attention_bitwise_under_perturbed_schedules(tl, W, s_r):
    S, heads = s_r * W, 2          # s_r = 200: the ragged (masking) kernel, KV blocks straddling shards
    Qs, Ks, Vs = (_cuda(L) for L in TI.attention_inputs(S, heads, 128, W, seed=8))
    c = tl.Comm.loopback(W, 0, max_M=S, max_H=2 * heads * 128)
    c.set_option("comm_tile_rows", 32)
    outs = [torch.empty_like(q) for q in Qs]
    tl.sp_attention_lb(c, Qs, Ks, Vs, outs)
    assert c.check()[0] == 0
    ref = [o.clone() for o in outs]
    for d in DELAYS:
        c.set_option("debug_delay_ns", d)
        for o in outs:
            o.fill_(float("nan"))
        tl.sp_attention_lb(c, Qs, Ks, Vs, outs)
        st, diag = c.check()
        assert st == 0, diag
        for r in range(W):
            assert torch.equal(outs[r], ref[r]), f"delay {d} rank {r}"


def test_thousand_back_to_back_calls_epoch_isolation(tl):
    """SURVEY §4 test_epochs: 1000 back-to-back fused MLP calls over W = 4 loopback
    ranks, alternating two input sets and interleaving standalone AG-GEMM / GEMM-RS calls (the AG and
    RS epoch counters and banks cycle independently); every call is checked bit for bit against its
    input set's first result."""
    W, M, H, I = 4, 512, 256, 1024
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    sets = []
    for seed in (31, 32):
        X, G, U, W2 = TI.mlp_full(M, H, I, seed=seed)
        sets.append(tuple(_cuda(L) for L in TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)))
    outs = [[torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)] for _ in range(2)]
    Cs = [torch.empty(M, 2 * (I // W), device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    Ps = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    Zs = [torch.zeros(M, I // W, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    got = []
    for i in range(1000):                  # queued back to back: no host synchronisation in the loop
        k = (i * 7 // 3) % 2
        c.mlp_forward_lb(*sets[k], outs[k], act=TI.ACT_SILU_MUL)
        got.append((k, torch.stack(outs[k]).clone()))
        if i % 5 == 0:
            c.ag_gemm_lb(sets[1 - k][0], sets[1 - k][1], Cs)     # an extra AG epoch
        if i % 11 == 0:
            c.gemm_rs_lb(Zs, sets[k][2], Ps)                      # an extra RS epoch
    st, diag = c.check()
    assert st == 0, diag
    first = {}
    for i, (k, o) in enumerate(got):
        if k not in first:
            first[k] = o
        else:
            assert torch.equal(o, first[k]), f"call {i}"
