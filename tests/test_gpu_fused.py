"""The fused MLP kernel (option mlp_fused, default on): tl_mlp_forward as ONE persistent launch whose work
list holds the AG + GEMM1 + activation tiles (phase 1) and then the GEMM2 + RS tiles (phase 2); a phase-2
tile waits (acquire) on per-m-block counters that the phase-1 epilogues release once their Z rows are
stored.  The arithmetic of every tile is the two-kernel path's, so the fused layer must be BIT-identical
to mlp_fused = 0 (two launches), and within the bf16 budget of the oracle."""
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


def _inputs(M, H, I, W, act, seed=0):
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=seed)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, act)
    return Xs, W1s, W2s


def _run(tl, c, xs, w1, w2, M, H, W, act):
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    if c.world == 1 and c.local_ranks == 1:
        c.mlp_forward(xs[0], w1[0], w2[0], outs[0], act=act)
        torch.cuda.synchronize()
    else:
        c.mlp_forward_lb(xs, w1, w2, outs, act=act)
    st, diag = c.check()
    assert st == 0, diag
    return outs


def _comm(tl, W, M, H):
    return tl.Comm.single(0, max_M=M, max_H=H) if W == 1 else tl.Comm.loopback(W, 0, max_M=M, max_H=H)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_SILU_MUL, TI.ACT_NONE])
@pytest.mark.parametrize("nsub", [1, 2])
def test_fused_equals_two_kernels(tl, W, act, nsub):
    M, H, I = 256 * W * 2, 384, 192 * W
    Xs, W1s, W2s = _inputs(M, H, I, W, act, seed=W)
    xs, w1, w2 = ([t.cuda() for t in L] for L in (Xs, W1s, W2s))
    c = _comm(tl, W, M, H)
    c.set_option("n_sub", nsub)
    c.set_option("mlp_fused", 0)
    ref = _run(tl, c, xs, w1, w2, M, H, W, act)
    c.set_option("mlp_fused", 2)
    got = _run(tl, c, xs, w1, w2, M, H, W, act)
    for r in range(W):
        assert torch.equal(got[r], ref[r]), f"rank {r}"
    f = lambda L: [TI.to_f64(t) for t in L]
    oracle = np.concatenate(O.mlp_forward(f(Xs), f(W1s), f(W2s), act), 0)
    assert_parity(torch.cat(got).double().cpu().numpy(), oracle)


@pytest.mark.parametrize("W,M", [(1, 1000), (1, 77), (3, 384 * 3), (2, 128 * 2 * 3)])
def test_fused_ragged_shapes(tl, W, M):
    """Ragged M (W = 1: a partial last m-block; W > 1: rank blocks of 128 rows, m-blocks straddling ranks)
    and a ragged N (I/W not a multiple of the tile)."""
    H, I = 200, 264 * W
    act = TI.ACT_SILU_MUL
    Xs, W1s, W2s = _inputs(M, H, I, W, act, seed=M)
    xs, w1, w2 = ([t.cuda() for t in L] for L in (Xs, W1s, W2s))
    c = _comm(tl, W, M, H)
    c.set_option("n_sub", 2)     # the same tile width on both paths (auto may pick per GEMM)
    c.set_option("mlp_fused", 0)
    ref = _run(tl, c, xs, w1, w2, M, H, W, act)
    c.set_option("mlp_fused", 2)
    got = _run(tl, c, xs, w1, w2, M, H, W, act)
    for r in range(W):
        assert torch.equal(got[r], ref[r]), f"rank {r}"


@pytest.mark.parametrize("W", [2, 8])
def test_fused_ring_and_pull(tl, W):
    M, H, I = 512 * W, 256, 128 * W
    act = TI.ACT_SILU_MUL
    Xs, W1s, W2s = _inputs(M, H, I, W, act, seed=11)
    xs, w1, w2 = ([t.cuda() for t in L] for L in (Xs, W1s, W2s))
    c = _comm(tl, W, M, H)
    c.set_option("n_sub", 1)
    for opts in ({"rs_order": 1}, {"ag_mode": 1}, {"rs_order": 1, "ag_mode": 1}):
        for k, v in opts.items():
            c.set_option(k, v)
        c.set_option("mlp_fused", 0)
        ref = _run(tl, c, xs, w1, w2, M, H, W, act)
        c.set_option("mlp_fused", 2)
        got = _run(tl, c, xs, w1, w2, M, H, W, act)
        for r in range(W):
            assert torch.equal(got[r], ref[r]), f"{opts} rank {r}"
        c.set_option("rs_order", 0)
        c.set_option("ag_mode", 0)


def test_fused_many_calls_and_shape_changes(tl):
    """Monotone Z-row counters across calls; a change of M or I resets them; interleaved standalone AG /
    RS calls (separate epochs) do not disturb the fused calls."""
    W, H = 4, 256
    c = tl.Comm.loopback(W, 0, max_M=4096, max_H=H)
    c.set_option("n_sub", 2)
    act = TI.ACT_SILU_MUL
    cases = [(2048, 512), (1024, 512), (2048, 768), (2048, 512)]
    refs = {}
    data = {}
    for M, I in cases:
        Xs, W1s, W2s = _inputs(M, H, I, W, act, seed=M + I)
        data[(M, I)] = [[t.cuda() for t in L] for L in (Xs, W1s, W2s)]
        c.set_option("mlp_fused", 0)
        refs[(M, I)] = _run(tl, c, *data[(M, I)], M, H, W, act)
    c.set_option("mlp_fused", 2)
    for rep in range(6):
        for M, I in cases:
            got = _run(tl, c, *data[(M, I)], M, H, W, act)
            for r in range(W):
                assert torch.equal(got[r], refs[(M, I)][r]), f"rep {rep} M={M} I={I} rank {r}"
            if rep % 2:   # a standalone AG-GEMM in between (advances the AG epoch alone)
                xs = data[(M, I)][0]
                Cs = [torch.empty(M, 64, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
                c.ag_gemm_lb(xs, [torch.zeros(64, H, device="cuda", dtype=torch.bfloat16)] * W, Cs)
                assert c.check()[0] == 0


@pytest.mark.parametrize("W", [2, 4])
def test_fused_bitwise_under_perturbed_schedules(tl, W):
    """Race detection: random delays before every AG notify / consumer wait / RS push / owner
    wait inside the fused launch; the Z-row counter protocol must hold under every interleaving."""
    M, H, I = 1024, 256, 128 * W
    act = TI.ACT_SILU_MUL
    Xs, W1s, W2s = _inputs(M, H, I, W, act, seed=5)
    xs, w1, w2 = ([t.cuda() for t in L] for L in (Xs, W1s, W2s))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    c.set_option("n_sub", 2)
    c.set_option("mlp_fused", 0)
    ref = _run(tl, c, xs, w1, w2, M, H, W, act)
    c.set_option("mlp_fused", 2)
    for d in (1000, 20000):
        c.set_option("debug_delay_ns", d)
        for _ in range(3):
            got = _run(tl, c, xs, w1, w2, M, H, W, act)
            for r in range(W):
                assert torch.equal(got[r], ref[r]), f"delay {d} rank {r}"


def test_fused_full_size_70b_w1(tl):
    """bench.py's N = 1 workload through the fused launch: bitwise equal to the two launches."""
    M, H, I = 8192, 8192, 28672
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    w1 = (torch.randn(2 * I, H, device="cuda", generator=g) * H ** -0.5).bfloat16()
    w2 = (torch.randn(H, I, device="cuda", generator=g) * I ** -0.5).bfloat16()
    c = tl.Comm.single(0, max_M=M, max_H=H)
    c.set_option("n_sub", 2)
    outs = []
    for fused in (0, 2):
        c.set_option("mlp_fused", fused)
        o = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
        c.mlp_forward(x, w1, w2, o, act=tl.ACT_SILU_MUL)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0], outs[1])
