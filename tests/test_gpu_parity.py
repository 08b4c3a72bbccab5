"""GPU parity of the CUDA path (through the C ABI) against the fp64 CPU oracle.

World sizes > 1 run as a loopback comm: all W ranks on the one GPU, driven by one launch, so
the flag protocol, peer pushes and owner reductions execute exactly as across NVLink (peer
stores land in local memory).  Tolerance: relative Frobenius <= 5e-3 (BASELINE.json north
star) for random inputs; bit-exact for the integer placement fixtures and the gathered tensor.
"""
import numpy as np
import pytest
import torch

import tl_inputs as TI
from oracle import tl_oracle as O
from parity import assert_parity

pytestmark = pytest.mark.gpu
TOL = 5e-3


@pytest.fixture(scope="module")
def tl():
    import paper_2503_20313_b200 as m
    m.lib()
    return m


def cuda(t):
    return t.to("cuda").contiguous()


def f64(t):
    return t.detach().to("cpu", torch.float64).numpy()


def empty(*shape):
    return torch.empty(*shape, device="cuda", dtype=torch.bfloat16)


# ----------------------------------------------------------------------------- W = 1 GEMM core
@pytest.mark.parametrize("pair,nsub", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (1000, 2752, 1376), (384, 520, 4096), (8, 16, 8)])
def test_gemm_w1_plain(tl, pair, nsub, M, N, K):
    A, Bs = TI.ag_gemm_inputs(M, N, K, 1, seed=M + N)
    c = tl.Comm.single(0, max_M=M, max_H=K)
    c.set_option("cta_pair", pair)
    c.set_option("n_sub", nsub)
    C = empty(M, N)
    c.ag_gemm(cuda(A[0]), cuda(Bs[0]), C)
    torch.cuda.synchronize()
    _, ref = O.ag_gemm([TI.to_f64(A[0])], [TI.to_f64(Bs[0])])
    assert_parity(f64(C), ref[0])


@pytest.mark.parametrize("pair,nsub", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("act", [TI.ACT_SILU_MUL, TI.ACT_GELU_TANH_MUL])
@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (1000, 1376, 520)])
def test_gemm_w1_gated(tl, pair, nsub, act, M, N, K):
    A, Bs = TI.ag_gemm_inputs(M, 2 * N, K, 1, seed=7)
    c = tl.Comm.single(0, max_M=M, max_H=K)
    c.set_option("cta_pair", pair)
    c.set_option("n_sub", nsub)
    C = empty(M, N)
    c.ag_gemm(cuda(A[0]), cuda(Bs[0]), C, act=act)
    torch.cuda.synchronize()
    _, Y = O.ag_gemm([TI.to_f64(A[0])], [TI.to_f64(Bs[0])])
    ref = O.activation(Y[0], act)
    assert_parity(f64(C), ref)


def test_gemm_k0_and_empty(tl):
    c = tl.Comm.single(0, max_M=256, max_H=256)
    A = torch.empty(256, 0, device="cuda", dtype=torch.bfloat16)
    B = torch.empty(64, 0, device="cuda", dtype=torch.bfloat16)
    C = torch.full((256, 64), 3.0, device="cuda", dtype=torch.bfloat16)
    c.ag_gemm(A, B, C)
    torch.cuda.synchronize()
    assert torch.count_nonzero(C).item() == 0
    # M = 0 is a no-op
    c.ag_gemm(torch.empty(0, 64, device="cuda", dtype=torch.bfloat16), cuda(torch.ones(8, 64).bfloat16()),
              torch.empty(0, 8, device="cuda", dtype=torch.bfloat16))


# ----------------------------------------------------------------------------- validation
def test_validation_errors(tl):
    from paper_2503_20313_b200 import TLError
    c = tl.Comm.loopback(2, 0, max_M=512, max_H=256)
    As = [cuda(torch.zeros(128, 64).bfloat16()) for _ in range(2)]
    Bs = [cuda(torch.zeros(64, 64).bfloat16()) for _ in range(2)]
    Cs = [empty(128, 64) for _ in range(2)]
    with pytest.raises(TLError, match="UNSUPPORTED"):     # M/W = 64 not a multiple of 128
        c.gemm_rs_lb(As, Bs, [empty(64, 64) for _ in range(2)])
    with pytest.raises(TLError, match="INVALID"):          # over capacity
        c.ag_gemm_lb([cuda(torch.zeros(512, 64).bfloat16())] * 2, Bs, [empty(1024, 64)] * 2)
    with pytest.raises(TLError, match="INVALID"):          # misaligned pointer
        big = empty(64 * 64 + 8)
        c.ag_gemm_lb([big[1:1 + 64 * 64].view(64, 64)] * 2, Bs, Cs)
    with pytest.raises(TLError, match="INVALID"):
        c.set_option("rs_order", 7)


# ----------------------------------------------------------------------------- AG-GEMM (loopback W)
@pytest.mark.parametrize("W", [2, 4, 8])
def test_ag_gemm_placement_bit_exact(tl, W):
    M, K, N = 128 * W * 2, 64, 256
    Xs, Bs = TI.ag_placement_inputs(M, K, N, W)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    Cs = [empty(M, N) for _ in range(W)]
    Ag = [empty(M, K) for _ in range(W)]
    c.ag_gemm_lb([cuda(x) for x in Xs], [cuda(b) for b in Bs], Cs, Ag)
    st, diag = c.check()
    assert st == 0, diag
    X, ref = O.ag_gemm([TI.to_f64(x) for x in Xs], [TI.to_f64(b) for b in Bs])
    full = torch.cat(Xs, 0)
    for r in range(W):
        assert torch.equal(Ag[r].cpu().view(torch.int16), full.view(torch.int16))   # gathered tensor, bitwise
        assert np.array_equal(f64(Cs[r]), ref[r])                                    # integer products, exact


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
@pytest.mark.parametrize("nsub", [1, 2])
def test_ag_gemm_random(tl, W, act, nsub):
    M, K, N = 256 * W, 320, 200 if act else 392
    As, Bs = TI.ag_gemm_inputs(M, (2 if act else 1) * N, K, W, seed=W)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("n_sub", nsub)
    Cs = [empty(M, N) for _ in range(W)]
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs, act=act)
    st, diag = c.check()
    assert st == 0, diag
    _, Y = O.ag_gemm([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    for r in range(W):
        assert_parity(f64(Cs[r]), O.activation(Y[r], act))


@pytest.mark.parametrize("W", [2, 3])
def test_ag_gemm_ragged_rank_rows(tl, W):
    # M/W not a multiple of the tile: consumer tiles straddle ranks and wait on both
    M, K, N = 200 * W, 64, 128
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=11)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("comm_tile_rows", 48)
    Cs = [empty(M, N) for _ in range(W)]
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    st, diag = c.check()
    assert st == 0, diag
    _, Y = O.ag_gemm([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    for r in range(W):
        assert_parity(f64(Cs[r]), Y[r])


def test_ag_decoupling_soundness(tl):
    """Changing only the communication tile / channel count never changes output bits."""
    W, M, K, N = 4, 1024, 256, 256
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=5)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    A_d, B_d = [cuda(a) for a in As], [cuda(b) for b in Bs]
    outs = []
    for tm, ch, cc in [(64, 0, 0), (16, 0, 0), (128, 1, 0), (32, 2, 3), (256, 0, 1)]:
        c.set_option("comm_tile_rows", tm)
        c.set_option("channels_per_rank", ch)
        c.set_option("copy_ctas", cc)
        Cs = [empty(M, N) for _ in range(W)]
        c.ag_gemm_lb(A_d, B_d, Cs)
        st, diag = c.check()
        assert st == 0, diag
        outs.append([x.clone() for x in Cs])
    for o in outs[1:]:
        for r in range(W):
            assert torch.equal(o[r], outs[0][r])


# ----------------------------------------------------------------------------- GEMM-RS (loopback W)
@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("ring", [0, 1])
@pytest.mark.parametrize("nsub", [1, 2])
def test_gemm_rs_placement_bit_exact(tl, W, ring, nsub):
    M, N, K = 128 * W, 520, 32
    As, Bs = TI.rs_placement_inputs(M, N, K, W)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    c.set_option("rs_order", ring)
    c.set_option("n_sub", nsub)
    Cs = [empty(M // W, N) for _ in range(W)]
    c.gemm_rs_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    st, diag = c.check()
    assert st == 0, diag
    ref = O.gemm_rs([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    for r in range(W):
        assert np.array_equal(f64(Cs[r]), ref[r]), f"rank {r}"


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("ring", [0, 1])
@pytest.mark.parametrize("nsub", [1, 2])
def test_gemm_rs_random(tl, W, ring, nsub):
    M, N, K = 256 * W, 392 if nsub == 1 else 1032, 1376 // 4
    As, Bs = TI.gemm_rs_inputs(M, N, K, W, seed=3)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    c.set_option("rs_order", ring)
    c.set_option("n_sub", nsub)
    Cs = [empty(M // W, N) for _ in range(W)]
    c.gemm_rs_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    st, diag = c.check()
    assert st == 0, diag
    ref = O.gemm_rs([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    got = np.concatenate([f64(x) for x in Cs], 0)
    assert_parity(got, np.concatenate(ref, 0))


def test_gemm_rs_deterministic(tl):
    W, M, N, K = 4, 1024, 512, 256
    As, Bs = TI.gemm_rs_inputs(M, N, K, W, seed=9)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    A_d, B_d = [cuda(a) for a in As], [cuda(b) for b in Bs]
    first = None
    for _ in range(5):
        Cs = [empty(M // W, N) for _ in range(W)]
        c.gemm_rs_lb(A_d, B_d, Cs)
        if first is None:
            first = [x.clone() for x in Cs]
        else:
            for r in range(W):
                assert torch.equal(Cs[r], first[r])


# ----------------------------------------------------------------------------- MLP (the layer)
def _mlp_case(tl, W, M, H, I, act, pair=2, seed=0, nsub=0):
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=seed)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, act)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H) if W > 1 else tl.Comm.single(0, max_M=M, max_H=H)
    c.set_option("cta_pair", pair)
    c.set_option("n_sub", nsub)
    outs = [empty(M // W, H) for _ in range(W)]
    if W > 1:
        c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs, act=act)
        st, diag = c.check()
        assert st == 0, diag
    else:
        c.mlp_forward(cuda(Xs[0]), cuda(W1s[0]), cuda(W2s[0]), outs[0], act=act)
        torch.cuda.synchronize()
    return Xs, W1s, W2s, outs


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL, TI.ACT_GELU_TANH_MUL])
@pytest.mark.parametrize("nsub", [1, 2])
def test_mlp_tiny_config(tl, W, act, nsub):
    """BASELINE.json configs[0]: M=256 tokens, hidden 128, ffn 512 (W=2 in the config; all W here)."""
    M, H, I = 256 * W if W > 2 else 256, 128, 512
    Xs, W1s, W2s, outs = _mlp_case(tl, W, M, H, I, act, nsub=nsub)
    ref = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s], [TI.to_f64(w) for w in W2s], act)
    got = np.concatenate([f64(o) for o in outs], 0)
    assert_parity(got, np.concatenate(ref, 0))


def test_mlp_hand_example_padded_bit_exact(tl, golden_dir):
    """The hand-computed W=2 example (tests/golden/hand_example_w2.json), zero-padded to the
    kernel's granularity (M/W = 128, H = 64, I/W = 64): the valid block must be bit-exact."""
    import json, os
    g = json.load(open(os.path.join(golden_dir, "hand_example_w2.json")))
    W, Mr, H, Il = 2, 128, 64, 64
    Xs = [torch.zeros(Mr, H) for _ in range(W)]
    W1 = [torch.zeros(Il, H) for _ in range(W)]
    W2 = [torch.zeros(H, Il) for _ in range(W)]
    for r in range(W):
        Xs[r][:2, :2] = torch.tensor(g["X_shards"][r], dtype=torch.float32)
        W1[r][:2, :2] = torch.tensor(g["W1"][r], dtype=torch.float32)
        W2[r][:2, :2] = torch.tensor(g["W2"][r], dtype=torch.float32)
    c = tl.Comm.loopback(W, 0, max_M=W * Mr, max_H=H)
    outs = [empty(Mr, H) for _ in range(W)]
    c.mlp_forward_lb([cuda(x.bfloat16()) for x in Xs], [cuda(w.bfloat16()) for w in W1],
                     [cuda(w.bfloat16()) for w in W2], outs, act=TI.ACT_NONE)
    assert c.check()[0] == 0
    for r in range(W):
        o = outs[r].float().cpu()
        assert torch.equal(o[:2, :2], torch.tensor(g["out"][r], dtype=torch.float32))
        assert torch.count_nonzero(o[2:]).item() == 0 and torch.count_nonzero(o[:, 2:]).item() == 0


def test_mlp_epoch_isolation(tl):
    """Back-to-back calls alternating two input sets (AG and RS banks and flag epochs cycle):
    every call must reproduce its input set's first result bit for bit."""
    W, M, H, I = 4, 512, 256, 1024
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    sets = []
    for seed in (1, 2):
        X, G, U, W2 = TI.mlp_full(M, H, I, seed=seed)
        Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
        sets.append(([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s]))
    first = {}
    for i in range(40):
        k = i % 2 if i < 20 else (i // 3) % 2
        outs = [empty(M // W, H) for _ in range(W)]
        c.mlp_forward_lb(*sets[k], outs, act=TI.ACT_SILU_MUL)
        if i % 7 == 0:  # also interleave a standalone AG and RS call (separate epoch counters)
            Cs = [empty(M, 2 * (I // W)) for _ in range(W)]
            c.ag_gemm_lb(sets[k][0], sets[k][1], Cs)
        if k not in first:
            first[k] = [o.clone() for o in outs]
        else:
            for r in range(W):
                assert torch.equal(outs[r], first[k][r]), f"call {i} rank {r}"
    assert c.check()[0] == 0


# ----------------------------------------------------------------------------- failure detection
def test_dropped_notify_times_out_with_diag(tl):
    W, M, K, N = 2, 512, 64, 128
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=1)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("timeout_ms", 200)
    c.set_option("debug_drop_rank", 0)
    c.set_option("debug_drop_notify", 1)
    Cs = [empty(M, N) for _ in range(W)]
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    st, diag = c.check()
    assert st == 4  # TL_ERR_TIMEOUT
    status, rank, kind, src, index, observed, expected, epoch = diag
    assert (rank, kind, src, index) == (1, 1, 0, 1)
    assert observed < expected == epoch
    # the comm keeps working once the fault is removed
    c.set_option("debug_drop_notify", -1)
    c.set_option("timeout_ms", 10000)
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    assert c.check()[0] == 0


# ----------------------------------------------------------------------------- static mapping index test
@pytest.mark.parametrize("M,R,C,Tm", [(8192, 8, 4, 128), (8192, 8, 8, 128), (4096, 4, 2, 64), (256, 2, 1, 128)])
def test_device_static_map_matches_paper_formula(tl, M, R, C, Tm):
    n = M // Tm
    dev = tl.static_map_device(M, R, Tm, C, n)
    for t in range(n):
        lo, hi = O.static_shape_range(t, M, Tm)
        assert dev[t] == (lo, hi, O.static_src_rank(t, M, R, Tm), O.static_channel(t, M, R, C, Tm))


@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
def test_split_tail_items(tl, act):
    """512-wide tiles whose last wave is at most half full run as 256-wide half items
    (M=8192, N=4096 -> 256 tiles on 74 pairs: 222 whole tiles + 68 half items)."""
    M, N, K = 8192, 4096 if act == TI.ACT_NONE else 2048, 256
    A, Bs = TI.ag_gemm_inputs(M, (2 if act else 1) * N, K, 1, seed=21)
    c = tl.Comm.single(0, max_M=M, max_H=K)
    c.set_option("n_sub", 2)
    C = empty(M, N)
    c.ag_gemm(cuda(A[0]), cuda(Bs[0]), C, act=act)
    torch.cuda.synchronize()
    _, Y = O.ag_gemm([TI.to_f64(A[0])], [TI.to_f64(Bs[0])])
    assert_parity(f64(C), O.activation(Y[0], act))


# ----------------------------------------------------------------------------- copy-engine AG binding (NEXT-1)
@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
def test_ag_dma_binding_parity(tl, W, act):
    """AllGather on the copy engines (cudaMemcpyAsync + stream write-value flags, the paper's
    benchmarked binding) feeding the same consumer waits: placement bit-exact + parity."""
    M, K, N = 256 * W, 320, 200 if act else 392
    As, Bs = TI.ag_gemm_inputs(M, (2 if act else 1) * N, K, W, seed=W + 40)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("ag_binding", 1)
    Cs = [empty(M, N) for _ in range(W)]
    Ag = [empty(M, K) for _ in range(W)]
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs, Ag, act=act)
    st, diag = c.check()
    assert st == 0, diag
    full = torch.cat(As, 0)
    _, Y = O.ag_gemm([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    for r in range(W):
        assert torch.equal(Ag[r].cpu().view(torch.int16), full.view(torch.int16))
        assert_parity(f64(Cs[r]), O.activation(Y[r], act))


def test_ag_dma_binding_matches_sm_binding_and_epochs(tl):
    W, M, H, I = 4, 1024, 256, 1024
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=8)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    args = ([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s])
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    ref = [empty(M // W, H) for _ in range(W)]
    c.mlp_forward_lb(*args, ref, act=TI.ACT_SILU_MUL)
    c.set_option("ag_binding", 1)
    for i in range(12):   # banks and epochs cycle; DMA and SM bindings give identical bits
        outs = [empty(M // W, H) for _ in range(W)]
        c.set_option("dma_tile_rows", [0, 64, 128][i % 3])
        c.mlp_forward_lb(*args, outs, act=TI.ACT_SILU_MUL)
        for r in range(W):
            assert torch.equal(outs[r], ref[r]), f"call {i} rank {r}"
    assert c.check()[0] == 0


def test_ag_dma_dropped_notify_times_out(tl):
    W, M, K, N = 2, 512, 64, 128
    As, Bs = TI.ag_gemm_inputs(M, N, K, W, seed=2)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=K)
    c.set_option("ag_binding", 1)
    c.set_option("timeout_ms", 200)
    c.set_option("debug_drop_rank", 1)
    c.set_option("debug_drop_notify", 0)
    Cs = [empty(M, N) for _ in range(W)]
    c.ag_gemm_lb([cuda(a) for a in As], [cuda(b) for b in Bs], Cs)
    st, diag = c.check()
    assert st == 4
    assert diag[1:5] == [0, 1, 1, 0]   # waiting rank 0, AG wait, source rank 1, producer tile 0


# ----------------------------------------------------------------------------- full-size sampled parity
@pytest.mark.parametrize("name,M,H,I,W,block", [
    ("llama70b", 8192, 8192, 28672, 1, 0),    # bench.py's default N=1 workload and launch configuration
    ("llama7b", 8192, 4096, 11008, 1, 0),
    ("llama7b", 8192, 4096, 11008, 8, 3),     # BASELINE configs[1] (8 ranks, loopback): rank 3's whole block
    ("llama70b", 8192, 8192, 28672, 2, None),  # configs[2] at W=2
    ("mixtral", 16384, 4096, 14336, 4, None),  # configs[3] at W=4
    ("llama7b_M32768", 32768, 4096, 11008, 1, None),  # configs[4] M sweep, largest M
    ("llama7b_M1024", 1024, 4096, 11008, 8, 5),       # configs[4] M sweep, smallest M at 8 ranks (128 rows/rank)
])
def test_full_size_sampled_rows(tl, name, M, H, I, W, block):
    """Full BASELINE.json sizes; the oracle is evaluated exactly on sampled rows (rows are
    independent): rows spread over every rank's output block, the first 128-row tile, and (block =
    rank index) one rank's whole output block -- every tile of it checked element-wise."""
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=0)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    del X, G, U, W2
    Mr = M // W
    outs = [empty(Mr, H) for _ in range(W)]
    if W == 1:
        c = tl.Comm.single(0, max_M=M, max_H=H)
        c.mlp_forward(cuda(Xs[0]), cuda(W1s[0]), cuda(W2s[0]), outs[0], act=TI.ACT_SILU_MUL)
        torch.cuda.synchronize()
    else:
        c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
        c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs,
                         act=TI.ACT_SILU_MUL)
        assert c.check()[0] == 0
    rows = {r * Mr + o for r in range(W) for o in (0, Mr // 2, Mr - 1)} | {M // 3, 2 * M // 3} | set(range(128))
    if block is not None:
        rows |= set(range(block * Mr, (block + 1) * Mr))
    rows = sorted(rows)
    ref = O.mlp_forward_rows([TI.to_f64(t) for t in Xs], [TI.to_f64(t) for t in W1s], [TI.to_f64(t) for t in W2s],
                             TI.ACT_SILU_MUL, rows)
    full = torch.cat(outs).float().cpu().double().numpy()
    assert_parity(full[rows], np.stack([ref[i] for i in rows]))
    if block is not None:   # the whole block again on its own, tiles aligned to the block
        b = list(range(block * Mr, (block + 1) * Mr))
        assert_parity(full[b], np.stack([ref[i] for i in b]))
    del c


# ----------------------------------------------------------------------------- odd worlds / option matrix
@pytest.mark.parametrize("W", [3, 5, 6, 7])
@pytest.mark.parametrize("ring", [0, 1])
def test_mlp_odd_worlds(tl, W, ring):
    """Non-power-of-two world sizes (ring successor/predecessor arithmetic, rotations, 128-row owner
    blocks that straddle 256-row pair tiles when M/W is an odd multiple of 128)."""
    M, H, I = 128 * W * (1 if W % 2 else 2), 192, 96 * W
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=W)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    c.set_option("rs_order", ring)
    outs = [empty(M // W, H) for _ in range(W)]
    c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs,
                     act=TI.ACT_SILU_MUL)
    st, diag = c.check()
    assert st == 0, diag
    ref = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s], [TI.to_f64(w) for w in W2s],
                        TI.ACT_SILU_MUL)
    assert_parity(np.concatenate([f64(o) for o in outs], 0), np.concatenate(ref, 0))


@pytest.mark.parametrize("opts", [
    {"cta_pair": 1},
    {"n_sub": 2, "ag_binding": 1},
    {"n_sub": 1, "rs_order": 1, "comm_tile_rows": 16},
    {"n_sub": 2, "rs_order": 1, "channels_per_rank": 1, "copy_ctas": 2},
    {"raster_group": 1, "num_ctas": 8},
    {"raster_group": 3, "num_ctas": 30, "n_sub": 2},
])
def test_mlp_option_matrix(tl, opts):
    W, M, H, I = 4, 1024, 320, 1536
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=11)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    for k, v in opts.items():
        c.set_option(k, v)
    outs = [empty(M // W, H) for _ in range(W)]
    for _ in range(3):
        c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs,
                         act=TI.ACT_SILU_MUL)
    st, diag = c.check()
    assert st == 0, diag
    ref = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s], [TI.to_f64(w) for w in W2s],
                        TI.ACT_SILU_MUL)
    assert_parity(np.concatenate([f64(o) for o in outs], 0), np.concatenate(ref, 0))


def test_small_m_many_ranks(tl):
    """M/W = 128 at W = 8 (the M = 1024 point of the M sweep): one CTA tile per owner block."""
    W, M, H, I = 8, 1024, 256, 2048
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=13)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    outs = [empty(M // W, H) for _ in range(W)]
    c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs,
                     act=TI.ACT_SILU_MUL)
    assert c.check()[0] == 0
    ref = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s], [TI.to_f64(w) for w in W2s],
                        TI.ACT_SILU_MUL)
    assert_parity(np.concatenate([f64(o) for o in outs], 0), np.concatenate(ref, 0))


def test_binding_shape_and_dtype_checks(tl):
    """Shape / dtype / layout mistakes are caught in the binding (ValueError), not by a kernel."""
    c = tl.Comm.single(0, max_M=512, max_H=256)
    X, W1, W2 = empty(256, 128), empty(2 * 64, 128), empty(128, 64)
    out = empty(256, 128)
    c.mlp_forward(X, W1, W2, out, act=tl.ACT_SILU_MUL)                   # consistent: runs
    assert c.check()[0] == 0
    with pytest.raises(ValueError, match="shape"):
        c.mlp_forward(X, empty(64, 128), W2, out, act=tl.ACT_SILU_MUL)     # W1 must be [2*I_l, H] gated
    with pytest.raises(ValueError, match="bfloat16"):
        c.mlp_forward(X.float(), W1, W2, out)
    with pytest.raises(ValueError, match="contiguous"):
        c.gemm_rs(empty(256, 128).t(), empty(64, 256), empty(128, 64))
    with pytest.raises(ValueError, match="shape"):
        c.ag_gemm(X, empty(64, 128), empty(256, 32))                      # B rows != C cols


@pytest.mark.parametrize("W", [2, 4, 8])
def test_rs_dma_binding_matches_sm_binding(tl, W):
    """GEMM-RS with the paper's hybrid binding (scatter on the copy engines, reduction on SMs,
    rs_binding = 1): partial tiles go to a local outbox, the copy engines move each finished chunk to
    its owner after a stream wait on the kernel's chunk flag, and the owner reduces exactly as in the
    SM binding -> bitwise-identical results over epoch-cycling calls, for whole-block and 128-row
    chunks, plus parity with the oracle."""
    M, N, K = 256 * W, 384, 192
    As, Bs = TI.gemm_rs_inputs(M, N, K, W, seed=W + 60)
    a, b = [cuda(x) for x in As], [cuda(x) for x in Bs]
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    ref = [empty(M // W, N) for _ in range(W)]
    c.gemm_rs_lb(a, b, ref)
    assert c.check()[0] == 0
    c.set_option("rs_binding", 1)
    for i, rows in enumerate([0, 128, 0, 256]):
        c.set_option("rs_dma_rows", rows)
        outs = [empty(M // W, N) for _ in range(W)]
        c.gemm_rs_lb(a, b, outs)
        st, diag = c.check()
        assert st == 0, diag
        for r in range(W):
            assert torch.equal(outs[r], ref[r]), f"call {i} rank {r}"
    oracle = O.gemm_rs([TI.to_f64(x) for x in As], [TI.to_f64(x) for x in Bs])
    got = np.concatenate([f64(o) for o in ref], 0)
    assert_parity(got, np.concatenate(oracle, 0))


def test_mlp_both_dma_bindings(tl):
    """The whole layer with AllGather and scatter both on the copy engines (the paper's benchmarked
    bindings) equals the all-SM layer bit for bit."""
    W, M, H, I = 4, 1024, 256, 1024
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=9)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    args = ([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s])
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    ref = [empty(M // W, H) for _ in range(W)]
    c.mlp_forward_lb(*args, ref, act=TI.ACT_SILU_MUL)
    c.set_option("ag_binding", 1)
    c.set_option("rs_binding", 1)
    for i in range(4):
        outs = [empty(M // W, H) for _ in range(W)]
        c.mlp_forward_lb(*args, outs, act=TI.ACT_SILU_MUL)
        for r in range(W):
            assert torch.equal(outs[r], ref[r]), f"call {i} rank {r}"
    assert c.check()[0] == 0


@pytest.mark.parametrize("W,M,N", [(2, 2048, 2048), (4, 2048, 1536), (8, 4096, 4096)])
def test_rs_dma_binding_many_items_per_cta(tl, W, M, N):
    """Shapes where CTAs own several items: with the copy-engine scatter a chunk needs all of its
    remote tiles, so the schedule must run every remote tile before any own-block tile (an
    interleaved raster deadlocked here); bitwise equal to the SM binding."""
    K = 192
    As, Bs = TI.gemm_rs_inputs(M, N, K, W, seed=W + 70)
    a, b = [cuda(x) for x in As], [cuda(x) for x in Bs]
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=N)
    ref = [empty(M // W, N) for _ in range(W)]
    c.gemm_rs_lb(a, b, ref)
    c.set_option("rs_binding", 1)
    c.set_option("timeout_ms", 5000)
    for rows in (0, 128):
        c.set_option("rs_dma_rows", rows)
        outs = [empty(M // W, N) for _ in range(W)]
        c.gemm_rs_lb(a, b, outs)
        st, diag = c.check()
        assert st == 0, diag
        for r in range(W):
            assert torch.equal(outs[r], ref[r])


def test_debug_options_not_read_from_env(tl, monkeypatch):
    """The fault-injection / debug switches change results on purpose, so the environment cannot turn
    them on (only tl_set_option can); the tunables are still read from TL_<KEY>."""
    monkeypatch.setenv("TL_DEBUG_MODE", "3")
    monkeypatch.setenv("TL_DEBUG_DELAY_NS", "1000")
    monkeypatch.setenv("TL_DEBUG_DROP_NOTIFY", "0")
    monkeypatch.setenv("TL_COMM_TILE_ROWS", "128")
    c = tl.Comm.single(0, max_M=256, max_H=128)
    assert c.get_option("debug_mode") == 0 and c.get_option("debug_delay_ns") == 0
    assert c.get_option("debug_drop_notify") == -1
    assert c.get_option("comm_tile_rows") == 128
    c.close()


def test_parity_check_rejects_a_corrupted_gpu_tile(tl):
    """Negative control on real GPU output: the element-wise parity check of every GPU test accepts the
    fused layer's output and rejects the same output with ONE 128 x 256 tile scaled by 1 % (which the
    global relative-Frobenius norm alone accepts)."""
    from parity import parity_report
    W, M, H, I = 4, 2048, 1024, 2048
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=21)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    outs = [empty(M // W, H) for _ in range(W)]
    c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs, act=TI.ACT_SILU_MUL)
    assert c.check()[0] == 0
    ref = np.concatenate(O.mlp_forward([TI.to_f64(t) for t in Xs], [TI.to_f64(t) for t in W1s],
                                       [TI.to_f64(t) for t in W2s], TI.ACT_SILU_MUL), 0)
    got = torch.cat(outs).double().cpu().numpy()
    assert parity_report(got, ref)["ok"]
    bad = got.copy()
    bad[640:768, 512:768] *= 1.01
    rep = parity_report(bad, ref)
    assert not rep["ok"] and rep["worst_tile"] == (640, 512) and rep["global"] < TOL


@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_GELU_TANH_MUL])
@pytest.mark.parametrize("W", [1, 8])
def test_full_size_other_activations(tl, act, W):
    """The LLaMA-7B layer (M = 8192) with the two other activations of R1/R2 (identity: GEMM1 is I/W wide;
    GeLU(tanh)*up), at W = 1 and over 8 loopback ranks: sampled rows of every rank's block plus the first
    128-row tile, element-wise against the fp64 oracle."""
    M, H, I = 8192, 4096, 11008
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=1)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, act)
    del X, G, U, W2
    Mr = M // W
    outs = [empty(Mr, H) for _ in range(W)]
    if W == 1:
        c = tl.Comm.single(0, max_M=M, max_H=H)
        c.mlp_forward(cuda(Xs[0]), cuda(W1s[0]), cuda(W2s[0]), outs[0], act=act)
        torch.cuda.synchronize()
    else:
        c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
        c.mlp_forward_lb([cuda(x) for x in Xs], [cuda(w) for w in W1s], [cuda(w) for w in W2s], outs, act=act)
    assert c.check()[0] == 0
    rows = sorted({r * Mr + o for r in range(W) for o in (0, 7, Mr // 2, Mr - 1)} | set(range(128)))
    ref = O.mlp_forward_rows([TI.to_f64(t) for t in Xs], [TI.to_f64(t) for t in W1s], [TI.to_f64(t) for t in W2s],
                             act, rows)
    full = torch.cat(outs).float().cpu().double().numpy()
    assert_parity(full[rows], np.stack([ref[i] for i in rows]))
    del c
