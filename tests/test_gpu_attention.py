"""GPU parity of the sequence-parallel attention (AllGather of the K/V sequence shards
fused with flash attention) against the fp64 oracle `sp_attention`.

Tolerance: relative Frobenius error < 5e-3.  Inputs are bf16; the kernel keeps the softmax statistics
and O in fp32 and rounds twice: P to bf16 before the P.V MMA (relative error <= 2^-9 per weight,
random sign, so the row error of O averages down) and O to bf16 at the end (2^-9).  Both are rms
~1e-3 of |O|; 5e-3 leaves the margin the MLP tests use."""
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


def _comm(tl, W, S, heads, D=128):
    need = 2 * S * heads * D
    max_H = 4096
    max_M = max(128, (need + max_H - 1) // max_H)
    return tl.Comm.loopback(W, 0, max_M=max_M, max_H=max_H) if W > 1 else tl.Comm.single(0, max_M=max_M, max_H=max_H)


def _run(tl, W, S, heads, scale=None, seed=0, comm=None, calls=1, inputs=None):
    D = 128
    scale = D ** -0.5 if scale is None else scale
    Qs, Ks, Vs = inputs if inputs is not None else TI.attention_inputs(S, heads, D, W, seed=seed)
    comm = comm or _comm(tl, W, S, heads)
    qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
    outs = [torch.empty_like(q) for q in qd]
    results = []
    for _ in range(calls):
        if W > 1:
            tl.sp_attention_lb(comm, qd, kd, vd, outs, scale=scale)
        else:
            tl.sp_attention(comm, qd[0], kd[0], vd[0], outs[0], scale=scale)
        st, diag = comm.check()
        assert st == 0, diag
        results.append([o.clone() for o in outs])
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = O.sp_attention(f(Qs), f(Ks), f(Vs), scale)
    return results, ref


def _err(outs, ref):
    """Element-wise parity (tests/parity.py: global, per 128-row tile, per (token, head) row, per element);
    returns the global relative Frobenius error."""
    got = np.concatenate([o.float().cpu().double().numpy() for o in outs], 0)
    return assert_parity(got, np.concatenate(ref, 0))["global"]


@pytest.mark.parametrize("S,heads", [(128, 1), (256, 3), (1024, 4)])
def test_attention_w1(tl, S, heads):
    results, ref = _run(tl, 1, S, heads)
    assert _err(results[0], ref) < TOL


@pytest.mark.parametrize("W,S", [(1, 1), (1, 100), (1, 200), (1, 333), (1, 1000), (2, 200), (2, 384), (3, 450),
                                 (4, 400), (8, 576), (8, 8 * 200)])
def test_attention_ragged(tl, W, S):
    """Ragged shapes (the masking kernel variant): S % 128 != 0 (the last KV block is loaded with TMA
    zero fill and its missing keys are masked to -inf), S/world % 128 != 0 (KV blocks straddle shards;
    the last query tile is partial, with rows split inside a warp, and only valid rows are stored),
    S/world < 128, and a single token."""
    results, ref = _run(tl, W, S, 3)
    assert _err(results[0], ref) < TOL


@pytest.mark.parametrize("poly", [0, 2, 8])
def test_attention_ragged_exp2_split(tl, poly):
    """The ragged instantiation honours option attn_poly (every n-th exponential pair on the FMA pipe,
    0 = all on MUFU): each split meets the bound, and the splits differ only by rounding."""
    W, S, heads = 2, 2 * 200, 2
    comm = _comm(tl, W, S, heads)
    comm.set_option("attn_poly", poly)
    results, ref = _run(tl, W, S, heads, comm=comm, seed=5)
    assert _err(results[0], ref) < TOL


def test_attention_ragged_no_store_beyond_rows(tl):
    """A partial last query tile writes only its S_r rows: the bytes after O are left untouched."""
    S, heads = 200, 2
    Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, 1, seed=3)
    comm = _comm(tl, 1, S, heads)
    big = torch.full((S + 128, heads, 128), 7.0, device="cuda", dtype=torch.bfloat16)
    tl.sp_attention(comm, Qs[0].cuda(), Ks[0].cuda(), Vs[0].cuda(), big[:S])
    assert comm.check()[0] == 0
    assert torch.all(big[S:] == 7.0)
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = O.sp_attention(f(Qs), f(Ks), f(Vs), 128 ** -0.5)
    assert _err([big[:S]], ref) < TOL


@pytest.mark.parametrize("binding", [0, 1])
def test_attention_ragged_tile_height_invariance(tl, binding):
    """Ragged shards (S/world = 200): the result does not depend on the producer tile height or on the
    resource binding of the K/V AllGather."""
    W, S, heads = 2, 400, 2
    inputs = TI.attention_inputs(S, heads, 128, W, seed=9)
    outs = []
    for rows in (16, 64, 200):
        comm = _comm(tl, W, S, heads)
        comm.set_option("comm_tile_rows", rows)
        comm.set_option("dma_tile_rows", rows)
        comm.set_option("ag_binding", binding)
        results, ref = _run(tl, W, S, heads, comm=comm, inputs=inputs)
        outs.append(torch.cat(results[0], 0))
    assert _err(results[0], ref) < TOL
    assert all(torch.equal(o, outs[0]) for o in outs)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_attention_loopback(tl, W):
    results, ref = _run(tl, W, 256 * W, 2)
    assert _err(results[0], ref) < TOL


@pytest.mark.parametrize("scale", [0.02, 0.5])
def test_attention_scales(tl, scale):
    """A flat (0.02) and a peaked (0.5: logits ~ N(0, 32), the row max moves often, exercising the
    lazy O rescale) softmax."""
    results, ref = _run(tl, 2, 1024, 2, scale=scale)
    assert _err(results[0], ref) < TOL


def test_attention_growing_max(tl):
    """Keys whose magnitude grows along the sequence: every KV block raises every row max, so the
    online rescale runs on every block (and in every rank's visiting order)."""
    W, S, heads, D = 2, 1024, 2, 128
    g = torch.Generator().manual_seed(7)
    Q = torch.randn(S, heads, D, generator=g)
    K = torch.randn(S, heads, D, generator=g) * torch.linspace(0.2, 3.0, S)[:, None, None]
    V = torch.randn(S, heads, D, generator=g)
    sh = lambda T: [t.contiguous() for t in T.to(torch.bfloat16).chunk(W, 0)]
    results, ref = _run(tl, W, S, heads, inputs=(sh(Q), sh(K), sh(V)))
    assert _err(results[0], ref) < TOL


def test_attention_one_hot_is_exact_gather(tl):
    """Closed form: with scale large and Q_i = K_{pi(i)} direction scaled up, the softmax is one-hot
    (exp underflows to 0 off the max), so O_i = V_{pi(i)} exactly in bf16 -- an index check that a
    transposed operand, a wrong KV block order or a wrong rank offset cannot pass."""
    W, S, heads, D = 4, 512, 2, 128
    g = torch.Generator().manual_seed(3)
    # keys: random signs (orthogonal-ish rows), queries: the key of a permuted token
    K = (torch.randint(0, 2, (S, heads, D), generator=g) * 2 - 1).float()
    perm = torch.randperm(S, generator=g)
    Q = K[perm].clone()
    V = torch.randn(S, heads, D, generator=g).to(torch.bfloat16).float()
    sh = lambda T: [t.contiguous() for t in T.to(torch.bfloat16).chunk(W, 0)]
    results, ref = _run(tl, W, S, heads, scale=1.0, inputs=(sh(Q), sh(K), sh(V)))
    got = torch.cat([o.float().cpu() for o in results[0]], 0)
    assert torch.equal(got, V[perm])
    assert np.array_equal(got.double().numpy(), np.concatenate(ref, 0).astype(np.float32).astype(np.float64)) or \
        O.rel_frobenius(got.double().numpy(), np.concatenate(ref, 0)) < 1e-6


def test_attention_epochs_and_options(tl):
    """Repeated calls (AG banks / epochs cycling) are bitwise identical; producer tile height and
    channel grouping (the static mapping) and the CTA count never change the result."""
    W, S, heads = 4, 1024, 2
    comm = _comm(tl, W, S, heads)
    results, ref = _run(tl, W, S, heads, comm=comm, calls=3)
    for later in results[1:]:
        for a, b in zip(later, results[0]):
            assert torch.equal(a, b)
    for tile_rows, ch, ctas in [(16, 0, 0), (100, 2, 0), (256, 1, 7)]:
        comm.set_option("comm_tile_rows", tile_rows)
        comm.set_option("channels_per_rank", ch)
        comm.set_option("num_ctas", ctas)
        r2, _ = _run(tl, W, S, heads, comm=comm)
        for a, b in zip(r2[0], results[0]):
            assert torch.equal(a, b)


def test_attention_lost_peer_times_out(tl):
    """A dropped producer notify (debug option) surfaces as TL_ERR_TIMEOUT via tl_comm_check with the
    waiting rank and tile, instead of hanging."""
    W, S, heads = 2, 512, 1
    comm = _comm(tl, W, S, heads)
    comm.set_option("timeout_ms", 200)
    comm.set_option("debug_drop_rank", 0)
    comm.set_option("debug_drop_notify", 0)
    Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, W, seed=1)
    qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
    outs = [torch.empty_like(q) for q in qd]
    tl.sp_attention_lb(comm, qd, kd, vd, outs)
    st, diag = comm.check()
    assert st != 0
    assert diag[0] != 0 and diag[1] == 1 and diag[3] == 0 and diag[4] == 0   # rank 1 waited on rank 0's tile 0
    comm.set_option("debug_drop_rank", -1)
    results, ref = _run(tl, W, S, heads, comm=comm)
    assert _err(results[0], ref) < TOL


def test_attention_validation(tl):
    comm = tl.Comm.single(0, max_M=1024, max_H=1024)
    q = torch.zeros(128, 2, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(tl.TLError):
        tl.sp_attention(comm, q, q, q, torch.empty_like(q))           # head_dim 64
    q = torch.zeros(128, 2, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(tl.TLError):
        tl.sp_attention(comm, q, q, q, torch.empty_like(q), scale=-1.0)
    lb = tl.Comm.loopback(2, 0, max_M=128, max_H=128)                 # capacity: 2*S*heads*D > 128*128
    qs = [torch.zeros(128, 2, 128, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    with pytest.raises(tl.TLError):
        tl.sp_attention_lb(lb, qs, qs, qs, [torch.empty_like(x) for x in qs])
    e = torch.zeros(0, 2, 128, device="cuda", dtype=torch.bfloat16)
    tl.sp_attention(comm, e, e, e, torch.empty_like(e))               # empty: no-op


def test_attention_paper_shape_attn1_16k_sampled(tl):
    """Attn-1 (32 heads, d 128, S = 16k) over 8 ranks: the full shape in the launch
    configuration the bench times, checked on sampled query rows of every rank against the oracle
    evaluated row by row."""
    W, S, heads, D = 8, 16384, 32, 128
    Qs, Ks, Vs = TI.attention_inputs(S, heads, D, W, seed=5)
    comm = _comm(tl, W, S, heads)
    qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
    outs = [torch.empty_like(q) for q in qd]
    tl.sp_attention_lb(comm, qd, kd, vd, outs)
    st, diag = comm.check()
    assert st == 0, diag
    rng = np.random.default_rng(0)
    K64, V64 = (np.concatenate([TI.to_f64(t) for t in L], 0) for L in (Ks, Vs))
    for r in range(W):
        rows = rng.choice(S // W, 6, replace=False)
        q = TI.to_f64(Qs[r])[rows]
        ref = O.sp_attention([q], [K64], [V64], D ** -0.5)[0]
        got = outs[r][torch.as_tensor(rows, device="cuda")].float().cpu().double().numpy()
        assert_parity(got, ref)


def test_attention_bench_config_w1_sampled(tl):
    """bench.py --workload attention at N = 1, exactly: Attn-1 heads (32 x 128), S = 16384, W = 1, the
    bench's seeded inputs and comm; sampled query rows of every 2k-row block against the oracle
    evaluated row by row over the full K/V."""
    import bench_workloads as BW
    S, heads, D = BW.ATTN["S"], BW.ATTN["heads"], BW.ATTN["D"]
    Qs, Ks, Vs = TI.attention_inputs(S, heads, D, 1, seed=0)
    comm = tl.Comm.single(0, S, 2 * heads * D)
    q, k, v = Qs[0].cuda(), Ks[0].cuda(), Vs[0].cuda()
    o = torch.empty_like(q)
    tl.sp_attention(comm, q, k, v, o)
    st, diag = comm.check()
    assert st == 0, diag
    rows = np.arange(0, S, 2048) + np.random.default_rng(3).integers(0, 2048, S // 2048)
    K64, V64 = TI.to_f64(Ks[0]), TI.to_f64(Vs[0])
    ref = O.sp_attention([TI.to_f64(Qs[0])[rows]], [K64], [V64], D ** -0.5)[0]
    got = o[torch.as_tensor(rows, device="cuda")].float().cpu().double().numpy()
    assert_parity(got, ref)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_attention_copy_engine_binding(tl, W):
    """ag_binding = 1: the K/V AllGather runs on the copy engines (cudaMemcpyAsync per producer tile
    and destination + stream write-value flags; the paper's binding for this workload) and the
    kernel's waits are unchanged: bitwise equal to the SM binding over epoch-cycling calls, and
    correct against the oracle."""
    S, heads = 512 * W, 2
    comm = _comm(tl, W, S, heads)
    sm, ref = _run(tl, W, S, heads, comm=comm)
    comm.set_option("ag_binding", 1)
    dma, _ = _run(tl, W, S, heads, comm=comm, calls=3)
    for call in dma:
        for a, b in zip(call, sm[0]):
            assert torch.equal(a, b)
    assert _err(dma[-1], ref) < TOL


def test_attention_copy_engine_dropped_notify_times_out(tl):
    W, S, heads = 2, 512, 1
    comm = _comm(tl, W, S, heads)
    comm.set_option("ag_binding", 1)
    comm.set_option("timeout_ms", 200)
    comm.set_option("debug_drop_rank", 0)
    comm.set_option("debug_drop_notify", 0)
    Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, W, seed=2)
    qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
    outs = [torch.empty_like(q) for q in qd]
    tl.sp_attention_lb(comm, qd, kd, vd, outs)
    st, diag = comm.check()
    assert st != 0 and diag[1] == 1


def test_attention_paper_shape_attn2_32k_sampled(tl):
    """Attn-2 (64 heads, d 128) at S = 32k over 4 ranks: sampled query rows of every rank against
    the oracle evaluated row by row over the whole gathered K/V."""
    W, S, heads, D = 4, 32768, 64, 128
    Qs, Ks, Vs = TI.attention_inputs(S, heads, D, W, seed=6)
    comm = _comm(tl, W, S, heads)
    qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
    outs = [torch.empty_like(q) for q in qd]
    tl.sp_attention_lb(comm, qd, kd, vd, outs)
    st, diag = comm.check()
    assert st == 0, diag
    rng = np.random.default_rng(1)
    K64, V64 = (np.concatenate([TI.to_f64(t) for t in L], 0) for L in (Ks, Vs))
    for r in range(W):
        rows = rng.choice(S // W, 3, replace=False)
        ref = O.sp_attention([TI.to_f64(Qs[r])[rows]], [K64], [V64], D ** -0.5)[0]
        got = outs[r][torch.as_tensor(rows, device="cuda")].float().cpu().double().numpy()
        assert_parity(got, ref)


def test_attention_longest_sequence_sampled(tl):
    """The paper's longest sequence (S = 128k) on one GPU with 4 heads: 1024 KV blocks per
    query tile, so the online softmax (lazy max, fp32 O and row sums) runs its longest accumulation;
    sampled rows against the oracle."""
    S, heads, D = 131072, 4, 128
    Qs, Ks, Vs = TI.attention_inputs(S, heads, D, 1, seed=7)
    comm = tl.Comm.single(0, max_M=128, max_H=128)
    q, k, v = Qs[0].cuda(), Ks[0].cuda(), Vs[0].cuda()
    o = torch.empty_like(q)
    tl.sp_attention(comm, q, k, v, o)
    st, diag = comm.check()
    assert st == 0, diag
    rows = np.sort(np.random.default_rng(2).choice(S, 12, replace=False))
    ref = O.sp_attention([TI.to_f64(Qs[0])[rows]], [TI.to_f64(Ks[0])], [TI.to_f64(Vs[0])], D ** -0.5)[0]
    got = o[torch.as_tensor(rows, device="cuda")].float().cpu().double().numpy()
    assert_parity(got, ref)
