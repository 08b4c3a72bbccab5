"""GPU parity of the MoE first half (AllGather + Gather + GroupGEMM with the dynamic
tile-centric mapping) against the fp64 oracle.  The grouped order itself (row_ids)
is an index result and is compared bit-exactly; Y within 5e-3 relative Frobenius (bit-exact for the
integer placement fixture)."""
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


def _run(tl, W, M, H, E, topk, N_out, act, skew=0.0, pair=2, placement=False, seed=0, nsub=0, options=None):
    N1 = N_out * (1 if act == TI.ACT_NONE else 2)
    if placement:
        Xs, Ws = TI.moe_placement_inputs(M, H, E, N1, W)
    else:
        X = TI._randn((M, H), seed, 0)
        Xs = TI.shard_rows(X, W)
        Ws = TI.moe_weights(E, N1, H, W, seed=seed + 1)
    ids = TI.moe_routing(M, E, topk, seed=seed + 2, skew=skew)
    comm = tl.Comm.loopback(W, 0, max_M=M, max_H=H) if W > 1 else tl.Comm.single(0, max_M=M, max_H=H)
    comm.set_option("cta_pair", pair)
    comm.set_option("n_sub", nsub)
    for k, v in (options or {}).items():
        comm.set_option(k, v)
    R = tl.moe_capacity(comm, M, topk, E)
    Ys = [torch.empty(R, N_out, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    rows = [torch.empty(R, device="cuda", dtype=torch.int32) for _ in range(W)]
    offs = [torch.empty(E + 1, device="cuda", dtype=torch.int32) for _ in range(W)]
    idd = [ids.cuda() for _ in range(W)]
    if W > 1:
        tl.moe_ag_gemm_lb(comm, [x.cuda() for x in Xs], idd, [w.cuda() for w in Ws], Ys, rows, offs, act=act)
        st, diag = comm.check()
        assert st == 0, diag
    else:
        tl.moe_ag_gemm(comm, Xs[0].cuda(), idd[0], Ws[0].cuda(), Ys[0], rows[0], offs[0], act=act)
        torch.cuda.synchronize()
    ref_rows, ref_Y = O.moe_ag_group_gemm([TI.to_f64(x) for x in Xs], ids.numpy(), [TI.to_f64(w) for w in Ws], act)
    return ref_rows, ref_Y, Ys, rows, offs, topk


def _check(ref_rows, ref_Y, Ys, rows, offs, topk, exact=False):
    want = [t * topk + k for (_, t, k) in ref_rows]
    for r in range(len(Ys)):
        rid = rows[r].cpu().numpy()
        off = offs[r].cpu().numpy()
        valid = rid[:off[-1]] >= 0
        assert list(rid[:off[-1]][valid]) == want                    # grouped order, bit-exact
        for e in range(len(off) - 1):                                # groups padded to the tile height
            grp = rid[off[e]:off[e + 1]]
            assert all(rid_ == -1 for rid_ in grp[np.argmax(grp < 0):]) if (grp < 0).any() else True
        got = Ys[r].float().cpu().double().numpy()[:off[-1]][valid]
        if exact:
            assert np.array_equal(got, ref_Y[r])
        else:
            assert_parity(got, ref_Y[r])


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
@pytest.mark.parametrize("nsub", [1, 2])
def test_moe_parity(tl, W, act, nsub):
    res = _run(tl, W, M=256 * W if W > 1 else 512, H=192, E=8, topk=2, N_out=320, act=act, nsub=nsub)
    _check(*res)


@pytest.mark.parametrize("pair,nsub", [(1, 1), (2, 1), (2, 2)])
def test_moe_placement_bit_exact(tl, pair, nsub):
    res = _run(tl, 4, M=512, H=64, E=6, topk=3, N_out=520, act=TI.ACT_NONE, placement=True, pair=pair, nsub=nsub)
    _check(*res, exact=True)


def test_moe_skewed_routing_empty_experts(tl):
    # weights ~ (e+1)^-3 over 32 experts: the tail experts get no tokens at all
    res = _run(tl, 2, M=512, H=128, E=32, topk=2, N_out=128, act=TI.ACT_SILU_MUL, skew=3.0)
    _check(*res)


def test_moe_single_expert_is_ag_gemm(tl):
    res = _run(tl, 2, M=512, H=128, E=1, topk=1, N_out=128, act=TI.ACT_NONE)
    _check(*res)


def test_moe_paper_shape_moe4_w8(tl):
    """MoE-4 of the paper's Table (S=8192, H=4096, I=2048, E=8, topk=2), TP over 8 ranks
    (N_out = I/8 = 256 per expert shard), loopback on one GPU."""
    res = _run(tl, 8, M=8192, H=4096, E=8, topk=2, N_out=256, act=TI.ACT_SILU_MUL)
    _check(*res)


# ----------------------------------------------------------------------------- MoE second half + full layer
def _moe_layer(tl, W, M, H, I, E, topk, act=TI.ACT_SILU_MUL, skew=0.0, calls=1, pair=2, nsub=0, seed=0,
               options=None):
    il = I // W
    X = TI._randn((M, H), seed, 0)
    Xs = TI.shard_rows(X, W)
    W1s = TI.moe_weights(E, 2 * il, H, W, seed=seed + 1)
    W2s = TI.moe_down_weights(E, H, il, W, seed=seed + 3)
    ids = TI.moe_routing(M, E, topk, seed=seed + 2, skew=skew)
    wts = TI.moe_topk_weights(M, topk, seed=seed + 4)
    comm = (tl.Comm.loopback(W, 0, max_M=M, max_H=H, max_topk=topk) if W > 1
            else tl.Comm.single(0, max_M=M, max_H=H, max_topk=topk))
    comm.set_option("cta_pair", pair)
    comm.set_option("n_sub", nsub)
    for k, v in (options or {}).items():
        comm.set_option(k, v)
    R = tl.moe_capacity(comm, M, topk, E)
    Zg = [torch.empty(R, il, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    rows = [torch.empty(R, device="cuda", dtype=torch.int32) for _ in range(W)]
    offs = [torch.empty(E + 1, device="cuda", dtype=torch.int32) for _ in range(W)]
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    xd, idd, w1d, w2d, wtd = ([x.cuda() for x in Xs], [ids.cuda() for _ in range(W)], [w.cuda() for w in W1s],
                              [w.cuda() for w in W2s], [wts.cuda() for _ in range(W)])
    results = []
    for _ in range(calls):
        if W > 1:
            tl.moe_ag_gemm_lb(comm, xd, idd, w1d, Zg, rows, offs, act=act)
            tl.moe_gemm_rs_lb(comm, Zg, rows, offs, wtd, w2d, outs)
            st, diag = comm.check()
            assert st == 0, diag
        else:
            tl.moe_ag_gemm(comm, xd[0], idd[0], w1d[0], Zg[0], rows[0], offs[0], act=act)
            tl.moe_gemm_rs(comm, Zg[0], rows[0], offs[0], wtd[0], w2d[0], outs[0])
            st, diag = comm.check()
            assert st == 0, diag
        results.append([o.clone() for o in outs])
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = O.moe_forward(f(Xs), ids.numpy(), wts.double().numpy(), f(W1s), f(W2s), act)
    return results, ref


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("topk", [2, 5])
def test_moe_layer_parity(tl, W, topk):
    """Full TP MoE FFN: AG + Gather + GroupGEMM + SiLU*up, then GroupGEMM + Scatter + TopK + RS."""
    results, ref = _moe_layer(tl, W, M=256 * W if W > 1 else 512, H=256, I=256 * W, E=8, topk=topk)
    got = np.concatenate([o.float().cpu().double().numpy() for o in results[0]], 0)
    assert_parity(got, np.concatenate(ref, 0))


@pytest.mark.parametrize("pair,nsub", [(1, 1), (2, 1), (2, 2)])
def test_moe_layer_options_and_epochs(tl, pair, nsub):
    """Tile shapes / CTA pairing never change the result beyond rounding; repeated calls (banks and
    epochs cycling, completion counters accumulating) are bitwise identical."""
    results, ref = _moe_layer(tl, 4, M=1024, H=512, I=1024, E=16, topk=3, skew=1.0, calls=4, pair=pair, nsub=nsub)
    got = np.concatenate([o.float().cpu().double().numpy() for o in results[0]], 0)
    assert_parity(got, np.concatenate(ref, 0))
    for later in results[1:]:
        for a, b in zip(later, results[0]):
            assert torch.equal(a, b)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_moe_layer_copy_engine_binding(tl, W):
    """ag_binding = 1 (the paper's binding: AllGather on the copy engines) for the MoE first half:
    bitwise equal to the SM-copy binding over epoch-cycling calls."""
    kw = dict(M=256 * W, H=256, I=256 * W, E=8, topk=2, skew=0.5, calls=2)
    sm_res, ref = _moe_layer(tl, W, **kw)
    dma_res, _ = _moe_layer(tl, W, **kw, options={"ag_binding": 1})
    for call in dma_res:
        for a, b in zip(call, sm_res[0]):
            assert torch.equal(a, b)
    got = np.concatenate([o.float().cpu().double().numpy() for o in dma_res[-1]], 0)
    assert_parity(got, np.concatenate(ref, 0))


def test_moe_layer_single_expert_matches_dense_mlp_kernels(tl):
    """E = 1, top-1, weight 1: the MoE path must agree with the dense MLP path on the GPU."""
    W, M, H, I = 2, 512, 256, 512
    results, ref = _moe_layer(tl, W, M, H, I, E=1, topk=1)
    got = np.concatenate([o.float().cpu().double().numpy() for o in results[0]], 0)
    assert_parity(got, np.concatenate(ref, 0))


def test_moe_layer_bench_config_w1_sampled(tl):
    """bench.py --workload moe at N = 1, exactly: MoE-4 (S = 8192, H = 4096, I = 2048, E = 8, top-2), both
    halves, the bench's seeded inputs and comm; 32 sampled tokens against the oracle (tokens are
    independent, so the token-sampled oracle is exact for them)."""
    import bench_workloads as BW
    S, H, I, E, k = (BW.MOE[n] for n in ("S", "H", "I", "E", "topk"))
    X, ids, wts, W1s, W2s = BW._moe_inputs(1)
    comm = tl.Comm.single(0, S, H, max_topk=k)
    R = tl.moe_capacity(comm, S, k, E)
    Y = torch.empty(R, I, device="cuda", dtype=torch.bfloat16)
    rows = torch.empty(R, device="cuda", dtype=torch.int32)
    offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
    out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
    tl.moe_ag_gemm(comm, X.cuda(), ids.cuda(), W1s[0].cuda(), Y, rows, offs, act=tl.ACT_SILU_MUL)
    tl.moe_gemm_rs(comm, Y, rows, offs, wts.cuda(), W2s[0].cuda(), out)
    st, diag = comm.check()
    assert st == 0, diag
    toks = np.sort(np.random.default_rng(5).choice(S, 32, replace=False))
    f = lambda L: [TI.to_f64(t) for t in L]
    ref = BW._moe_oracle_tokens(X, ids, wts, f(W1s), f(W2s), toks)
    got = out[torch.as_tensor(toks, device="cuda")].float().cpu().double().numpy()
    assert_parity(got, ref)


@pytest.mark.parametrize("M,H,N_out,E,topk", [(8192, 4096, 2048, 8, 2), (2048, 512, 512, 4, 2), (1024, 256, 384, 3, 1)])
def test_moe_split_tail_bitwise(tl, M, H, N_out, E, topk):
    """Option moe_split (default on): the gather GroupGEMM's last wave of 512-wide tiles runs as 256-wide
    half items when it is at most half full (decided on the device from the routing tables; MoE-4 at W = 1:
    552 tiles on 74 pairs).  Tiles are computed the same way, so the output is bitwise identical to whole
    tiles; also with CTA counts that put the split on other remainders."""
    X = TI._randn((M, H), 3, 0).cuda()
    W1 = TI.moe_weights(E, 2 * N_out, H, 1, seed=4)[0].cuda()
    ids = TI.moe_routing(M, E, topk, seed=5).cuda()
    outs = []
    for split, ctas in ((0, 0), (1, 0), (1, 100), (1, 60)):
        c = tl.Comm.single(0, max_M=M, max_H=H)
        c.set_option("moe_split", split)
        c.set_option("num_ctas", ctas)
        R = tl.moe_capacity(c, M, topk, E)
        Y = torch.empty(R, N_out, device="cuda", dtype=torch.bfloat16)
        rows = torch.empty(R, device="cuda", dtype=torch.int32)
        offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
        tl.moe_ag_gemm(c, X, ids, W1, Y, rows, offs, act=tl.ACT_SILU_MUL)
        torch.cuda.synchronize()
        assert c.check()[0] == 0
        n = int(offs[-1].item())
        outs.append((Y[:n].clone(), rows[:n].clone()))
        c.close()
    for Y, rows in outs[1:]:
        assert torch.equal(rows, outs[0][1]) and torch.equal(Y, outs[0][0])
