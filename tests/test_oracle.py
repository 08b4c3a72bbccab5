"""Pins for the CPU oracle (SURVEY.md §8(c) "Pins"): nothing here re-types the
oracle's own formulas; every check compares against a hand-computed fixture, a
closed form, a mathematical invariant or an independent pure-Python implementation."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import pyloop
from oracle import tl_oracle as O
import tl_inputs as TI


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# --- pin 1: hand example ------------------------------------------------
def test_hand_example(golden_dir):
    g = _load(golden_dir, "hand_example_w2.json")
    Xs = [np.array(x, float) for x in g["X_shards"]]
    W1 = [np.array(x, float) for x in g["W1"]]
    W2 = [np.array(x, float) for x in g["W2"]]
    X, Ys = O.ag_gemm(Xs, W1)
    np.testing.assert_array_equal(X, np.array(g["X_shards"][0] + g["X_shards"][1], float))
    np.testing.assert_array_equal(Ys[1], np.array(g["Y1"], float))
    outs = O.mlp_forward(Xs, W1, W2, g["act"])
    for r in range(g["W"]):
        np.testing.assert_array_equal(outs[r], np.array(g["out"][r], float))
    # the standalone GEMM-RS on the hand partials' operands
    outs2 = O.gemm_rs(Ys, W2)
    for r in range(g["W"]):
        np.testing.assert_array_equal(outs2[r], np.array(g["out"][r], float))


def test_hand_example_pyloop(golden_dir):
    g = _load(golden_dir, "hand_example_w2.json")
    outs = pyloop.mlp_forward(g["X_shards"], g["W1"], g["W2"], g["act"])
    assert outs == [[[float(v) for v in row] for row in blk] for blk in g["out"]]


# --- pin 2: sharding invariant (concat_r out_r == unsharded MLP) ---------------
@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL, TI.ACT_GELU_TANH_MUL])
def test_sharding_invariant(W, act):
    M, H, I = 64, 32, 48
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=3)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, act)
    outs = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s],
                         [TI.to_f64(w) for w in W2s], act)
    got = np.concatenate(outs, 0)
    # unsharded reference, written without any sharding: full gate/up, full W2
    Xf, Gf, Uf, W2f = (TI.to_f64(t) for t in (X, G, U, W2))
    g = Xf @ Gf.T
    if act == TI.ACT_NONE:
        Z = g
    elif act == TI.ACT_SILU_MUL:
        Z = g * (1.0 / (1.0 + np.exp(-g))) * (Xf @ Uf.T)
    else:
        Z = 0.5 * g * (1 + np.tanh(np.sqrt(2 / np.pi) * (g + 0.044715 * g ** 3))) * (Xf @ Uf.T)
    ref = Z @ W2f.T
    assert O.rel_frobenius(got, ref) < 1e-12


# --- pin 3: W = 1 degeneration -----------------------------------------
def test_world1_identity():
    A = np.arange(12, dtype=float).reshape(3, 4)
    assert np.array_equal(O.all_gather_rows([A]), A)
    assert np.array_equal(O.reduce_scatter_rows([A])[0], A)


# --- pin 4: closed forms --------------------------------------------------------
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_all_ones_closed_forms(W):
    M, H, I = 16, 8, 24
    il = I // W
    Xs = [np.ones((M // W, H)) for _ in range(W)]
    W1 = [np.ones((il, H)) for _ in range(W)]
    W2 = [np.ones((H, il)) for _ in range(W)]
    outs = O.mlp_forward(Xs, W1, W2, O.ACT_NONE)
    for o in outs:
        assert np.all(o == H * I)          # out = H * I everywhere
    Kl = 5
    As = [np.ones((M, Kl)) for _ in range(W)]
    Bs = [np.ones((7, Kl)) for _ in range(W)]
    for o in O.gemm_rs(As, Bs):
        assert np.all(o == W * Kl)         # every output = K * R


def test_reduce_scatter_order_and_owner():
    # rank s contributes the constant s+1 in every row; out_r rows come from global rows of r
    W, m = 4, 3
    parts = [np.full((W * m, 2), float(10 ** s)) for s in range(W)]
    parts[2][5, 1] = 7.0  # global row 5 belongs to rank 1 (rows 3..5)
    outs = O.reduce_scatter_rows(parts)
    assert outs[0].shape == (m, 2)
    assert outs[1][2, 1] == 1 + 10 + 7 + 1000
    assert np.all(outs[3] == 1111)


# --- pin 5: pure-Python triple loop == numpy oracle ----------------------------
@pytest.mark.parametrize("act", [TI.ACT_NONE, TI.ACT_SILU_MUL])
def test_pyloop_matches_numpy(act):
    W, M, H, I = 2, 16, 16, 32
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=5)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, act)
    a = O.mlp_forward([TI.to_f64(x) for x in Xs], [TI.to_f64(w) for w in W1s],
                      [TI.to_f64(w) for w in W2s], act)
    b = pyloop.mlp_forward([x.float().tolist() for x in Xs], [w.float().tolist() for w in W1s],
                           [w.float().tolist() for w in W2s], act)
    for r in range(W):
        assert O.rel_frobenius(a[r], np.array(b[r])) < 1e-13


def test_row_sampled_oracle_is_exact():
    W, M, H, I = 4, 32, 16, 32
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=7)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    f = lambda L: [TI.to_f64(t) for t in L]
    full = np.concatenate(O.mlp_forward(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL), 0)
    rows = [0, 5, 17, 31]
    samp = O.mlp_forward_rows(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL, rows)
    for i in rows:
        np.testing.assert_allclose(samp[i], full[i], rtol=1e-13, atol=1e-14)


# --- activations: closed forms and symmetries -------------------------------------
def test_activation_values(golden_dir):
    g = _load(golden_dir, "activation_values.json")
    for x, v in g["silu"]:
        assert abs(float(O.silu(x)) - v) < 1e-15
    for x, v in g["gelu_tanh"]:
        assert abs(float(O.gelu_tanh(x)) - v) < 1e-15
    xs = np.linspace(-6, 6, 101)
    # x*s(x) - (-x)*s(-x) = x  because s(x) + s(-x) = 1, for both sigmoid-like gates
    np.testing.assert_allclose(O.silu(xs) - O.silu(-xs), xs, atol=1e-14)
    np.testing.assert_allclose(O.gelu_tanh(xs) - O.gelu_tanh(-xs), xs, atol=1e-14)
    assert abs(float(O.silu(40.0)) - 40.0) < 1e-12


def test_activation_wiring():
    # gate half goes through act, up half multiplies; gate=0 -> 0; up=1 -> act(gate)
    Y = np.array([[0.0, 2.0, 5.0, 1.0]])
    Z = O.activation(Y, O.ACT_SILU_MUL)
    assert Z[0, 0] == 0.0
    assert abs(Z[0, 1] - 2.0 / (1 + math.exp(-2.0))) < 1e-15
    assert np.array_equal(O.activation(Y, O.ACT_NONE), Y)


# --- pin 6: mapping fixtures and invariants ------------------
def test_static_mapping_fixtures(golden_dir):
    g = _load(golden_dir, "spec_static_mapping.json")
    for c in g["shape_range"]:
        assert list(O.static_shape_range(c["t"], c["M"], c["Tm"])) == c["expect"]
    for c in g["src_rank"]:
        assert O.static_src_rank(c["t"], c["M"], c["R"], c["Tm"]) == c["expect"]
    for c in g["channel"]:
        assert O.static_channel(c["t"], c["M"], c["R"], c["C"], c["Tm"]) == c["expect"]


@pytest.mark.parametrize("M,R,C,Tm", [(8192, 8, 4, 128), (8192, 8, 8, 128), (256, 2, 1, 128),
                                       (4096, 4, 2, 64), (1024, 8, 1, 128)])
def test_static_mapping_invariants(M, R, C, Tm):
    n = O.ceil_div(M, Tm)
    covered = []
    prev_r = prev_c = -1
    mpr = O.ceil_div(M, R)
    for t in range(n):
        lo, hi = O.static_shape_range(t, M, Tm)
        covered.extend(range(lo, hi))
        r = O.static_src_rank(t, M, R, Tm)
        c = O.static_channel(t, M, R, C, Tm)
        assert r >= prev_r and c >= prev_c            # monotone
        assert r * mpr <= lo and hi <= (r + 1) * mpr   # tile inside its rank's rows
        assert r == c // C                              # channel belongs to the same rank
        prev_r, prev_c = r, c
    assert covered == list(range(M))                    # partition


def test_mapping_undefined_is_rejected():
    with pytest.raises(ValueError):
        O.static_src_rank(0, 8192, 8, 2048)   # Tm > M_per_rank (reading R4)


def test_consumer_wait_channels():
    # a 256-row consumer tile at rows [1024, 1280) of M=8192, R=8, C=4 spans channels 4 only
    assert O.consumer_wait_channels(1024, 1280, 8192, 8, 4) == [4]
    # a tile straddling ranks waits on both ranks' channels
    assert O.consumer_wait_channels(896, 1152, 8192, 8, 4) == [3, 4]


# --- overlap ratio ------------------------------------------
def test_overlap_ratio(golden_dir):
    g = _load(golden_dir, "overlap_ratio.json")
    for c in g["cases"]:
        assert O.overlap_ratio(c["comp"], c["comm"], c["overlap"]) == pytest.approx(c["expect"], abs=1e-15)
    with pytest.raises(ValueError):
        O.overlap_ratio(1, 0, 1)


# --- placement fixtures: closed forms of the index-check inputs ------------------
def test_ag_placement_closed_form():
    W, M, K, N = 4, 512, 32, 8
    Xs, Bs = TI.ag_placement_inputs(M, K, N, W)
    X, Cs = O.ag_gemm([TI.to_f64(x) for x in Xs], [TI.to_f64(b) for b in Bs])
    i = np.arange(M)
    for r in range(W):
        for n in range(N):
            q = (n + r) % 4
            assert np.array_equal(Cs[r][:, n], ((i >> (4 * q)) & 15).astype(float))


def test_rs_placement_closed_form():
    W, M, N, K = 4, 256, 12, 24
    As, Bs = TI.rs_placement_inputs(M, N, K, W)
    outs = O.gemm_rs([TI.to_f64(a) for a in As], [TI.to_f64(b) for b in Bs])
    m = M // W
    for r in range(W):
        i = np.arange(r * m, (r + 1) * m)
        for h in range(N):
            q = h % 4
            exp = W * ((i >> (4 * q)) & 15) + (h % 3) * W * (W - 1) // 2
            assert np.array_equal(outs[r][:, h], exp.astype(float))


def test_rel_frobenius():
    a = np.array([3.0, 4.0])
    assert O.rel_frobenius(a, a) == 0.0
    assert O.rel_frobenius(np.array([3.0, 5.0]), a) == pytest.approx(0.2)


# --- MoE first half (NEXT-3): pins ------------------------------------------------
def test_moe_grouping_is_a_stable_permutation():
    ids = np.array([[1, 0], [0, 2], [1, 2], [2, 1]])
    rows = O.moe_group_rows(ids, 3)
    assert rows == [(0, 0, 1), (0, 1, 0), (1, 0, 0), (1, 2, 0), (1, 3, 1), (2, 1, 1), (2, 2, 1), (2, 3, 0)]
    ids = TI.moe_routing(64, 8, 3, seed=1).numpy()
    rows = O.moe_group_rows(ids, 8)
    assert sorted((t, k) for _, t, k in rows) == [(t, k) for t in range(64) for k in range(3)]   # S:374 conservation
    assert all(ids[t, k] == e for e, t, k in rows)
    assert rows == sorted(rows, key=lambda x: (x[0], x[1], x[2]))


def test_moe_single_expert_is_plain_ag_gemm():
    W, M, H, N1 = 2, 16, 8, 6
    Xs, _ = TI.ag_gemm_inputs(M, N1, H, W, seed=2)
    Ws = TI.moe_weights(1, N1, H, W, seed=3)
    ids = np.zeros((M, 1), dtype=np.int64)
    rows, Ys = O.moe_ag_group_gemm([TI.to_f64(x) for x in Xs], ids, [TI.to_f64(w) for w in Ws], O.ACT_NONE)
    _, Cs = O.ag_gemm([TI.to_f64(x) for x in Xs], [TI.to_f64(w[0]) for w in Ws])
    for r in range(W):
        np.testing.assert_array_equal(Ys[r], Cs[r])   # identity routing: row j is token j


def test_moe_pyloop_and_placement_closed_form():
    W, M, H, E, N1 = 2, 12, 16, 3, 4
    Xs, Ws = TI.moe_placement_inputs(M, H, E, N1, W)
    ids = TI.moe_routing(M, E, 2, seed=4).numpy()
    rows, Ys = O.moe_ag_group_gemm([TI.to_f64(x) for x in Xs], ids, [TI.to_f64(w) for w in Ws], O.ACT_NONE)
    for r in range(W):
        for j, (e, t, k) in enumerate(rows):
            for n in range(N1):
                assert Ys[r][j, n] == (t >> (4 * ((n + e + r) % 4))) & 15
    # brute force, pure Python, one routed row at a time
    X = [x for s in Xs for x in s.float().tolist()]
    W1 = Ws[1].float().tolist()
    for j, (e, t, k) in enumerate(rows):
        for n in range(N1):
            assert sum(a * b for a, b in zip(X[t], W1[e][n])) == Ys[1][j, n]


def test_moe_single_expert_is_dense_mlp():
    """E = 1, top-1, weight 1: the TP MoE FFN is exactly the dense TP MLP."""
    W, M, H, I = 2, 16, 8, 12
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=6)
    Xs, W1s, W2s = TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL)
    f = lambda L: [TI.to_f64(t) for t in L]
    ids = np.zeros((M, 1), dtype=np.int64)
    w = np.ones((M, 1))
    outs = O.moe_forward(f(Xs), ids, w, [x[None] for x in f(W1s)], [x[None] for x in f(W2s)], TI.ACT_SILU_MUL)
    ref = O.mlp_forward(f(Xs), f(W1s), f(W2s), TI.ACT_SILU_MUL)
    for r in range(W):
        np.testing.assert_allclose(outs[r], ref[r], rtol=1e-12, atol=1e-12)


def test_moe_second_half_closed_form_and_brute_force():
    # all-ones Zg and W2, weights summing to 1 per token: every output = W * I_l (S:347 analogue)
    W, M, H, E, topk, Il = 2, 8, 4, 3, 2, 5
    ids = TI.moe_routing(M, E, topk, seed=1).numpy()
    rows = O.moe_group_rows(ids, E)
    w = TI.moe_topk_weights(M, topk, seed=2).double().numpy()
    w = w / w.sum(1, keepdims=True)          # exactly 1 per token in fp64
    Zg = [np.ones((len(rows), Il)) for _ in range(W)]
    W2 = [np.ones((E, H, Il)) for _ in range(W)]
    outs = O.moe_group_gemm_rs(rows, Zg, W2, w, M)
    np.testing.assert_allclose(np.concatenate(outs), W * Il, rtol=1e-14)
    # brute force on random data, per token, pure Python sums
    Zg = [np.random.default_rng(3 + r).standard_normal((len(rows), Il)) for r in range(W)]
    W2 = [np.random.default_rng(9 + r).standard_normal((E, H, Il)) for r in range(W)]
    outs = O.moe_group_gemm_rs(rows, Zg, W2, w, M)
    for t in range(M):
        for h in range(H):
            ref = 0.0
            for r in range(W):
                for j, (e, tt, k) in enumerate(rows):
                    if tt == t:
                        ref += w[t, k] * sum(Zg[r][j, i] * W2[r][e, h, i] for i in range(Il))
            assert abs(outs[t // (M // W)][t % (M // W), h] - ref) < 1e-12


# --- sequence-parallel attention (NEXT-4): pins ------------------------------------
def test_attention_closed_forms():
    W, S, Hh, D = 2, 8, 2, 4
    Qs, Ks, Vs = TI.attention_inputs(S, Hh, D, W, seed=1)
    f = lambda L: [TI.to_f64(t) for t in L]
    # equal keys -> uniform weights -> every output row is the mean of V (per head)
    Kc = [np.ones_like(k) for k in f(Ks)]
    outs = O.sp_attention(f(Qs), Kc, f(Vs), 0.5)
    Vall = np.concatenate(f(Vs), 0)
    for o in outs:
        np.testing.assert_allclose(o, np.broadcast_to(Vall.mean(0), o.shape), rtol=1e-12, atol=1e-12)
    # V = 0 -> O = 0; V = const -> O = const
    assert all(np.all(o == 0) for o in O.sp_attention(f(Qs), f(Ks), [np.zeros_like(v) for v in f(Vs)], 0.3))
    outs = O.sp_attention(f(Qs), f(Ks), [np.full_like(v, 2.5) for v in f(Vs)], 0.3)
    assert all(np.allclose(o, 2.5, rtol=1e-14) for o in outs)


def test_attention_kv_permutation_invariance_and_brute_force():
    W, S, Hh, D = 2, 6, 1, 3
    Qs, Ks, Vs = TI.attention_inputs(S, Hh, D, W, seed=2)
    f = lambda L: [TI.to_f64(t) for t in L]
    a = O.sp_attention(f(Qs), f(Ks), f(Vs), 0.7)
    b = O.sp_attention(f(Qs), f(Ks)[::-1], f(Vs)[::-1], 0.7)       # gather order of the shards
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-13, atol=1e-14)
    # pure-Python softmax(q.k) v for one row
    K = [r for k in Ks for r in k.float().tolist()]
    V = [r for v in Vs for r in v.float().tolist()]
    q = Qs[1].float().tolist()[2][0]
    sc = [0.7 * sum(qi * ki for qi, ki in zip(q, kr[0])) for kr in K]
    mx = max(sc)
    e = [math.exp(x - mx) for x in sc]
    want = [sum(ei * vr[0][d] for ei, vr in zip(e, V)) / sum(e) for d in range(D)]
    np.testing.assert_allclose(a[1][2, 0], want, rtol=1e-12)
