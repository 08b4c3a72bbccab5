"""CPU oracle for the TileLink tensor-parallel MLP hot path (arXiv 2503.20313).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product path (paper_2503_20313_b200/) never imports, links or executes it,
and it shares no code, headers, helpers or constants with the CUDA library.

What it computes (plain definitions, fp64, simulated W ranks, no blocking,
no fusion, no reordering):

  * TP-FFN, PAPER.md P:56 (Sec. 2.1 "Intra-Layer Parallelism ..."): "First, input
    data is gathered from different ranks, followed by local computation using the
    corresponding weight shards. Finally, the partial results are reduced and
    scattered to the appropriate ranks."  -> AllGather, GEMM, activation, GEMM,
    ReduceScatter.
  * Activation between the two parts, PAPER.md P:607 (Sec. 7.2 "MLP Layer"):
    "there is one activation layer (e.g., SiLUMul or GeLUMul) between these two
    parts".
  * Static tile-centric mapping, PAPER.md P:410-420 (Sec. 4.1, the AllGather (pull)
    + GEMM example equations).
  * Overlap ratio, PAPER.md P:656-664 (Sec. 7.2 "Self-Attention Layer").

Readings of the paper where it is silent (listed in DESIGN.md "Readings"):
  R1 gated GEMM1 width 2*I/W with W1_r = [gate_r; up_r] (SiLUMul / GeLUMul);
  R5 after RS rank r owns rows [r*M_r, (r+1)*M_r) (global-view offset);
  R7 reduction order: ascending source rank (SPEC S:375-383 phase-separated oracle);
  R8 the oracle models NO intermediate rounding (fp64 end to end).

Every input is a float64 numpy array; bf16 inputs are converted exactly.
Parity pins for every function live in tests/test_oracle.py.
"""
from __future__ import annotations

import math

import numpy as np

ACT_NONE = 0
ACT_SILU_MUL = 1
ACT_GELU_TANH_MUL = 2


# ----------------------------------------------------------------------------
# Collectives (operator-centric definitions)
# ----------------------------------------------------------------------------
def all_gather_rows(shards):
    """AllGather along rows: concatenate rank shards in ascending rank order."""
    return np.concatenate([np.asarray(s, dtype=np.float64) for s in shards], axis=0)


def reduce_scatter_rows(partials):
    """ReduceScatter along rows: out_r = sum_{s=0}^{W-1} P_s[rows of r], ascending s.

    Rank r owns rows [r*M_r, (r+1)*M_r) with M_r = M / W (reading R5).
    """
    W = len(partials)
    M = partials[0].shape[0]
    assert M % W == 0
    m = M // W
    outs = []
    for r in range(W):
        acc = np.zeros_like(partials[0][r * m:(r + 1) * m], dtype=np.float64)
        for s in range(W):  # ascending source rank (reading R7)
            acc = acc + partials[s][r * m:(r + 1) * m]
        outs.append(acc)
    return outs


# ----------------------------------------------------------------------------
# Activation: act(gate) * up on the two halves of GEMM1's output
# ----------------------------------------------------------------------------
def silu(x):
    """SiLU(x) = x / (1 + exp(-x))."""
    x = np.asarray(x, dtype=np.float64)
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    """GeLU, tanh approximation: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def activation(Y, act: int):
    """Z = Y (NONE) or act(Y[:, :I_l]) * Y[:, I_l:] (SiLUMul / GeLUMul, reading R1)."""
    Y = np.asarray(Y, dtype=np.float64)
    if act == ACT_NONE:
        return Y
    n = Y.shape[1]
    assert n % 2 == 0
    il = n // 2
    gate, up = Y[:, :il], Y[:, il:]
    if act == ACT_SILU_MUL:
        return silu(gate) * up
    if act == ACT_GELU_TANH_MUL:
        return gelu_tanh(gate) * up
    raise ValueError(f"unknown act {act}")


# ----------------------------------------------------------------------------
# The three operations of the boundary
# ----------------------------------------------------------------------------
def ag_gemm(A_shards, B_list):
    """AG-GEMM: X = AllGather_rows(A_r);  C_r = X . B_r^T  (B_r in nn.Linear layout [N_l, K]).

    Returns (X, [C_r]).  P:56 first half ("gathered ... followed by local computation").
    """
    X = all_gather_rows(A_shards)
    Cs = [X @ np.asarray(B, dtype=np.float64).T for B in B_list]
    return X, Cs


def gemm_rs(A_list, B_list):
    """GEMM-RS: P_r = A_r . B_r^T, out_r = sum_s P_s[rows of r].  P:56 second half."""
    partials = [np.asarray(A, dtype=np.float64) @ np.asarray(B, dtype=np.float64).T
                for A, B in zip(A_list, B_list)]
    return reduce_scatter_rows(partials)


def mlp_forward(X_shards, W1_list, W2_list, act: int):
    """Tensor-parallel FFN: out_r = RS(act(AG(X) . W1_r^T) . W2_r^T)."""
    X, Ys = ag_gemm(X_shards, W1_list)
    Zs = [activation(Y, act) for Y in Ys]
    return gemm_rs(Zs, W2_list)


def mlp_forward_rows(X_shards, W1_list, W2_list, act: int, rows):
    """Exact oracle restricted to global output rows `rows` (rows are independent).

    Returns {global_row: out_row}.  Same steps as mlp_forward, evaluated only on the
    requested rows of the gathered X: out[i] = sum_s act(X[i] . W1_s^T) . W2_s^T.
    """
    X = all_gather_rows(X_shards)
    Xs = X[np.asarray(rows)]
    acc = None
    for W1, W2 in zip(W1_list, W2_list):  # ascending source rank
        Z = activation(Xs @ np.asarray(W1, dtype=np.float64).T, act)
        P = Z @ np.asarray(W2, dtype=np.float64).T
        acc = P if acc is None else acc + P
    return {int(i): acc[j] for j, i in enumerate(rows)}


# ----------------------------------------------------------------------------
# Static tile-centric mapping, PAPER.md P:410-420 (Sec. 4.1), literal
# ----------------------------------------------------------------------------
def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def static_shape_range(t: int, M: int, Tm: int):
    """range_M = [t*Tm, t*Tm + Tm), last tile clamped to M."""
    lo = t * Tm
    if lo >= M:
        raise ValueError("tile out of grid")
    return lo, min(lo + Tm, M)


def static_src_rank(t: int, M: int, R: int, Tm: int) -> int:
    """src_rank = floor(t / floor(M_per_rank / Tm)), M_per_rank = ceil(M/R)."""
    m_per_rank = ceil_div(M, R)
    tiles = m_per_rank // Tm
    if tiles == 0:
        raise ValueError("Tm > M_per_rank: the paper's formula is undefined (reading R4)")
    return t // tiles


def static_channel(t: int, M: int, R: int, C: int, Tm: int) -> int:
    """channel = floor(t / floor(M_per_channel / Tm)), M_per_channel = ceil(M/(R*C))."""
    m_per_channel = ceil_div(M, R * C)
    tiles = m_per_channel // Tm
    if tiles == 0:
        raise ValueError("Tm > M_per_channel: the paper's formula is undefined (reading R4)")
    return t // tiles


def consumer_wait_channels(m0: int, m1: int, M: int, R: int, C: int):
    """Channels a consumer tile covering rows [m0, m1) waits on ("Similarly").

    A consumer tile depends on every producer row it reads; with channel granularity
    M_per_channel = ceil(M/(R*C)) those are channels floor(m0/Mpc) .. floor((m1-1)/Mpc).
    """
    mpc = ceil_div(M, R * C)
    return list(range(m0 // mpc, (m1 - 1) // mpc + 1))


# ----------------------------------------------------------------------------
# Overlap ratio
# ----------------------------------------------------------------------------
def overlap_ratio(comp_only: float, comm_only: float, overlap: float) -> float:
    """ratio = (comp_only + comm_only - overlap) / comm_only."""
    if comm_only <= 0:
        raise ValueError("comm_only must be > 0")
    return (comp_only + comm_only - overlap) / comm_only


# ----------------------------------------------------------------------------
# Comparison rule (BASELINE.json north star)
# ----------------------------------------------------------------------------
def rel_frobenius(got, ref) -> float:
    """||G - O||_F / ||O||_F in fp64."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / den) if den > 0 else float(np.linalg.norm(got - ref))


# ----------------------------------------------------------------------------
# MoE first half: AllGather + Gather + GroupGEMM
# ----------------------------------------------------------------------------
def moe_group_rows(topk_ids, E: int):
    """Grouped order of the routed rows (the dynamic shape mapping of P:422-431 made concrete):
    every (token t, slot k) with expert e = topk_ids[t, k], sorted stably by (expert, token) --
    tokens are rank-sharded contiguously, so this is (expert, source rank, token).
    Returns a list of (e, t, k)."""
    ids = np.asarray(topk_ids)
    M, topk = ids.shape
    rows = []
    for t in range(M):
        for k in range(topk):
            e = int(ids[t, k])
            if not 0 <= e < E:
                raise ValueError("expert id out of range")
            rows.append((e, t, k))
    rows.sort(key=lambda x: (x[0], x[1]))   # Python's sort is stable: equal (e, t) keep slot order
    return rows


def moe_ag_group_gemm(X_shards, topk_ids, W1_list, act: int):
    """AG + Gather + GroupGEMM: X = AllGather_rows(X_r); for every routed row
    (e, t, k) in grouped order, Y_r[row] = act(X[t] . W1_r[e]^T), W1_r[e] in nn.Linear layout
    ([N1, H]; [gate; up] halves for the *_MUL acts).  Returns (rows, [Y_r])."""
    X = all_gather_rows(X_shards)
    E = np.asarray(W1_list[0]).shape[0]
    rows = moe_group_rows(topk_ids, E)
    Ys = []
    for W1 in W1_list:
        W1 = np.asarray(W1, dtype=np.float64)
        Y = np.stack([activation(X[t][None, :] @ W1[e].T, act)[0] for (e, t, k) in rows]) if rows else \
            np.zeros((0, W1.shape[1] // (1 if act == ACT_NONE else 2)))
        Ys.append(Y)
    return rows, Ys


# ----------------------------------------------------------------------------
# MoE second half: GroupGEMM + Scatter + TopK reduce + ReduceScatter
# ----------------------------------------------------------------------------
def moe_group_gemm_rs(rows, Zg_list, W2_list, topk_weights, M: int):
    """P:632/P:647 second part: P_s[j] = Zg_s[j] . W2_s[e_j]^T for every grouped row j = (e, t, k);
    scatter back to the token and reduce over its top-k slots with the router weights,
    Q_s[t] = sum_k w[t, k] P_s[j(t, k)]; then ReduceScatter over ranks: out_r = sum_s Q_s[rows of r]."""
    w = np.asarray(topk_weights, dtype=np.float64)
    Qs = []
    for Zg, W2 in zip(Zg_list, W2_list):
        Zg = np.asarray(Zg, dtype=np.float64)
        W2 = np.asarray(W2, dtype=np.float64)
        Q = np.zeros((M, W2.shape[1]))
        for j, (e, t, k) in enumerate(rows):   # scatter + top-k reduce, in grouped order
            Q[t] += w[t, k] * (Zg[j] @ W2[e].T)
        Qs.append(Q)
    return reduce_scatter_rows(Qs)


def moe_forward(X_shards, topk_ids, topk_weights, W1_list, W2_list, act: int):
    """TP MoE FFN: AG + Gather + GroupGEMM + act, then GroupGEMM + Scatter + TopK reduce + RS."""
    rows, Zs = moe_ag_group_gemm(X_shards, topk_ids, W1_list, act)
    M = sum(np.asarray(x).shape[0] for x in X_shards)
    return moe_group_gemm_rs(rows, Zs, W2_list, topk_weights, M)


# ----------------------------------------------------------------------------
# Sequence-parallel attention: AllGather KV + self-attention
# ----------------------------------------------------------------------------
def softmax_rows(S):
    """Row softmax: exp(S - max) / sum(exp(S - max)) (the max shift is exact algebra)."""
    S = np.asarray(S, dtype=np.float64)
    E = np.exp(S - S.max(axis=1, keepdims=True))
    return E / E.sum(axis=1, keepdims=True)


def sp_attention(Q_shards, K_shards, V_shards, scale: float):
    """"the context (key and value) is sharded across devices. Before computation, these context
    shards are gathered to form a complete context for self-attention".  Shards are [S_r, heads, D];
    K = AllGather(K_r), V = AllGather(V_r); O_r[:, h] = softmax(scale * Q_r[:, h] K[:, h]^T) V[:, h]
    (non-causal).  Returns [O_r]."""
    K = all_gather_rows(K_shards)
    V = all_gather_rows(V_shards)
    outs = []
    for Q in Q_shards:
        Q = np.asarray(Q, dtype=np.float64)
        O = np.zeros_like(Q)
        for h in range(Q.shape[1]):
            O[:, h] = softmax_rows(scale * (Q[:, h] @ K[:, h].T)) @ V[:, h]
        outs.append(O)
    return outs
