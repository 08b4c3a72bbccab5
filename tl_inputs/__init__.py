"""Seeded synthetic input generators shared by the oracle tests and the CUDA tests.

This module holds NO arithmetic of the method (no gather, no GEMM, no activation,
no reduction): it only draws seeded random tensors, rounds them to bf16 and slices
them into the per-rank layout the C ABI expects.  Both `oracle/` and the CUDA
path consume its outputs; neither side imports the other.

Recipe:
  * X  ~ N(0, 1)        [M, H]   post-norm activations
  * G, U ~ N(0, 1/H)    [I, H]   gate / up projection rows (nn.Linear layout)
  * W2 ~ N(0, 1/I)      [H, I]   down projection (nn.Linear layout)
  all rounded to bf16 (round-to-nearest-even, torch's cast), generated on the CPU
  with `torch.Generator().manual_seed(seed + tensor_id)` so every world size W
  sees the same full problem.

Shard layout (the tensor-parallel FFN of PAPER.md P:56, reading SURVEY §8(c)#1):
  X_r  = X[r*M_r:(r+1)*M_r]                    row shard, M_r = M / W
  W1_r = [G[r*I_l:(r+1)*I_l]; U[r*I_l:(r+1)*I_l]]   (gated acts)   [2*I_l, H]
       =  G[r*I_l:(r+1)*I_l]                         (act NONE)     [I_l, H]
  W2_r = W2[:, r*I_l:(r+1)*I_l]                                  [H, I_l]
"""
from __future__ import annotations

import torch

ACT_NONE = 0
ACT_SILU_MUL = 1
ACT_GELU_TANH_MUL = 2

_TID_X, _TID_G, _TID_U, _TID_W2, _TID_A, _TID_B = 0, 1, 2, 3, 4, 5


def _randn(shape, seed: int, tid: int, std: float = 1.0, device=None) -> torch.Tensor:
    """Seeded N(0, std^2) draw rounded to bf16.  `device=None`: CPU generator (the tests' recipe);
    a CUDA device: the same recipe with that device's (Philox) generator -- a different but equally
    seeded stream, identical on every rank that draws it (bench.py's large shapes)."""
    dev = torch.device("cpu") if device is None else torch.device(device)
    g = torch.Generator(device=dev).manual_seed(int(seed) * 1000 + tid)
    t = torch.randn(*shape, generator=g, dtype=torch.float32, device=dev)
    if std != 1.0:
        t.mul_(std)
    return t.to(torch.bfloat16)


def mlp_full(M: int, H: int, I: int, seed: int = 0, device=None):
    """Full (unsharded) LLaMA-style MLP problem: X [M,H], G [I,H], U [I,H], W2 [H,I], bf16 (CPU, or drawn
    on `device`)."""
    X = _randn((M, H), seed, _TID_X, device=device)
    G = _randn((I, H), seed, _TID_G, H ** -0.5, device=device)
    U = _randn((I, H), seed, _TID_U, H ** -0.5, device=device)
    W2 = _randn((H, I), seed, _TID_W2, I ** -0.5, device=device)
    return X, G, U, W2


def shard_rows(T: torch.Tensor, W: int):
    """Split rows into W equal contiguous shards (rank r gets rows [r*M/W, (r+1)*M/W))."""
    M = T.shape[0]
    assert M % W == 0, "M must be divisible by the world size"
    m = M // W
    return [T[r * m:(r + 1) * m].contiguous() for r in range(W)]


def shard_mlp(X, G, U, W2, W: int, act: int):
    """Per-rank tensors (X_r, W1_r, W2_r) for world size W (see module docstring)."""
    I = G.shape[0]
    assert I % W == 0, "I must be divisible by the world size"
    il = I // W
    Xs = shard_rows(X, W)
    W1s, W2s = [], []
    for r in range(W):
        g = G[r * il:(r + 1) * il]
        if act == ACT_NONE:
            W1s.append(g.contiguous())
        else:
            W1s.append(torch.cat([g, U[r * il:(r + 1) * il]], 0).contiguous())
        W2s.append(W2[:, r * il:(r + 1) * il].contiguous())
    return Xs, W1s, W2s


def gemm_rs_inputs(M: int, N: int, K_local: int, W: int, seed: int = 0):
    """Random per-rank GEMM-RS operands: A_r [M, K_l] ~ N(0,1), B_r [N, K_l] ~ N(0, 1/(W*K_l))."""
    As = [_randn((M, K_local), seed + 17 * r, _TID_A) for r in range(W)]
    Bs = [_randn((N, K_local), seed + 17 * r, _TID_B, (W * K_local) ** -0.5) for r in range(W)]
    return As, Bs


def ag_gemm_inputs(M: int, N_local: int, K: int, W: int, seed: int = 0):
    """Random AG-GEMM operands: A_r [M/W, K] ~ N(0,1), B_r [N_l, K] ~ N(0, 1/K)."""
    A = _randn((M, K), seed, _TID_A)
    Bs = [_randn((N_local, K), seed + 31 * r, _TID_B, K ** -0.5) for r in range(W)]
    return shard_rows(A, W), Bs


def _bits(i: torch.Tensor, nb: int) -> torch.Tensor:
    return torch.stack([(i >> b) & 1 for b in range(nb)], 1)


def ag_placement_inputs(M: int, K: int, N_local: int, W: int):
    """Index-check fixture for AG-GEMM (SURVEY §8(c) pin 7).

    X[i, b] = bit_b(i) for b < 16 (other columns 0).  Weight row n holds 2^(b-4q)
    on columns b in [4q, 4q+4) with q = n mod 4 (and a rank-dependent row shift so
    every rank's weight differs).  Then C_r[i, n] = nibble_{(n + r) mod 4}(i), a small
    integer (exact in bf16/fp32), so any misplaced row or column is detected.
    """
    assert K >= 16
    idx = torch.arange(M, dtype=torch.int64)
    X = torch.zeros(M, K, dtype=torch.float32)
    X[:, :16] = _bits(idx, 16).to(torch.float32)
    Bs = []
    for r in range(W):
        B = torch.zeros(N_local, K, dtype=torch.float32)
        for n in range(N_local):
            q = (n + r) % 4
            for j in range(4):
                B[n, 4 * q + j] = float(1 << j)
        Bs.append(B.to(torch.bfloat16))
    return shard_rows(X.to(torch.bfloat16), W), Bs


def rs_placement_inputs(M: int, N: int, K_local: int, W: int):
    """Index-check fixture for GEMM-RS (SURVEY §8(c) pin 7).

    A_r[i, b] = bit_b(i) (b < 16) and A_r[i, 16] = 1 (rank marker column).
    B_r[h, 4q + j] = 2^j with q = h mod 4, and B_r[h, 16] = (h mod 3) * r.
    Then out[i, h] = W * nibble_{h mod 4}(i) + (h mod 3) * W (W - 1) / 2, an integer <= 176 at W = 8.
    """
    assert K_local >= 17
    idx = torch.arange(M, dtype=torch.int64)
    A = torch.zeros(M, K_local, dtype=torch.float32)
    A[:, :16] = _bits(idx, 16).to(torch.float32)
    A[:, 16] = 1.0
    As, Bs = [], []
    for r in range(W):
        As.append(A.to(torch.bfloat16).clone())
        B = torch.zeros(N, K_local, dtype=torch.float32)
        h = torch.arange(N)
        q = h % 4
        for j in range(4):
            B[h, 4 * q + j] = float(1 << j)
        B[:, 16] = ((h % 3) * r).to(torch.float32)
        Bs.append(B.to(torch.bfloat16))
    return As, Bs


def to_f64(t: torch.Tensor):
    """bf16 torch tensor -> float64 numpy array (exact: every bf16 value is an fp64 value)."""
    return t.to(torch.float64).numpy()


def moe_routing(M: int, E: int, topk: int, seed: int = 0, skew: float = 0.0):
    """Seeded top-k routing: topk distinct experts per token, int32 [M, topk].

    skew = 0 draws experts uniformly; skew > 0 draws them with weights ~ (e + 1)^-skew (a few hot
    experts, as real routers produce).  No arithmetic of the method."""
    g = torch.Generator().manual_seed(int(seed) * 1000 + 7)
    w = (torch.arange(E, dtype=torch.float64) + 1.0) ** (-float(skew))
    ids = torch.multinomial(w.expand(M, E).contiguous(), topk, replacement=False, generator=g)
    return ids.to(torch.int32)


def moe_weights(E: int, N1: int, H: int, W: int, seed: int = 0):
    """Per-rank expert weights [E, N1, H] bf16 ~ N(0, 1/H) (each rank's TP shard of every expert)."""
    return [_randn((E, N1, H), seed + 13 * r, _TID_B, H ** -0.5) for r in range(W)]


def moe_placement_inputs(M: int, H: int, E: int, N1: int, W: int):
    """Index fixture for the gather: X[t, b] = bit_b(t) (b < 16), expert e's weight row n picks the
    nibble (n + e) mod 4 -> Y[row, n] = nibble_{(n + e) mod 4}(t): exact, unique per (token, expert)."""
    assert H >= 16
    idx = torch.arange(M, dtype=torch.int64)
    X = torch.zeros(M, H, dtype=torch.float32)
    X[:, :16] = _bits(idx, 16).to(torch.float32)
    Ws = []
    for r in range(W):
        B = torch.zeros(E, N1, H, dtype=torch.float32)
        for e in range(E):
            for n in range(N1):
                q = (n + e + r) % 4
                for j in range(4):
                    B[e, n, 4 * q + j] = float(1 << j)
        Ws.append(B.to(torch.bfloat16))
    return shard_rows(X.to(torch.bfloat16), W), Ws


def moe_topk_weights(M: int, topk: int, seed: int = 0):
    """Router weights: a seeded softmax-like positive row of topk values summing to 1, fp32 [M, topk]."""
    g = torch.Generator().manual_seed(int(seed) * 1000 + 9)
    w = torch.rand(M, topk, generator=g, dtype=torch.float32) + 0.1
    return (w / w.sum(1, keepdim=True)).contiguous()


def moe_down_weights(E: int, H: int, I_l: int, W: int, seed: int = 0):
    """Per-rank expert down projections [E, H, I_l] bf16 ~ N(0, 1/(W * I_l))."""
    return [_randn((E, H, I_l), seed + 19 * r, _TID_W2, (W * I_l) ** -0.5) for r in range(W)]


def attention_inputs(S: int, heads: int, D: int, W: int, seed: int = 0):
    """Q, K, V ~ N(0, 1) [S, heads, D] bf16, row-sharded along the sequence over W ranks."""
    Q = _randn((S, heads, D), seed, 10)
    K = _randn((S, heads, D), seed, 11)
    V = _randn((S, heads, D), seed, 12)
    return shard_rows(Q, W), shard_rows(K, W), shard_rows(V, W)
