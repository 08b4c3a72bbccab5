"""Pure-Python triple-loop TP-MLP for tiny inputs (TEST INFRASTRUCTURE ONLY).

An independent second implementation of the same definitions as tl_oracle.py
(PAPER.md P:56 AG -> GEMM -> act -> GEMM -> RS, P:607 activation), written with
Python lists and `math` only -- no numpy -- so that a numpy-level mistake in
tl_oracle.py (a transposed operand, a wrong axis) cannot be reproduced here.
"""
from __future__ import annotations

import math


def _matmul_bt(A, B):
    """C[i][j] = sum_k A[i][k] * B[j][k]  (A . B^T with B in nn.Linear layout)."""
    n = len(B)
    K = len(A[0]) if A else 0
    out = []
    for i in range(len(A)):
        row = [0.0] * n
        Ai = A[i]
        for j in range(n):
            Bj = B[j]
            s = 0.0
            for k in range(K):
                s += Ai[k] * Bj[k]
            row[j] = s
        out.append(row)
    return out


def _act(Y, act):
    if act == 0:
        return Y
    il = len(Y[0]) // 2
    out = []
    for row in Y:
        g, u = row[:il], row[il:]
        if act == 1:
            out.append([gi / (1.0 + math.exp(-gi)) * ui for gi, ui in zip(g, u)])
        else:
            c = math.sqrt(2.0 / math.pi)
            out.append([0.5 * gi * (1.0 + math.tanh(c * (gi + 0.044715 * gi ** 3))) * ui
                        for gi, ui in zip(g, u)])
    return out


def mlp_forward(X_shards, W1_list, W2_list, act):
    """Lists-of-lists in, lists-of-lists out (one [M_r][H] block per rank)."""
    X = [list(map(float, row)) for shard in X_shards for row in shard]   # AllGather
    W = len(X_shards)
    M = len(X)
    m = M // W
    partials = []
    for W1, W2 in zip(W1_list, W2_list):
        Z = _act(_matmul_bt(X, [list(map(float, r)) for r in W1]), act)
        partials.append(_matmul_bt(Z, [list(map(float, r)) for r in W2]))
    outs = []
    for r in range(W):                                                   # ReduceScatter
        block = []
        for i in range(r * m, (r + 1) * m):
            row = [0.0] * len(partials[0][0])
            for s in range(W):
                row = [a + b for a, b in zip(row, partials[s][i])]
            block.append(row)
        outs.append(block)
    return outs
