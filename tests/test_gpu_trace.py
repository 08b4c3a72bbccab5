"""Device event trace of the fused kernels (option trace_events): well-formed, complete, and without
effect on the results."""
import pytest
import torch

import tl_inputs as TI

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tl():
    import paper_2503_20313_b200 as m
    m.lib()
    return m


def test_trace_counts_and_no_effect_on_results(tl):
    from paper_2503_20313_b200 import trace as T
    W, M, H, I, rows = 4, 1024, 512, 2048, 32
    X, G, U, W2 = TI.mlp_full(M, H, I, seed=41)
    xs, w1s, w2s = ([t.cuda() for t in L] for L in TI.shard_mlp(X, G, U, W2, W, TI.ACT_SILU_MUL))
    c = tl.Comm.loopback(W, 0, max_M=M, max_H=H)
    c.set_option("comm_tile_rows", rows)
    Zs = [torch.empty(M, I // W, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    outs = [torch.empty(M // W, H, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    c.ag_gemm_lb(xs, w1s, Zs, act=tl.ACT_SILU_MUL)
    c.gemm_rs_lb(Zs, w2s, outs)
    ref = [o.clone() for o in outs]
    assert T.read_events(c, cap=16) == []                       # no trace while the option is off
    c.set_option("trace_events", 1 << 16)
    c.ag_gemm_lb(xs, w1s, Zs, act=tl.ACT_SILU_MUL)
    ev_ag = T.read_events(c)
    c.gemm_rs_lb(Zs, w2s, outs)
    ev_rs = T.read_events(c)
    assert c.check()[0] == 0
    for r in range(W):
        assert torch.equal(outs[r], ref[r])
    for evs in (ev_ag, ev_rs):
        rep = T.analyze_trace(evs)
        assert rep["diagnostics"] == []
        assert all(evs[i]["t_ns"] <= evs[i + 1]["t_ns"] for i in range(len(evs) - 1))
    # AG: every rank copies each of its (M/W)/rows producer tiles to all W ranks and notifies each
    tiles = (M // W) // rows
    for r in range(W):
        cs = [e for e in ev_ag if e["rank"] == r and e["kind"] == "copy_start"]
        nt = [e for e in ev_ag if e["rank"] == r and e["kind"] == "notify" and e["unit"] == "copy"]
        assert len(cs) == len(nt) == tiles * W
        assert sorted((e["tile"], e["peer"]) for e in nt) == sorted((t, d) for t in range(tiles) for d in range(W))
        ts = [e for e in ev_ag if e["rank"] == r and e["kind"] == "tile_start"]
        ws = [e for e in ev_ag if e["rank"] == r and e["kind"] == "wait_start"]
        assert len(ts) > 0 and len(ws) == len(ts)             # every GEMM1 tile waited for its rows
    # RS: every rank pushes its partial tiles of the W - 1 other owners' blocks
    for r in range(W):
        pushes = [e for e in ev_rs if e["rank"] == r and e["kind"] == "notify"]
        assert pushes and {e["peer"] for e in pushes} == set(range(W)) - {r}
