"""Tile periods (SM cycles) of the MoE GroupGEMMs from the device trace, against the MMA bound of one
256 x 512 (or 256 x 256) tile: is the gather GroupGEMM MMA-bound or gather-issue-bound?

  python tools/moe_timeline.py [opts]        e.g. "n_sub=1"  (MoE-4: S 8192, H 4096, I 2048, E 8, top-2, W 1)
"""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402
import tl_inputs as TI  # noqa: E402
from paper_2503_20313_b200.trace import read_events  # noqa: E402


def main():
    opts = sys.argv[1] if len(sys.argv) > 1 else ""
    S, H, I, E, topk = 8192, 4096, 2048, 8, 2
    X = TI._randn((S, H), 0, 0).cuda()
    Wt = TI.moe_weights(E, 2 * I, H, 1, seed=1)[0].cuda()
    ids = TI.moe_routing(S, E, topk, seed=2).cuda()
    c = tl.Comm.single(0, max_M=S, max_H=H)
    for kv in filter(None, opts.split(",")):
        k, v = kv.split("=")
        c.set_option(k, int(v))
    R = tl.moe_capacity(c, S, topk, E)
    Y = torch.empty(R, I, device="cuda", dtype=torch.bfloat16)
    rows = torch.empty(R, device="cuda", dtype=torch.int32)
    offs = torch.empty(E + 1, device="cuda", dtype=torch.int32)
    run = lambda: tl.moe_ag_gemm(c, X, ids, Wt, Y, rows, offs, act=tl.ACT_SILU_MUL)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    print(f"untraced: {a.elapsed_time(b) / 10 * 1e3:.1f} us per call")
    c.set_option("trace_events", 1 << 15)
    run()
    torch.cuda.synchronize()
    ev = read_events(c, clocks=True)
    clk = {e["tile"]: e["t_ns"] for e in ev if e["kind"] == "sm_clock"}
    n_pairs = 74
    by_pair = {}
    for t in sorted(clk):
        by_pair.setdefault(t % n_pairs, []).append(clk[t])
    per = []
    for v in by_pair.values():
        v.sort()
        per += [y - x for x, y in zip(v, v[1:])]
    nsub = c.get_option("n_sub") or 2
    kb = H // 64
    bound = kb * 512 * nsub
    print(f"tiles {len(clk)}; period (SM cycles) min {min(per)} med {statistics.median(per)} max {max(per)}; "
          f"MMA bound {bound} -> {bound / statistics.median(per):.3f}")


if __name__ == "__main__":
    main()
