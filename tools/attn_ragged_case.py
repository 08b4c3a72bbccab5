"""One SP-attention call at (W, S) checked against the oracle: python tools/attn_ragged_case.py W S
(used for the ragged-length memcheck runs, profiles/r01_sanitizer_memcheck_ragged_attention.log)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl
import tl_inputs as TI
from oracle import tl_oracle as O
W, S, heads = int(sys.argv[1]), int(sys.argv[2]), 3
Qs, Ks, Vs = TI.attention_inputs(S, heads, 128, W, seed=0)
need = 2 * S * heads * 128
comm = tl.Comm.loopback(W, 0, max_M=max(128, (need + 4095) // 4096), max_H=4096) if W > 1 else tl.Comm.single(0, max_M=max(128, (need + 4095) // 4096), max_H=4096)
comm.set_option("timeout_ms", 600000)
qd, kd, vd = ([t.cuda() for t in L] for L in (Qs, Ks, Vs))
outs = [torch.empty_like(q) for q in qd]
if W > 1:
    tl.sp_attention_lb(comm, qd, kd, vd, outs)
else:
    tl.sp_attention(comm, qd[0], kd[0], vd[0], outs[0])
st, diag = comm.check()
f = lambda L: [TI.to_f64(t) for t in L]
ref = np.concatenate(O.sp_attention(f(Qs), f(Ks), f(Vs), 128 ** -0.5), 0)
got = np.concatenate([o.float().cpu().double().numpy() for o in outs], 0)
print(f"W={W} S={S} status={st} err={O.rel_frobenius(got, ref):.3e}", flush=True)
