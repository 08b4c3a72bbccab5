"""Phase timeline of the attention kernel (trace build: nvcc ... -DTL_ATTN_TRACE, loaded via
TL_LIB_PATH).  Prints per KV block, for CTA 0's first unit: softmax A/B wait-for-S, max, exp+P
phases and the MMA issuer's waits for P (clock64 cycles)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_20313_b200 as tl  # noqa: E402

S, heads = int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 32
comm = tl.Comm.single(0, max_M=128, max_H=128)
for k, v in (("attn_poly", int(os.environ.get("POLY", "0"))), ("debug_drop_notify", int(os.environ.get("DROP", "-1")))):
    comm.set_option(k, v)
q = torch.randn(S, heads, 128, device="cuda").to(torch.bfloat16)
k_ = torch.randn_like(q)
v_ = torch.randn_like(q)
o = torch.empty_like(q)
for _ in range(3):
    tl.sp_attention(comm, q, k_, v_, o)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (5 * 64 * 4))()
C.CDLL(os.environ["TL_LIB_PATH"]).tl_debug_attn_trace(buf)
t = [list(buf[i * 4:(i + 1) * 4]) for i in range(5 * 64)]
base = min(x for row in t for x in row if x)
A, B, M, K, PR = t[0:64], t[64:128], t[128:192], t[192:256], t[256:320]
print("j | A: s_wait  max  exp+P | B: s_wait max exp+P | MMA: waitP_A waitP_B | A_start B_start (rel)")
print("timeline (rel to A s_full of block j): A.ready A.Pdone B.ready B.Pdone | mma: kwait0 kwait1 vwait0 pA0 pA1 pB0 pB1")
for j in range(1, 12):
    r = A[j][1]
    f = lambda x: x - r
    print(j, f(A[j][1]), f(A[j][3]), f(B[j][1]), f(B[j][3]), "|", f(K[j][0]), f(K[j][1]), f(K[j][2]), f(M[j][0]), f(M[j][1]),
          f(M[j][2]), f(M[j][3]), " next:", f(K[j+1][0]), f(K[j+1][1]), f(A[j+1][1]),
          "| producer j+2: kw", f(PR[j+2][0]), f(PR[j+2][1]), "vw", f(PR[j+2][2]), f(PR[j+2][3]))
for j in range(1, 40):
    a, b, m = A[j], B[j], M[j]
    print(f"{j:2d} | {a[1]-a[0]:6d} {a[2]-a[1]:5d} {a[3]-a[2]:6d} | {b[1]-b[0]:6d} {b[2]-b[1]:5d} {b[3]-b[2]:6d} |"
          f" {m[1]-m[0]:6d} {m[3]-m[2]:6d} | {a[1]-base:9d} {b[1]-base:9d}  period {A[j][1]-A[j-1][1]}")
