"""Launch / host overhead of the C-ABI ops on tiny and small-M shapes (eager vs CUDA graph)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2503_20313_b200 as tl  # noqa: E402


def run(M, N, K, n=200, act=0):
    c = tl.Comm.single(0, max_M=M, max_H=K)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn((2 if act else 1) * N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    for _ in range(10):
        c.ag_gemm(A, B, C, act=act, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        c.ag_gemm(A, B, C, act=act, stream=s)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    eager_gpu = e0.elapsed_time(e1) / n * 1e3
    host = (t1 - t0) / n * 1e6
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            for _ in range(n):
                c.ag_gemm(A, B, C, act=act, stream=gs)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph_gpu = e0.elapsed_time(e1) / n * 1e3
    print(f"M={M} N={N} K={K} act={act}: eager {eager_gpu:.1f} us/call (host {host:.1f} us/call), "
          f"graph {graph_gpu:.1f} us/call", flush=True)


if __name__ == "__main__":
    run(256, 256, 64)
    run(1024, 1024, 1024)
    run(1024, 1376, 4096, act=1)
    run(1024, 4096, 1376)
    run(8192, 1376, 4096, n=50, act=1)
    run(8192, 4096, 1376, n=50)
