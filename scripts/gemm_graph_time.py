"""GEMM timing at the block's shapes (M = 16384 and the N = 8 shard M = 2048): 10 back-to-back
launches captured in one CUDA graph, L2 flushed before each replay; epilogues NONE / +residual /
GELU.  A/B across library variants via DSP_LIB_OVERRIDE."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
ctx = dsp.Context()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, reps=10, n=8):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        for _ in range(reps): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True); acc = []
    for _ in range(n):
        flush.zero_(); a.record(); g.replay(); b.record(); torch.cuda.synchronize(); acc.append(a.elapsed_time(b))
    acc.sort(); return acc[len(acc) // 2] / reps * 1e3
name = os.environ.get("DSP_LIB_OVERRIDE", "libdsp.so")[-22:]
C = 1152
for M in (16384, 2048):
    for K, N, epi, tag in ((C, 3 * C, 0, "QKV"), (C, C, 1, "PROJ+res"), (C, C, 0, "PROJ none"), (C, 2 * C, 0, "N=2304"), (C, 4 * C, 2, "FC1 gelu"), (C, 4 * C, 0, "FC1 none"),
                           (4 * C, C, 1, "FC2+res")):
        A = (torch.randn(M, K, device="cuda") * 0.1).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.03).to(torch.bfloat16)
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        R = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
        us = t(lambda: ctx.linear(A, W, D, R, epi))
        print(f"{name:22s} M={M:6d} {tag:9s} K={K:5d} N={N:5d}: {us:7.2f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s", flush=True)
