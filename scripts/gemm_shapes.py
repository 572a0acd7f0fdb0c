"""Scratch: our tcgen05 GEMM at several N for M=16384, K=1152 / 4608, epilogue NONE vs GELU
(bytes staged per k-block per SM vs MMA time: is the mainloop feed-bound?)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
ctx = dsp.Context()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n * 1e3
M = 16384
for K in (1152, 4608):
    A = (torch.randn(M, K, device="cuda") * 0.1).to(torch.bfloat16)
    for N, epi in ((3456, 0), (3584, 0), (4608, 0), (4608, 2), (1152, 0), (1152, 1), (1280, 0), (2304, 0), (2048, 0)):
        W = (torch.randn(N, K, device="cuda") * 0.03).to(torch.bfloat16)
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        R = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
        us = t(lambda: ctx.linear(A, W, D, R, epi))
        print(f"K={K:5d} N={N:5d} epi={epi}: {us:7.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s")
