"""Scratch: is a GEMM output element bitwise independent of the tile width BN?  Writes the
outputs of the out-projection / FC2 shapes (N = 1152) for the library in DSP_LIB_OVERRIDE."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
ctx = dsp.Context()
g = torch.Generator(device="cuda").manual_seed(0)
out = {}
for M, K in ((16384, 1152), (4096, 4608)):
    A = (torch.randn(M, K, device="cuda", generator=g)).to(torch.bfloat16)
    W = (torch.randn(1152, K, device="cuda", generator=g) * K ** -0.5).to(torch.bfloat16)
    R = torch.randn(M, 1152, device="cuda", generator=g).to(torch.bfloat16)
    for epi in (0, 1):
        D = torch.empty(M, 1152, device="cuda", dtype=torch.bfloat16)
        ctx.linear(A, W, D, R if epi else None, epi)
        out[f"{M}x{K}e{epi}"] = D.cpu()
torch.save(out, sys.argv[1])
