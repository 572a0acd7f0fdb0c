"""Temporal FMHA at the long-video shape (T=128, 1024 columns of the 4096), for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
C = 1152
ctx = dsp.Context()
QL = (torch.randn(128 * 1024, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
OL = torch.empty(128 * 1024, C, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    ctx.attention_core(1, 128, 1024, C, 16, "T", QL, OL)
torch.cuda.synchronize()
print("ok")
