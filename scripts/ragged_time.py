"""Cost of ragged sequence lengths (R33) in the attention core: time per token of the
temporal / spatial FMHA at aligned vs ragged lengths, same token count order (C = 1152)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
C = 1152
ctx = dsp.Context()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n * 1e3
for dim, cases in (("T", [(16, 1024), (51, 1024), (64, 1024), (100, 1024), (128, 1024)]),
                   ("S", [(16, 1000), (16, 1024), (16, 576), (16, 640)])):
    for a, b in cases:
        T, S = (a, b)
        tok = T * S
        QKV = (torch.randn(tok, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
        O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
        us = t(lambda: ctx.attention_core(1, T, S, C, 16, dim, QKV, O))
        L = T if dim == "T" else S
        print(f"{dim} L={L:5d} (T={T}, S={S}): {us:8.1f} us  {us * 1e3 / tok:6.3f} ns/token  "
              f"{4 * tok * L * C / us / 1e6:7.1f} TFLOP/s (attention flops over valid keys)")
