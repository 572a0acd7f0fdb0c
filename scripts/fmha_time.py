"""Scratch timing of the FMHA at blk N=1 (spatial / temporal) and the long-video temporal
shape (T=128, 1024 columns), CUDA events over 20 launches."""
import sys, os
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
QKV = (torch.randn(16384, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
O = torch.empty(16384, C, dtype=torch.bfloat16, device="cuda")
QL = (torch.randn(128 * 1024, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
OL = torch.empty(128 * 1024, C, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    us = t(lambda: ctx.attention_core(1, 16, 1024, C, 16, "S", QKV, O))
    ut = t(lambda: ctx.attention_core(1, 16, 1024, C, 16, "T", QKV, O))
    ul = t(lambda: ctx.attention_core(1, 128, 1024, C, 16, "T", QL, OL))
    name = os.environ.get('DSP_LIB_OVERRIDE', 'libdsp.so')[-20:]
    print(f"{name:20s} spatial {us:7.1f} us  temporal {ut:6.1f} us ({4*16384*C*2/ut/1e3:6.0f} GB/s)  "
          f"temporal T=128 x 1024 cols {ul:7.1f} us ({4*128*1024*C*2/ul/1e3:6.0f} GB/s)")
