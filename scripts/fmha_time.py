"""Scratch timing of the spatial / temporal FMHA at blk N=1 (CUDA events, 20 launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
tok, C = 16384, 1152
QKV = (torch.randn(tok, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
ctx = dsp.Context()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n * 1e3
for _ in range(2):
    us = t(lambda: ctx.attention_core(1, 16, 1024, C, 16, "S", QKV, O))
    ut = t(lambda: ctx.attention_core(1, 16, 1024, C, 16, "T", QKV, O))
    print(f"{os.environ.get('DSP_LIB_OVERRIDE', 'libdsp.so'):50s} spatial {us:7.1f} us ({4*16*1024*1024*C/us/1e6:6.1f} TFLOP/s)  temporal {ut:6.1f} us")
