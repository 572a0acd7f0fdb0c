"""LayerNorm backward (dsp_layer_norm_bwd: dx pass, dgamma/dbeta partials, column sums) at configs[1]
(16384 rows, C = 1152), graph replay 20x, for the variant selected by the environment (A/B runs of the row-group count used DSP_LN_RG, since removed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp

tok, C = 16384, 1152
ctx = dsp.Context()
r = lambda *s: (torch.rand(*s, device="cuda") * 2 - 1).to(torch.bfloat16)
x, dh, dres, dx, gam = r(tok, C), r(tok, C), r(tok, C), r(tok, C), r(C) + 1
gb = torch.zeros(2 * C, dtype=torch.float32, device="cuda")
ctx.ensure_workspace(64 << 20)
f = lambda: ctx.layer_norm_bwd(x, gam, dh, dres, dx, gb)
for _ in range(3):
    f()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
g.replay()
a.record()
for _ in range(20):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"DSP_LN_RG={os.environ.get('DSP_LN_RG', 'default')} ln_bwd_us {a.elapsed_time(b) / 20 * 1e3:.1f}")
