"""Attention-backward time at configs[1] (B=1 T=16 S=1024 C=1152, 16 heads) for the CTA item walk
chosen by DSP_FMHA_BWD_CH (set per process by the caller): graph replay, 20x, L2 not flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp

tok, C, NH = 16384, 1152, 16
ctx = dsp.Context()
g0 = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s: (torch.rand(*s, device="cuda", generator=g0) * 2 - 1).to(torch.bfloat16)
qkv, o, do, dqkv = r(tok, 3 * C), r(tok, C), r(tok, C), torch.empty(tok, 3 * C, dtype=torch.bfloat16, device="cuda")
lse = torch.zeros(tok, NH, dtype=torch.float32, device="cuda")
ctx.ensure_workspace(400 << 20)
res = {}
for dim in ("S", "T"):
    ctx.attention_core_lse(1, 16, 1024, C, NH, dim, qkv, o, lse)
    f = lambda: ctx.attention_core_bwd(1, 16, 1024, C, NH, dim, qkv, o, do, lse, dqkv)
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
    res[dim] = round(a.elapsed_time(b) / 20 * 1e3, 1)
print(f"DSP_FMHA_BWD_CH={os.environ.get('DSP_FMHA_BWD_CH', 'default')} attn_bwd_us {res}")
