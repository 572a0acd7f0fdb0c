"""Per-operation graph-replay times of the block backward's building blocks at configs[1] (B=1 T=16
S=1024 C=1152, N=1), each op captured alone and replayed 20x (L2 not flushed): compare their sum with
the backward graph of bench.py --config train to size the inter-kernel gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp

tok, C, NH = 16384, 1152, 16
dev = "cuda"
ctx = dsp.Context()
r = lambda *s: (torch.rand(*s, device=dev) * 2 - 1).to(torch.bfloat16)
A = {"dz": r(tok, C), "g": r(tok, 4 * C), "u": r(tok, 4 * C), "du": r(tok, 4 * C), "h": r(tok, C), "x": r(tok, C),
     "qkv": r(tok, 3 * C), "o": r(tok, C), "do": r(tok, C), "dqkv": r(tok, 3 * C), "dh": r(tok, C), "y": r(tok, C)}
W = {"fc1": r(4 * C, C) * 0.03, "fc2": r(C, 4 * C) * 0.03, "qkv": r(3 * C, C) * 0.03, "o": r(C, C) * 0.03,
     "ln": r(C) + 1}
G = {k: torch.zeros(v.shape, dtype=torch.float32, device=dev) for k, v in W.items()}
gb = torch.zeros(2 * C, dtype=torch.float32, device=dev)
lse = torch.zeros(tok, NH, dtype=torch.float32, device=dev)
ctx.attention_core_lse(1, 16, 1024, C, NH, "S", A["qkv"], A["o"], lse)
ctx.attention_core_lse(1, 16, 1024, C, NH, "T", A["qkv"], A["o"], lse)
big = 600 << 20
ctx.ensure_workspace(big)
out = {k: torch.empty_like(v) for k, v in A.items()}
ops = {
    "dgrad FC2 +gelu'": lambda: ctx.linear_dgrad(A["dz"], W["fc2"], out["du"], u=A["u"]),
    "wgrad FC2": lambda: ctx.linear_wgrad(A["dz"], A["g"], G["fc2"]),
    "dgrad FC1": lambda: ctx.linear_dgrad(A["du"], W["fc1"], out["dh"]),
    "wgrad FC1": lambda: ctx.linear_wgrad(A["du"], A["h"], G["fc1"]),
    "LN bwd": lambda: ctx.layer_norm_bwd(A["y"], W["ln"], A["dh"], A["dz"], out["x"], gb),
    "dgrad PROJ": lambda: ctx.linear_dgrad(A["dz"], W["o"], out["do"]),
    "wgrad PROJ": lambda: ctx.linear_wgrad(A["dz"], A["o"], G["o"]),
    "attn bwd T": lambda: ctx.attention_core_bwd(1, 16, 1024, C, NH, "T", A["qkv"], A["o"], A["do"], lse, out["dqkv"]),
    "attn bwd S": lambda: ctx.attention_core_bwd(1, 16, 1024, C, NH, "S", A["qkv"], A["o"], A["do"], lse, out["dqkv"]),
    "dgrad QKV": lambda: ctx.linear_dgrad(A["dqkv"], W["qkv"], out["dh"]),
    "wgrad QKV": lambda: ctx.linear_wgrad(A["dqkv"], A["h"], G["qkv"]),
}
tot = 0.0
for name, f in ops.items():
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
    us = a.elapsed_time(b) / 20 * 1e3
    tot += us * (2 if ("PROJ" in name or "QKV" in name or "LN" in name) else 1) if "attn" not in name else us
    print(f"{name:20s} {us:8.1f} us")
print(f"backward estimate (PROJ/QKV/LN x2 + both attentions): {tot:.1f} us")
