"""Scratch timing of the block and its kernels at blk N=1 (not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp, synth
sh = synth.CONFIGS["blk"]
to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
X = to(synth.make_x(sh, 7)); W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
ctx = dsp.Context(); shape = dsp.make_shape(1, 16, 1024, 1152, 16, "bf16")
ctx.ensure_workspace(dsp.workspace_bytes(shape, 1)); Y = torch.empty_like(X)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = torch.cuda.Event(True); b = torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n * 1e3
tok = 16384; C = 1152
us = t(lambda: ctx.st_block_forward(shape, W, X, Y))
print(f"block: {us:.1f} us  -> {tok/us*1e6/1e6:.2f} M tok/s; roofline 462 us -> frac {462/us:.3f}")
WP = dict(W); WP["prepared"] = ctx.prepare_block(shape, W)
us = t(lambda: ctx.st_block_forward(shape, WP, X, Y))
print(f"block prepared: {us:.1f} us  -> {tok/us*1e6/1e6:.2f} M tok/s; roofline 462 us -> frac {462/us:.3f}")
H = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda"); QKV = torch.empty(tok, 3*C, dtype=torch.bfloat16, device="cuda")
O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda"); HID = torch.empty(tok, 4*C, dtype=torch.bfloat16, device="cuda")
for name, fn, fl in [("qkv gemm", lambda: ctx.linear(X, W["w_qkv_s"], QKV), 2*tok*3*C*C),
                     ("out gemm+res", lambda: ctx.linear(O, W["w_o_s"], H, X, 1), 2*tok*C*C),
                     ("fc1 gelu", lambda: ctx.linear(X, W["w_fc1"], HID, None, 2), 2*tok*4*C*C),
                     ("fc2 res", lambda: ctx.linear(HID, W["w_fc2"], H, X, 1), 2*tok*4*C*C),
                     ("fmha spatial", lambda: ctx.attention_core(1, 16, 1024, C, 16, "S", QKV, O), 4*16*1024*1024*C),
                     ("fmha temporal", lambda: ctx.attention_core(1, 16, 1024, C, 16, "T", QKV, O), 4*1024*16*16*C),
                     ("layernorm", lambda: ctx.layer_norm(X, W["ln1_w"], W["ln1_b"], 1e-5, H), 0)]:
    u = t(fn)
    print(f"{name:14s} {u:8.1f} us  {fl/u/1e6:8.1f} TFLOP/s  ({fl/u/1e6/1674.9*100 if fl else 0:.1f}% of 1674.9)" + (f"  HBM {2*tok*C*2/u/1e3:.0f} GB/s" if not fl else ""))
