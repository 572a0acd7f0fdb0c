"""Run each hot kernel of the blk N=1 block a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp, synth
which = sys.argv[1] if len(sys.argv) > 1 else "all"
sh = synth.CONFIGS["blk"]
to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
X = to(synth.make_x(sh, 7)); W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
ctx = dsp.Context(); tok, C = 16384, 1152
H = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda"); QKV = torch.empty(tok, 3*C, dtype=torch.bfloat16, device="cuda")
O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda"); HID = torch.empty(tok, 4*C, dtype=torch.bfloat16, device="cuda")
ctx.linear(X, W["w_qkv_s"], QKV)
for _ in range(3):
    if which in ("all", "fmha"):
        ctx.attention_core(1, 16, 1024, C, 16, "S", QKV, O)
        ctx.attention_core(1, 16, 1024, C, 16, "T", QKV, O)
    if which in ("all", "gemm"):
        ctx.linear(O, W["w_o_s"], H, X, 1)
        ctx.linear(HID, W["w_fc2"], H, X, 1)
    if which in ("all", "ln"):
        ctx.layer_norm(X, W["ln1_w"], W["ln1_b"], 1e-5, H)
torch.cuda.synchronize()
print("ok")
