"""Run the long-video block (configs[3], T=128, S=4096) forward twice with prepared weights
(for ncu captures of the TSEQ temporal QKV GEMM and the single-tile temporal FMHA)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp, synth
sh = synth.CONFIGS["long"]
to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
X = to(synth.make_x(sh, 7)); W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
ctx = dsp.Context(); shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
ctx.ensure_workspace(dsp.workspace_bytes(shape, 1)); Y = torch.empty_like(X)
W["prepared"] = ctx.prepare_block(shape, W)
for _ in range(2):
    ctx.st_block_forward(shape, W, X, Y)
torch.cuda.synchronize()
print("ok")
