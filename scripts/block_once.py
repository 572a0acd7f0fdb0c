"""Run the blk N=1 block forward a few times (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp, synth
sh = synth.CONFIGS["blk"]
to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
X = to(synth.make_x(sh, 7)); W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
ctx = dsp.Context(); shape = dsp.make_shape(1, 16, 1024, 1152, 16, "bf16")
ctx.ensure_workspace(dsp.workspace_bytes(shape, 1)); Y = torch.empty_like(X)
if len(sys.argv) > 2 and sys.argv[2] == "prep":
    W["prepared"] = ctx.prepare_block(shape, W)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    ctx.st_block_forward(shape, W, X, Y)
torch.cuda.synchronize()
