"""The NCCL transport's pack / unpack copy kernels at the switch's shard sizes (for ncu captures):
T->S pack and S->T unpack of configs[1] at N = 2 and 8 and of configs[3] at N = 8 (B = 1), rank 0."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
import synth
for cfg, N in (("blk", 2), ("blk", 8), ("long", 8)):
    sh = synth.CONFIGS[cfg]
    ctx = dsp.Context(rank=0, world=N)
    shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    tok = sh.B * sh.T * sh.S // N
    X = torch.zeros(tok, sh.C, dtype=torch.bfloat16, device="cuda")
    Y = torch.empty_like(X)
    ctx.switch_pack(shape, "T", "S", X, Y)
    ctx.switch_unpack(shape, "S", "T", X, Y)
    torch.cuda.synchronize()
    print(cfg, N, "shard MB", tok * sh.C * 2 / 1e6)
