"""The block's GEMM launches at blk N=1 (QKV, out-proj+res, FC1+GELU, FC2+res), a few times each (ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2403_10266_b200 as dsp
tok, C = 16384, 1152
r = lambda *s: (torch.randn(*s, device="cuda") * 0.05).to(torch.bfloat16)
X, Wqkv, Wo, W1, W2 = r(tok, C), r(3 * C, C), r(C, C), r(4 * C, C), r(C, 4 * C)
QKV, O, H, HID = r(tok, 3 * C), r(tok, C), r(tok, C), r(tok, 4 * C)
ctx = dsp.Context()
for _ in range(2):
    ctx.linear(X, Wqkv, QKV)
    ctx.linear(O, Wo, H, X, 1)
    ctx.linear(X, W1, HID, None, 2)
    ctx.linear(HID, W2, H, X, 1)
torch.cuda.synchronize()
print("ok")
