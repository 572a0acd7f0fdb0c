"""Per-step clock64 trace of the attention backward (CTA 0; spatial L = 1024 by default).  Needs the
trace build:  python scripts/variant.py btrace -DDSP_FMHA_TRACE -DDSP_FMHA_BWD_TRACE, then
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_btrace.so python scripts/fmha_bwd_trace.py [S|T]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp
L = dsp.lib()
L.dsp_debug_fmha_trace.restype = ctypes.c_void_p
dim = sys.argv[1] if len(sys.argv) > 1 else "S"
B, Tl, Sl, C, NH = (1, 16, 1024, 1152, 16) if dim == "S" else (1, 16, 1024, 1152, 16)
tok = B * Tl * Sl
qkv = (torch.randn(tok, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
dout = (torch.randn(tok, C, device="cuda") * 0.5).to(torch.bfloat16)
o = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
lse = torch.empty(tok, NH, dtype=torch.float32, device="cuda")
dqkv = torch.empty(tok, 3 * C, dtype=torch.bfloat16, device="cuda")
ctx = dsp.Context()
ctx.attention_core_lse(B, Tl, Sl, C, NH, dim, qkv, o, lse)
for _ in range(3):
    ctx.attention_core_bwd(B, Tl, Sl, C, NH, dim, qkv, o, dout, lse, dqkv)
torch.cuda.synchronize()
ptr = L.dsp_debug_fmha_trace()
buf = np.zeros(64 * 8, dtype=np.uint64)
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaMemcpy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ptr), ctypes.c_size_t(buf.nbytes), 2)
t = buf.reshape(64, 8).astype(np.int64)
base = t[t > 0].min()
names = ["c.start", "c.Srdy", "c.Pdone", "m.qfull", "m.pfull", "m.Bgo", "w1.Srdy", "w1.Pdone"]
print("step " + " ".join(f"{n:>8s}" for n in names) + "   softmax  S->Bgo  Bgo->dq  dq->red  step")
prev = None
for g in range(40):
    r = t[g]
    if r[0] == 0:
        continue
    v = [int(x - base) if x else -1 for x in r]
    sm = v[2] - v[1]
    s2b = v[5] - v[2]
    b2d = v[6] - v[5]
    d2r = v[7] - v[6] if v[7] >= 0 else -1
    step = v[1] - prev if prev is not None else 0
    prev = v[1]
    print(f"{g:4d} " + " ".join(f"{x:8d}" for x in v) + f"   {sm:7d} {s2b:7d} {b2d:8d} {d2r:8d} {step:6d}")
