"""Per-item clock64 trace of the temporal FMHA (CTA 0).  DSP_FMHA_TRACE build."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp
L = dsp.lib(); L.dsp_debug_fmha_trace.restype = ctypes.c_void_p
tok, C = 16384, 1152
QKV = (torch.randn(tok, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
ctx = dsp.Context()
for _ in range(3):
    ctx.attention_core(1, 16, 1024, C, 16, "T", QKV, O)
torch.cuda.synchronize()
buf = np.zeros(2 * 64 * 16, dtype=np.uint64)
ctypes.CDLL("libcudart.so.12").cudaMemcpy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(L.dsp_debug_fmha_trace()), ctypes.c_size_t(buf.nbytes), 2)
t = buf.reshape(128, 16).astype(np.int64)
base = t[t > 0].min()
print("item | start  S_ready  P_done  O_ready  stored")
for k in range(10):
    r = t[k]
    if r[0]:
        v = [int(x - base) for x in r[:5]]
        print(k, *v, "  deltas", *[v[i + 1] - v[i] for i in range(4)])
