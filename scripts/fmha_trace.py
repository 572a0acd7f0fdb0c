"""Per-phase clock64 trace of the spatial FMHA (CTA 0, warp 0 of each softmax slot).
Needs the DSP_FMHA_TRACE build (libdsp_trace.so via DSP_LIB_OVERRIDE)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp
L = dsp.lib()
L.dsp_debug_fmha_trace.restype = ctypes.c_void_p
tok, C = 16384, 1152
QKV = (torch.randn(tok, 3 * C, device="cuda") * 0.5).to(torch.bfloat16)
O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
ctx = dsp.Context()
for _ in range(3):
    ctx.attention_core(1, 16, 1024, C, 16, "S", QKV, O)
torch.cuda.synchronize()
ptr = L.dsp_debug_fmha_trace()
buf = np.zeros(2 * 64 * 8, dtype=np.uint64)
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaMemcpy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ptr), ctypes.c_size_t(buf.nbytes), 2)
t = buf.reshape(2, 64, 8).astype(np.int64)
base = t[t > 0].min()
print("slot tile | wait_S_start  S_ready  exp_done  odone  tile_done   (cycles rel. to first stamp)")
for s in range(2):
    for k in range(0, 56):
        r = t[s, k]
        if r[0] == 0:
            continue
        rel = [int(x - base) if x else -1 for x in r[:5]]
        extra = ""
        if r[5]:
            extra = f"  | epi: start {int(r[5]-base)} odone {int(r[6]-base)} stored {int(r[7]-base)}"
        print(s, k, rel[0], rel[3], rel[1], rel[2], rel[4], " wait", rel[3] - rel[0], " soft", rel[4] - rel[3], extra)
