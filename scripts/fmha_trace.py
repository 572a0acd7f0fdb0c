"""Per-phase clock64 trace of the spatial FMHA pair kernel (CTA 0, first thread of each softmax
slot).  Needs the DSP_FMHA_TRACE build:  python scripts/variant.py trace -DDSP_FMHA_TRACE, then
DSP_LIB_OVERRIDE=paper_2403_10266_b200/libdsp_trace.so python scripts/fmha_trace.py"""
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
buf = np.zeros(2 * 64 * 16, dtype=np.uint64)
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaMemcpy(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(ptr), ctypes.c_size_t(buf.nbytes), 2)
t = buf.reshape(2, 64, 16).astype(np.int64)
base = t[t > 0].min()
# stamps: 0 wait S, 3 S ready, 8 S in regs, 9 max done, 10 pp go, 11 exps done, 1 after l, 2 o_done, 12 P stored, 4 arrive
if os.environ.get("PT"):  # fmha_pt_kernel: 0 wait S, 3 S ready, 8 S in regs, 9 max, 11 exps + P st issued, 12 st done, 4 arrive
    order = [0, 3, 8, 9, 11, 12, 4]
    names = ["waitS", "Srdy", "ldtm", "max", "exps", "stw", "done"]
else:
    order = [0, 3, 8, 9, 10, 11, 2, 12, 4]
    names = ["waitS", "Srdy", "ldtm", "max", "ppgo", "exps", "odone", "Pst", "done"]
print("slot tile  " + " ".join(f"{n:>7s}" for n in names) + "   deltas")
for s in range(2):
    for k in range(0, 40):
        r = t[s, k]
        if r[0] == 0:
            continue
        vals = [int(r[i] - base) if r[i] else -1 for i in order]
        d = [vals[i + 1] - vals[i] if vals[i + 1] >= 0 and vals[i] >= 0 else -1 for i in range(len(vals) - 1)]
        extra = f"  | epi odone {int(r[6]-r[5])} store {int(r[7]-r[6])}" if r[5] else ""
        print(f"{s} {k:3d}  " + " ".join(f"{v:7d}" for v in vals) + "   " + " ".join(f"{x:5d}" for x in d) + extra)
