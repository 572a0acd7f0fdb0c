"""Diagnose the layer-13 elements of the 28-layer prepared+cross model that exceed the R22 gate:
GPU chained (model_forward prefix), GPU single prepared block, GPU raw block, oracle stages."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp
import synth
from oracle import block as ob
from tests.gpu_util import to_dev, to_f64, weights_dev, weights_f64
sh = synth.CONFIGS["blk"]; Lc = 120; L = int(sys.argv[1]) if len(sys.argv) > 1 else 13
ctx = dsp.Context(); shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
ctx.ensure_workspace(dsp.workspace_bytes(shape, 1))
ctxt_np = synth.make_context(sh, 7, Lc); ctxt = to_dev(ctxt_np, "bf16").view(sh.B, Lc, sh.C)
layers, host = [], {}
for l in range(L + 1):
    Ws = synth.make_block_weights(sh, 7, layer=l); Ws.update(synth.make_cross_weights(sh, 7, layer=l))
    W = weights_dev(Ws, "bf16"); W["ctx_tokens"] = ctxt; W["prepared"] = ctx.prepare_block(shape, W)
    layers.append(W); host[l] = Ws
X = to_dev(synth.make_x(sh, 7), "bf16")
def prefix(n):
    Y = torch.empty_like(X); ctx.st_model_forward(shape, layers[:n], X, Y); torch.cuda.synchronize(); return Y
xin_t = prefix(L); xout_t = prefix(L + 1)
single = torch.empty_like(X); ctx.st_block_forward(shape, layers[L], xin_t, single)
Wraw = {k: v for k, v in layers[L].items() if k != "prepared"}
raw = torch.empty_like(X); ctx.st_block_forward(shape, Wraw, xin_t, raw); torch.cuda.synchronize()
cols = np.array([0, 5, 511, 1023])
xin = to_f64(xin_t); Wf = weights_f64(host[L], "bf16")
Wc = dict(ln_w=Wf["ln_c_w"], ln_b=Wf["ln_c_b"], w_q=Wf["w_q_c"], w_kv=Wf["w_kv_c"], w_o=Wf["w_o_c"])
y1 = ob.spatial_stage(xin, Wf, sh.NH)[:, :, cols]; y2 = ob.temporal_stage(y1, Wf, sh.NH)
y2c = ob.cross_stage(y2, synth.to_f64(ctxt_np, "bf16"), Wc, sh.NH); y = ob.mlp_stage(y2c, Wf)
print("input |x| max", np.abs(xin).max(), "mean |x|", np.abs(xin).mean(), "row std mean", xin.std(-1).mean(), "row mean max", np.abs(xin.mean(-1)).max())
for name, t in [("chained", xout_t), ("single-prep", single), ("raw", raw)]:
    g = to_f64(t)[:, :, cols]; err = np.abs(g - y)
    bad = err > 2e-2 + 1e-2 * np.abs(y)
    print(f"{name:12s} max-abs {err.max():.4f} rel-L2 {np.linalg.norm(g-y)/np.linalg.norm(y):.2e} violations {int(bad.sum())}")
g = to_f64(xout_t)[:, :, cols]; err = np.abs(g - y)
idx = np.argsort(err.ravel())[-6:]
for i in idx:
    b, t, s, c = np.unravel_index(i, y.shape)
    print(f"t={t} col={cols[s]} c={c}: gpu {g[b,t,s,c]:.4f} oracle {y[b,t,s,c]:.4f} | x {xin[b,t,cols[s],c]:.3f} y1 {y1[b,t,s,c]:.3f} y2 {y2[b,t,s,c]:.3f} y2c {y2c[b,t,s,c]:.3f} | single {to_f64(single)[b,t,cols[s],c]:.4f} raw {to_f64(raw)[b,t,cols[s],c]:.4f}")
