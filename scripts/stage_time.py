"""Scratch: per-stage times of the prepared blk N=1 block (one stage's events per pass, as in
bench.py) plus the whole block under graph replay.  Honours DSP_LIB_OVERRIDE for A/B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2403_10266_b200 as dsp, synth
sh = synth.CONFIGS["blk"]
to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
X = to(synth.make_x(sh, 7)); W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
ctx = dsp.Context(); shape = dsp.make_shape(1, 16, 1024, 1152, 16, "bf16")
ctx.ensure_workspace(dsp.workspace_bytes(shape, 1)); Y = torch.empty_like(X)
W["prepared"] = ctx.prepare_block(shape, W)
bw = ctx.block_weights(W)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
step = lambda: ctx.st_block_forward(shape, bw, X, Y)
for _ in range(5): step()
g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s): step()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(30)]
for a, b in ev:
    flush.zero_(); a.record(); g.replay(); b.record()
torch.cuda.synchronize()
blk = np.median([a.elapsed_time(b) for a, b in ev]) * 1e3
out = []
for i, name in enumerate(dsp.STAGES):
    e = [None] * (2 * len(dsp.STAGES)); e[2 * i], e[2 * i + 1] = torch.cuda.Event(True), torch.cuda.Event(True)
    ctx.set_stage_events(e)
    ts = []
    for _ in range(10):
        flush.zero_(); step(); torch.cuda.synchronize(); ts.append(e[2 * i].elapsed_time(e[2 * i + 1]) * 1e3)
    out.append(f"{name}={np.median(ts):.1f}")
ctx.set_stage_events(None)
print(f"{os.environ.get('DSP_LIB_OVERRIDE', 'libdsp.so')[-22:]:22s} block {blk:.1f} us | " + " ".join(out))
# the same, with each stage's events captured into its own graph (external event nodes)
out2 = []
for i, name in enumerate(dsp.STAGES):
    e = [None] * (2 * len(dsp.STAGES)); e[2 * i], e[2 * i + 1] = torch.cuda.Event(True), torch.cuda.Event(True)
    ctx.set_stage_events(e)
    gi = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(gi, stream=s): step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_(); gi.replay(); torch.cuda.synchronize(); ts.append(e[2 * i].elapsed_time(e[2 * i + 1]) * 1e3)
    out2.append(f"{name}={np.median(ts):.1f}")
ctx.set_stage_events(None)
print(f"{'graph-captured events':22s}             | " + " ".join(out2))
