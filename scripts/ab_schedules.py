"""DSP vs DeepSpeed-Ulysses on the SAME kernels over N virtual ranks on one B200.

All N ranks share one GPU (N contexts on N streams, peer buffers local), so the time is the whole
group's GPU work: the compute is identical between the schedules, and the difference is the data
movement of the exchanges (DSP: 2 switches per block; Ulysses: 8 all-to-alls) as HBM copy work
plus barriers -- not NVLink time (that needs an 8-GPU box).  Each rank's block is captured in its
own CUDA graph; the N graphs are replayed concurrently.  Prints one JSON line per (N, schedule).

    python scripts/ab_schedules.py [--shape blk|small] [--iters 20]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2403_10266_b200 as dsp
import synth
from tests.gpu_util import to_dev, weights_dev

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="blk")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--prepared", action="store_true")
args = ap.parse_args()
sh = synth.CONFIGS["blk"] if args.shape == "blk" else synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
xs = synth.make_x(sh, 7)
Ws = synth.make_block_weights(sh, 7)
W = weights_dev(Ws, "bf16")
if args.prepared:
    c0 = dsp.Context()
    W["prepared"] = c0.prepare_block(shape, W)
    torch.cuda.synchronize()


def run(N, schedule, impl):
    ws = max(dsp.workspace_bytes(shape, N), dsp.ulysses_workspace_bytes(shape, N))
    ws = (ws + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    region = [torch.zeros(ws + act, dtype=torch.uint8, device="cuda") for _ in range(N)]
    sig = [torch.zeros(dsp.SIGNAL_PAD_BYTES // 8, dtype=torch.int64, device="cuda") for _ in range(N)]
    ctx = [dsp.Context(rank=r, world=N) for r in range(N)]
    for c, r in zip(ctx, range(N)):
        c.set_peer_buffers([t.data_ptr() for t in region], [t.data_ptr() for t in sig], ws + act)
        c.set_workspace(region[r][:ws])
        if impl == "nccl":
            c.set_collective_emulation(True)
    Tn = sh.T // N
    xsh = [np.ascontiguousarray(xs[:, r * Tn:(r + 1) * Tn]) for r in range(N)]  # rank r's T-chunk
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [region[r][ws:ws + act].view(torch.bfloat16) for r in range(N)]
    streams = [torch.cuda.Stream() for _ in range(N)]
    bw = dsp.Context.block_weights(W)
    fn = (lambda r: ctx[r].st_block_forward_ulysses(shape, bw, X[r], Y[r], impl=impl)) if schedule == "ulysses" \
        else (lambda r: ctx[r].st_block_forward(shape, bw, X[r], Y[r], impl=impl))
    graphs = [torch.cuda.CUDAGraph() for _ in range(N)]
    for r in range(N):
        with torch.cuda.graph(graphs[r], stream=streams[r]):
            fn(r)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()

    def step():
        for s in streams:
            s.wait_stream(cur)
        for r in range(N):
            with torch.cuda.stream(streams[r]):
                graphs[r].replay()
        for s in streams:
            cur.wait_stream(s)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(args.iters):
        step()
    b.record()
    torch.cuda.synchronize()
    for c in ctx:
        c.check_errors()
    us = a.elapsed_time(b) / args.iters * 1e3
    sent, _ = dsp.switch_volume(shape, N)
    n_a2a = 8 if schedule == "ulysses" else 2
    return {"N": N, "schedule": schedule, "impl": impl, "group_us": round(us, 1),
            "per_rank_bytes_sent_per_block": sent * n_a2a,
            "a2a_per_block": n_a2a, "shape": args.shape, "prepared": args.prepared}


for N in (2, 4, 8):
    for schedule, impl in (("dsp", "p2p"), ("dsp", "fused"), ("dsp", "nccl"), ("ulysses", "p2p"), ("ulysses", "nccl")):
        print(json.dumps(run(N, schedule, impl)), flush=True)
