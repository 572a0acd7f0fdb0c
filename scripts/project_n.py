"""Per-rank time of the DSP ST block at the N = 2, 4, 8 shard shapes, measured on ONE GPU.

Rank r of an N-GPU DSP block runs exactly
  * LN1 + the spatial stage on its T-shard [B, T/N, S, C]            (LN1, QKV_S, ATTN_S, PROJ_S),
  * switch T->S,
  * the temporal stage + MLP on its S-shard [B, T, S/N, C]           (QKV_T, ATTN_T, PROJ_T, FC1, FC2),
  * switch S->T,
and at N > 1 one extra pass over its rows (LN2 partials recomputed after the switch, R30).
The kernels of each stage are the kernels of the N = 1 block at the matching global shape:
the spatial stages of block([B, T/N, S, C]) and the temporal + MLP stages of block([B, T, S/N, C])
are the rank's stages bit for bit (same launches, same M, same sequence counts).  This script
times both N = 1 blocks (prepared weights, CUDA-graph replay, L2 flushed, device stage clocks)
and adds:
  * the LN2 partials pass, taken as the LN1 statistics pass of block([B, T/N, S, C]) (the same
    kernel family reading the same tok_r x C bf16 rows);
  * the switch copy kernels (pack of T->S at B*Tn > 1, unpack of S->T at B > 1 are identities at
    B = 1: one copy kernel per switch), timed through dsp_switch_pack / dsp_switch_unpack;
  * the NVLink time of both switches: (N-1)/N^2 * M * 2 B per switch per rank / NVLINK_GBS
    (not measurable on the 1-GPU pool).
It is a projection from measured kernel times, not a multi-GPU measurement.
Output: one JSON object per N (stdout), and a summary table (stderr).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2403_10266_b200 as dsp
import synth

NVLINK_GBS = float(os.environ.get("NVLINK_GBS", "770"))  # peer copy per direction, B200_PROFILING.md
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 1590.0) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0
SPATIAL = ("LN1", "QKV_S", "ATTN_S", "PROJ_S")
TEMPORAL = ("QKV_T", "ATTN_T", "PROJ_T", "FC1", "FC2")
STEPS = int(os.environ.get("STEPS", "20"))


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()


def block_stages(B, T, S, C, NH, W, flush):
    """Stage spans (us) and the event time per step of the N = 1 prepared block at [B, T, S, C]."""
    ctx = dsp.Context()
    shape = dsp.make_shape(B, T, S, C, NH, "bf16")
    ctx.ensure_workspace(dsp.workspace_bytes(shape, 1))
    Wd = dict(W)
    Wd["prepared"] = ctx.prepare_block(shape, W)
    bw = ctx.block_weights(Wd)
    sh = synth.BlockShape(B, T, S, C, NH, "bf16")
    X = to_dev(synth.make_x(sh, 7))
    Y = torch.empty_like(X)
    for _ in range(3):
        ctx.st_block_forward(shape, bw, X, Y)
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        ctx.st_block_forward(shape, bw, X, Y)
    torch.cuda.synchronize()
    NS = len(dsp.STAGES)
    clk = torch.zeros(NS, 2, dtype=torch.int64, device="cuda")
    reset = torch.zeros_like(clk)
    reset[:, 0] = -1
    ctx.set_stage_clocks(clk)
    # re-capture with the clocks on (the clock pointer is baked into the launches)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        ctx.st_block_forward(shape, bw, X, Y)
    torch.cuda.synchronize()
    hist = torch.zeros(STEPS, NS, 2, dtype=torch.int64, device="cuda")
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(STEPS)]
    for i in range(STEPS):
        flush.zero_()
        clk.copy_(reset)
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
        hist[i].copy_(clk)
    torch.cuda.synchronize()
    ctx.set_stage_clocks(None)
    ch = hist.cpu().numpy().astype(np.uint64)
    spans = {}
    for i, n in enumerate(dsp.STAGES):
        ok = (ch[:, i, 0] != np.uint64(0xFFFFFFFFFFFFFFFF)) & (ch[:, i, 1] > ch[:, i, 0])
        spans[n] = float(np.mean((ch[ok, i, 1] - ch[ok, i, 0]).astype(np.float64))) / 1e3 if ok.any() else 0.0
    t_us = sum(a.elapsed_time(b) for a, b in ev) / STEPS * 1e3
    return spans, t_us


def switch_copy_us(B, T, S, C, NH, N, flush):
    """One NCCL-transport copy kernel per switch at B = 1 (dsp_switch_pack of T->S, unpack of
    S->T): timed through the exported building blocks on a world-N shape (rank 0)."""
    ctx = dsp.Context(rank=0, world=N)
    shape = dsp.make_shape(B, T, S, C, NH, "bf16")
    tok = B * T * S // N
    X = torch.zeros(tok, C, dtype=torch.bfloat16, device="cuda")
    Y = torch.empty_like(X)
    out = {}
    for name, fn in (("pack_T2S", lambda st=None: ctx.switch_pack(shape, "T", "S", X, Y, st)),
                     ("unpack_S2T", lambda st=None: ctx.switch_unpack(shape, "S", "T", X, Y, st))):
        try:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            # 10 back-to-back launches in one graph (as inside the block: no host launch gaps)
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
                for _ in range(10):
                    fn(cap)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            acc = 0.0
            for _ in range(STEPS):
                flush.zero_()
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                acc += a.elapsed_time(b)
            out[name] = acc / STEPS / 10 * 1e3
        except Exception as e:  # noqa: BLE001
            out[name] = None
            out[name + "_error"] = str(e)[:160]
    return out


def main():
    cfg = os.environ.get("CONFIG", "blk")
    sh = synth.CONFIGS[cfg]
    B, T, S, C, NH = sh.B, sh.T, sh.S, sh.C, sh.NH
    W = {k: to_dev(v) for k, v in synth.make_block_weights(sh, 7).items()}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    M = B * T * S * C
    flops = 32 * B * T * S * C * C + 4 * B * T * S * S * C + 4 * B * S * T * T * C
    rows = []
    for N in (1, 2, 4, 8):
        sp, t_sp = block_stages(B, T // N, S, C, NH, W, flush)
        te, t_te = (sp, t_sp) if N == 1 else block_stages(B, T, S // N, C, NH, W, flush)
        stages = {n: round(sp[n], 2) for n in SPATIAL}
        stages.update({n: round(te[n], 2) for n in TEMPORAL})
        compute = sum(stages.values())
        extra = {}
        if N > 1:
            extra["LN2_partials (= LN1 stats pass at tok_r)"] = round(sp["LN1"], 2)
            sw = switch_copy_us(B, T, S, C, NH, N, flush)
            extra.update({k: (round(v, 2) if isinstance(v, float) else v) for k, v in sw.items()})
        copies = sum(v for v in extra.values() if isinstance(v, float))
        nvl_bytes = 2 * (N - 1) * M * 2 // (N * N)
        nvl_us = nvl_bytes / (NVLINK_GBS * 1e3)
        t_rank = compute + copies + nvl_us
        roof = max(flops / N / (PEAK * 1e6), nvl_bytes / 900e3)
        row = {"config": cfg, "N": N, "stage_us": stages, "compute_us": round(compute, 1),
               "n_gt_1_kernels_us": extra, "nvlink_bytes_per_rank": nvl_bytes,
               "nvlink_us_at_%dGBps" % NVLINK_GBS: round(nvl_us, 2),
               "projected_block_us": round(t_rank, 1),
               "block_event_us": {"spatial_shape": round(t_sp, 1), "temporal_shape": round(t_te, 1)},
               "roofline_us": round(roof, 1), "projected_frac": round(roof / t_rank, 3),
               "projected_tokens_per_s": round(B * T * S / (t_rank * 1e-6)),
               "gate_60pct_us": round(roof / 0.6, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    for r in rows:
        sys.stderr.write(f"N={r['N']}: compute {r['compute_us']:7.1f} us + N>1 kernels + NVLink -> "
                         f"{r['projected_block_us']:7.1f} us (roofline {r['roofline_us']:.1f}, frac "
                         f"{r['projected_frac']:.3f}, 60% gate {r['gate_60pct_us']:.1f})\n")


if __name__ == "__main__":
    main()
