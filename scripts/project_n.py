"""Per-rank compute of the ST block at the N = 1, 2, 4, 8 shard shapes, measured on ONE GPU.

The DSP block on rank r runs exactly: LN1 + spatial attention on [B, T/N, S, C], LN2 +
temporal attention on [B, T, S/N, C], LN3 + MLP on B*T*S/N tokens, plus two switches.
This script times the compute part through the public C-ABI stage calls at those
shapes (world = 1 contexts) and adds the switch cost as bytes / (NVLink bandwidth) for
an estimate of the N-GPU block time.  It is a projection, not a multi-GPU measurement.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_10266_b200 as dsp
import synth

NVLINK_GBS = float(os.environ.get("NVLINK_GBS", "770"))  # measured peer copy per direction (B200_PROFILING.md)
try:
    PEAK_TFLOPS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    PEAK_TFLOPS = 1590.0  # B200_PROFILING.md fallback


def main():
    sh = synth.CONFIGS["blk"]
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).cuda()
    W = {k: to(v) for k, v in synth.make_block_weights(sh, 7).items()}
    B, T, S, C, NH = sh.B, sh.T, sh.S, sh.C, sh.NH
    ctx = dsp.Context()
    ctx.ensure_workspace(dsp.workspace_bytes(dsp.make_shape(B, T, S, C, NH, "bf16"), 1))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for N in (1, 2, 4, 8):
        tok = B * T * S // N
        X = torch.randn(tok, C, device="cuda").to(torch.bfloat16)
        H = torch.empty_like(X)
        Y = torch.empty_like(X)
        HID = torch.empty(tok, 4 * C, dtype=torch.bfloat16, device="cuda")
        shp_s = dsp.make_shape(B, T // N, S, C, NH, "bf16")   # spatial stage: whole frames, T/N of them
        shp_t = dsp.make_shape(B, T, S // N, C, NH, "bf16")   # temporal stage: whole columns, S/N of them

        QKV = torch.empty(tok, 3 * C, dtype=torch.bfloat16, device="cuda")
        O = torch.empty_like(X)
        stages = [
            ("LN1", lambda: ctx.layer_norm(X, W["ln1_w"], W["ln1_b"], 1e-5, H)),
            ("QKV_S", lambda: ctx.linear(H, W["w_qkv_s"], QKV)),
            ("ATTN_S", lambda: ctx.attention_core(B, T // N, S, C, NH, "S", QKV, O)),
            ("PROJ_S", lambda: ctx.linear(O, W["w_o_s"], Y, X, dsp.DSP_EPI_RESIDUAL)),
            ("LN2", lambda: ctx.layer_norm(Y, W["ln2_w"], W["ln2_b"], 1e-5, H)),
            ("QKV_T", lambda: ctx.linear(H, W["w_qkv_t"], QKV)),
            ("ATTN_T", lambda: ctx.attention_core(B, T, S // N, C, NH, "T", QKV, O)),
            ("PROJ_T", lambda: ctx.linear(O, W["w_o_t"], Y, Y, dsp.DSP_EPI_RESIDUAL)),
            ("LN3", lambda: ctx.layer_norm(Y, W["ln3_w"], W["ln3_b"], 1e-5, H)),
            ("FC1", lambda: ctx.linear(H, W["w_fc1"], HID, None, dsp.DSP_EPI_GELU)),
            ("FC2", lambda: ctx.linear(HID, W["w_fc2"], Y, Y, dsp.DSP_EPI_RESIDUAL)),
        ]

        def step():
            for _, f in stages:
                f()

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        # CUDA graphs: replay removes host launch overhead (what the block run gets from capture)
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_):
            with torch.cuda.graph(g, stream=s_):
                step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        comp = float(np.median(ts))
        per = {}
        for name, f in stages:  # each stage alone, graph of 20 launches (L2-warm), for the breakdown
            gs = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s_):
                with torch.cuda.graph(gs, stream=s_):
                    for _ in range(20):
                        f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            gs.replay()
            b.record()
            torch.cuda.synchronize()
            per[name] = round(a.elapsed_time(b) * 1e3 / 20, 1)
        sw_bytes = 2 * (N - 1) * sh.M // (N * N) * 2
        sw_us = sw_bytes / (NVLINK_GBS * 1e3)
        flops = (32 * B * T * S * C * C + 4 * B * T * S * S * C + 4 * B * S * T * T * C) / N
        roof = max(flops / PEAK_TFLOPS / 1e12 * 1e6, sw_bytes / 900e3)
        est = comp + sw_us
        res[N] = {"compute_us": round(comp, 1), "switch_us_at_%dGBps" % NVLINK_GBS: round(sw_us, 1),
                  "block_us_est": round(est, 1), "tokens_per_s_est": round(B * T * S / est * 1e6),
                  "roofline_us": round(roof, 1), "frac_est": round(roof / est, 3), "stages_us": per}
        print(N, json.dumps(res[N]), flush=True)


if __name__ == "__main__":
    main()
