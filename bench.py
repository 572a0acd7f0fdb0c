"""bench.py — ST-block forward tokens/s of the DSP hot path on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dsp|reference]
                    [--config blk|long|tiny] [--switch nccl|p2p]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step = one dsp_st_block_forward (LN1, spatial QKV GEMM,
spatial FMHA, out-proj+residual, switch T->S, LN2, temporal QKV / FMHA / out-proj,
LN3, FC1+GELU, FC2+residual, switch S->T) over one synthetic [B,T,S,C] activation
already resident in HBM.  The global config is fixed as N grows (strong scaling, as in
the paper's experiment P:153: "keep the batch size to 1 and sequence length constant").
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (oracle/) on a
bounded sample of the same workload instead (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

CONFIGS = {
    "blk": (synth.CONFIGS["blk"], "configs[1] single ST block: B=1 T=16 S=1024 (32x32) C=1152 16 heads bf16"),
    "long": (synth.CONFIGS["long"], "configs[3] long-video stress: B=1 T=128 S=4096 C=1152 16 heads bf16"),
    "tiny": (synth.CONFIGS["tiny"], "configs[0] tiny ST block: B=1 T=4 S=16 C=64 4 heads fp32"),
}
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ CPU oracle
def oracle_sample(sh, seed, frames, cols, mlp_tokens):
    """Time the float64 oracle on a bounded, stage-sampled slice of the block.

    Each stage of the block touches every token once, so the per-token cost of the
    block is the sum of the per-token costs of its stages: spatial stage (LN1 + MHA_S +
    residual) on `frames` whole frames, temporal stage (LN2 + MHA_T + residual) on
    `cols` whole columns, MLP stage on `mlp_tokens` tokens.  Slice independence
    makes each sample a faithful piece of the full computation.
    """
    from oracle import block as ob
    x = synth.to_f64(synth.make_x(sh, seed, t_range=(0, frames)), sh.dtype)
    W = {k: synth.to_f64(v, sh.dtype) for k, v in synth.make_block_weights(sh, seed).items()}
    t0 = time.perf_counter()
    ob.spatial_stage(x, W, sh.NH)
    t1 = time.perf_counter()
    xc = synth.to_f64(synth.make_x(sh, seed, s_range=(0, cols)), sh.dtype)
    ob.temporal_stage(xc, W, sh.NH)
    t2 = time.perf_counter()
    flat = xc.reshape(-1, sh.C)[:mlp_tokens]
    ob.mlp_stage(flat, W)
    t3 = time.perf_counter()
    per_tok = (t1 - t0) / (sh.B * frames * sh.S) + (t2 - t1) / (sh.B * cols * sh.T) + (t3 - t2) / flat.shape[0]
    return 1.0 / per_tok, t3 - t0


def oracle_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_sizes(sh, budget="baseline"):
    if budget == "baseline":   # ~10-30 s of float64 numpy on 8 cores
        return min(4, sh.T), min(256, sh.S), min(4096, sh.B * sh.T * sh.S)
    return 1, min(64, sh.S), min(1024, sh.B * sh.T * sh.S)  # ~1-2 s per reference step


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sh, desc = CONFIGS[args.config]
    frames, cols, toks = sample_sizes(sh, "step")
    for _ in range(args.warmup):
        oracle_sample(sh, args.seed, frames, cols, toks)
    t0 = time.perf_counter()
    rates = [oracle_sample(sh, args.seed, frames, cols, toks)[0] for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    layers = getattr(args, "layers", 1)
    v = float(np.mean(rates)) / layers
    sample = (f"per step: oracle spatial stage on {frames} frame(s), temporal stage on {cols} columns, MLP stage on "
              f"{toks} tokens (float64 numpy, BLAS threads = cores); tokens/s = 1 / sum of per-token stage costs"
              + (f", divided by {layers} layers" if layers > 1 else ""))
    metric = "ST-block fwd tokens/s" if layers == 1 else f"{layers}-layer ST-DiT forward tokens/s"
    out = {"impl": "reference", "metric": metric, "value": v, "unit": "tokens/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": wall / max(args.steps, 1) * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": desc, "global_tokens": sh.B * sh.T * sh.S},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": oracle_threads(), "cpu_model": cpu_model(),
                            "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML polling thread (SM clock + throttle reasons) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ GPU arm
def stage_work(name, sh, N, prepared=True):
    """(algorithmic amount, unit, bound) per rank per launch of a block stage.

    Prepared weights (R30): LN1 is a row-statistics pass that only READS the activation
    (tok*C*elem); LN2 at N > 1 likewise; LN2 at N = 1 and LN3 are folded into the consuming GEMM
    epilogues (no kernel, no traffic: None).  Raw weights: each LN reads and writes the activation.
    """
    B, T, S, C = sh.B, sh.T, sh.S, sh.C
    tok = B * T * S // N
    e = sh.elem_bytes
    gem = {"QKV_S": 6, "QKV_T": 6, "PROJ_S": 2, "PROJ_T": 2, "FC1": 8, "FC2": 8}
    if name in gem:
        return gem[name] * tok * C * C, "flop", "tensor"
    if name == "ATTN_S":
        return 4 * B * (T // N) * S * S * C, "flop", "tensor"
    if name == "ATTN_T":
        return 4 * tok * C * e, "byte", "hbm"  # q, k, v read + o write, once each
    if name.startswith("LN"):
        if not prepared:
            return 2 * tok * C * e, "byte", "hbm"
        if name == "LN1" or (name == "LN2" and N > 1):
            return tok * C * e, "byte", "hbm"
        return None, "folded", ""
    if name.startswith("SWITCH"):
        return (N - 1) * B * (T // N) * (S // N) * C * e, "byte", "nvlink"
    return 0, "", ""


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def run_dsp(args):
    import torch
    import torch.distributed as dist

    import paper_2403_10266_b200 as dsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torchrun --nproc-per-node {args.gpus}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    sh, desc = CONFIGS[args.config]
    N = world
    Tn = sh.T // N
    ctx = dsp.Context(pg=pg, device=dev)
    shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    tdt = torch.bfloat16 if sh.dtype == "bf16" else torch.float32

    def to_dev(a):
        a = np.ascontiguousarray(a)
        t = torch.from_numpy(a.view(np.int16)).view(torch.bfloat16) if sh.dtype == "bf16" else torch.from_numpy(a)
        return t.to(dev)

    xs = synth.make_x(sh, args.seed, t_range=(rank * Tn, (rank + 1) * Tn))
    W = {k: to_dev(v) for k, v in synth.make_block_weights(sh, args.seed).items()}
    prep_note = "raw weights (LayerNorm kernels in the block)"
    if args.prepare and sh.dtype == "bf16":
        # one-time weight preparation (model-load time, untimed): LayerNorm gamma/beta folded
        # into the consuming GEMMs' weights (dsp_st_block_prepare, R30)
        W["prepared"] = ctx.prepare_block(shape, W)
        prep_note = "prepared weights (dsp_st_block_prepare once before timing: LN folded into the GEMMs)"
    bw = ctx.block_weights(W)
    X = to_dev(xs)
    act_bytes = X.numel() * X.element_size()
    ws_bytes = dsp.workspace_bytes(shape, N)
    if args.schedule == "ulysses":
        ws_bytes = max(ws_bytes, dsp.ulysses_workspace_bytes(shape, N))
    impl = args.switch
    if impl in ("p2p", "fused") and N > 1:
        import torch.distributed._symmetric_memory as symm
        ws_pad = (ws_bytes + 4095) // 4096 * 4096
        buf = symm.empty(ws_pad + 2 * act_bytes, dtype=torch.uint8, device=dev)
        hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
        ctx.set_peer_buffers(hdl.buffer_ptrs, hdl.signal_pad_ptrs, ws_pad + 2 * act_bytes)
        ctx.set_workspace(buf[:ws_pad])
        Y = buf[ws_pad:ws_pad + act_bytes].view(tdt)
        Y2 = buf[ws_pad + act_bytes:ws_pad + 2 * act_bytes].view(tdt)  # second staging buffer (e2e)
    else:
        ctx.ensure_workspace(ws_bytes)
        Y = torch.empty_like(X)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    ulysses = args.schedule == "ulysses" and N > 1

    def step_eager():
        if ulysses:  # the comparison system of P:99 / P:153 on the same kernels
            ctx.st_block_forward_ulysses(shape, bw, X, Y, impl=impl)
        else:
            ctx.st_block_forward(shape, bw, X, Y, impl=impl)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    # device-side stage clocks (dsp_ctx_set_stage_clocks): each kernel of the block records its span
    # (first CTA past its dependency wait -> last CTA exit, %globaltimer) with one atomic per CTA,
    # inside the timed, graph-replayed steps themselves
    NS = len(dsp.STAGES)
    clk = torch.zeros(NS, 2, dtype=torch.int64, device=dev)
    clk_reset = torch.zeros(NS, 2, dtype=torch.int64, device=dev)
    clk_reset[:, 0] = -1  # UINT64_MAX for the atomicMin
    ctx.set_stage_clocks(clk)
    # warm-up (eager), then capture one block in a CUDA graph: replay removes the host launch
    # overhead of the ~13 launches per block (the kernels and NCCL calls are the same)
    for _ in range(args.warmup):
        flush.zero_()
        step_eager()
    barrier()
    step, graph_note, per_step_launches = step_eager, "eager", None
    if args.graph:
        try:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            l0 = ctx.launch_count()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    step_eager()
            per_step_launches = ctx.launch_count() - l0
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            step, graph_note = g.replay, "cuda graph replay of one captured dsp_st_block_forward"
        except Exception as e:  # noqa: BLE001 - fall back to eager launches
            step, graph_note = step_eager, f"eager (graph capture failed: {str(e)[:120]})"
        barrier()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    l0 = ctx.launch_count()
    clk_hist = torch.zeros(K, NS, 2, dtype=torch.int64, device=dev)
    with ClockSampler(local) as clocks:
        barrier()
        for i in range(K):
            flush.zero_()                      # L2 flush between timed steps (outside the events)
            clk.copy_(clk_reset)
            ev[i][0].record()
            step()
            ev[i][1].record()
            clk_hist[i].copy_(clk)
        barrier()
    ctx.set_stage_clocks(None)
    ch = clk_hist.cpu().numpy().astype(np.uint64)
    span_us = np.zeros(NS)
    for i in range(NS):
        ok = (ch[:, i, 0] != np.uint64(0xFFFFFFFFFFFFFFFF)) & (ch[:, i, 1] > ch[:, i, 0])
        if ok.any():
            span_us[i] = float(np.mean((ch[ok, i, 1] - ch[ok, i, 0]).astype(np.float64))) / 1e3
    if world > 1:
        st_ = torch.tensor(span_us, dtype=torch.float64, device=dev)
        dist.all_reduce(st_, op=dist.ReduceOp.MAX)
        span_us = st_.cpu().numpy()
    launches = ctx.launch_count() - l0 if per_step_launches is None else per_step_launches * K
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    tokens = sh.B * sh.T * sh.S
    value = tokens * K / (t_ms / 1e3)

    # per-stage timing: the block is captured once per stage with a pair of CUDA events around
    # that stage only (event-record nodes inside the graph, on the library's launch stream), and
    # each graph is replayed KP times with L2 flushed before every replay.  Only the two stage
    # boundaries lose their programmatic-dependent-launch overlap, so a stage time is the full
    # duration of its kernel(s) from first CTA to last, launch ramp and tail included.
    KP = max(3, min(K, 10))
    prepared = args.prepare and sh.dtype == "bf16"
    stage_ms = np.zeros(len(dsp.STAGES))
    for i in range(len(dsp.STAGES)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stage_ev = [None] * (2 * len(dsp.STAGES))
        stage_ev[2 * i], stage_ev[2 * i + 1] = e0, e1
        ctx.set_stage_events(stage_ev)
        run, gi = step_eager, None
        if args.graph and step is not step_eager:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(torch.cuda.current_stream())
            gi = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap), torch.cuda.graph(gi, stream=cap):
                step_eager()
            torch.cuda.synchronize()
            run = gi.replay
        ctx.set_stage_events(None)
        barrier()
        acc = 0.0
        for _ in range(KP):
            flush.zero_()
            run()
            torch.cuda.synchronize()
            acc += e0.elapsed_time(e1)
        stage_ms[i] = acc / KP
        del gi
    if world > 1:
        st = torch.tensor(stage_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
        stage_ms = st.cpu().numpy()
    P, peak_src = peaks()
    traffic = {}
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.config, {}) if N == 1 else {}
        except Exception:
            traffic = {}
    stages = {}
    for i, name in enumerate(dsp.STAGES):
        amt, unit, bound = stage_work(name, sh, N, prepared)
        us = span_us[i] if span_us[i] > 0 else stage_ms[i] * 1e3
        if amt is None:
            stages[name] = {"us": round(us, 2), "folded": "into the consuming GEMM epilogue (R30): no kernel"}
            continue
        if amt == 0 or us <= 0.05:
            stages[name] = {"us": round(us, 2)}
            continue
        if unit == "flop":
            ach, pk, u = amt / (us * 1e-6) / 1e12, P["bf16_tflops"], "TFLOP/s"
        elif bound == "hbm":
            ach, pk, u = amt / (us * 1e-6) / 1e9, P["hbm_gbs"], "GB/s"
        else:
            ach, pk, u = amt / (us * 1e-6) / 1e9, 900.0, "GB/s"
        stages[name] = {"us": round(us, 2), "achieved": round(ach, 1), "unit": u, "frac": round(ach / pk, 3),
                        "bound": bound, "algorithmic_per_launch": amt, "algorithmic_unit": unit + "s",
                        "traffic": traffic.get(name), "timing": "device clock" if span_us[i] > 0 else "events",
                        "event_us": round(stage_ms[i] * 1e3, 2)}
    # dominant kernel = the compute stage with the largest measured time (one kernel per stage)
    KERNELS = {"QKV_S": "gemm_bf16_tc_kernel<192, LN-folded> (spatial QKV)",
               "ATTN_S": "fmha_pt_kernel (spatial FMHA, P in TMEM)",
               "PROJ_S": "gemm_bf16_tc_kernel<192, +residual +LN partials> (spatial out-proj)",
               "QKV_T": "gemm_bf16_tc_kernel<192, LN-folded> (temporal QKV)",
               "ATTN_T": "fmha_bf16_tc_kernel (temporal FMHA, block-diagonal packed)",
               "PROJ_T": "gemm_bf16_tc_kernel<192, +residual +LN partials> (temporal out-proj)",
               "FC1": "gemm_bf16_tc_kernel<256, LN-folded +GELU> (FC1)",
               "FC2": "gemm_bf16_tc_kernel<192, +residual> (FC2)",
               "LN1": "row_stats_bf16_kernel (LN1 statistics)", "LN2": "row_stats_bf16_kernel (LN2 statistics)"}
    cands = [n for n in stages if "frac" in stages[n] and stages[n]["bound"] in ("tensor", "hbm")]
    dom = max(cands, key=lambda n: stages[n]["us"])
    d = stages[dom]
    roof = {"kernel": KERNELS.get(dom, dom), "stage": dom, "bound": d["bound"], "achieved": d["achieved"],
            "peak": P["bf16_tflops"] if d["bound"] == "tensor" else P["hbm_gbs"], "unit": d["unit"],
            "frac": d["frac"], "traffic": traffic.get(dom),
            "peak_source": peak_src + ", burst figure (conservative: the kernel runs inside a sub-ms step)",
            "algorithmic_per_launch": d["algorithmic_per_launch"], "algorithmic_unit": d["algorithmic_unit"],
            "launch_us": d["us"], "launches_timed": K,
            "timing": "device stage clock: span from the first CTA past its dependency wait to the last CTA "
                      "exit (%globaltimer, one atomic per CTA), averaged over the K timed graph replays; "
                      "dominant = the longest compute stage",
            "event_us": d["event_us"],
            "event_timing": f"CUDA events around this stage only in a separately captured graph, {KP} replays"}
    kernels = {n: {"kernel": KERNELS[n], **{k: stages[n][k] for k in ("us", "achieved", "unit", "frac", "bound")}}
               for n in KERNELS if n in stages and "frac" in stages[n]}
    clocked_sum_us = float(span_us.sum())
    flops_block = 32 * tokens * sh.C ** 2 + 4 * sh.B * sh.T * sh.S ** 2 * sh.C + 4 * sh.B * sh.S * sh.T ** 2 * sh.C
    t_roof_us = flops_block / N / (P["bf16_tflops"] * 1e12) * 1e6
    nvl_us = 2 * (N - 1) * sh.M // (N * N) * sh.elem_bytes / 900e9 * 1e6
    block_roof = {"t_roofline_us": round(max(t_roof_us, nvl_us), 1), "t_block_us": round(t_ms / K * 1e3, 1),
                  "sum_of_stage_spans_us": round(clocked_sum_us, 1),
                  "frac": round(max(t_roof_us, nvl_us) / (t_ms / K * 1e3), 3),
                  "basis": "max(block FLOPs/N / measured bf16 peak, 2 switches' bytes / 900 GB/s)"}

    # switch bus bandwidth (N > 1): busbw = (N-1)/N * shard_bytes / t
    switch = None
    if world > 1:
        Z = torch.empty_like(X) if impl == "nccl" else None
        if impl != "nccl":
            Z = Y
            src = torch.empty_like(X)
        else:
            src = Y
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for _ in range(3):
            ctx.switch(shape, "T", "S", src, Z, impl=impl)
        barrier()
        for i in range(K):
            evs[i][0].record()
            ctx.switch(shape, "T", "S", src, Z, impl=impl)
            evs[i][1].record()
        barrier()
        ts = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / K], dtype=torch.float64, device=dev)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        sent, _ = dsp.switch_volume(shape, N)
        switch = {"direction": "T->S", "impl": impl, "us": round(float(ts.item()) * 1e3, 2),
                  "busbw_GBps": round(sent / (float(ts.item()) * 1e-3) / 1e9, 1),
                  "algbw_GBps": round(act_bytes / (float(ts.item()) * 1e-3) / 1e9, 1),
                  "nvlink_peak_GBps": 900.0, "bytes_sent_per_rank": sent}

    # e2e through the C ABI with host buffers: dsp_st_block_forward_host_pipelined over K steps,
    # every step's H2D of x (pinned) and D2H of y inside the timed region, the copies of steps
    # i +/- 1 overlapping the block of step i (serving a stream of independent inputs)
    xh = [torch.from_numpy(np.ascontiguousarray(xs).view(np.int16) if sh.dtype == "bf16" else xs).pin_memory()
          for _ in range(2)]
    yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(2)]
    Xd = [torch.empty_like(X), torch.empty_like(X)]
    Yd = [torch.empty_like(X), torch.empty_like(X)] if (impl == "nccl" or N == 1) else [Y, Y2]
    ctx.st_block_forward_host_pipelined(shape, bw, [xh[i % 2] for i in range(max(2, args.warmup))],
                                        [yh[i % 2] for i in range(max(2, args.warmup))], Xd, Yd, impl=impl)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.st_block_forward_host_pipelined(shape, bw, [xh[i % 2] for i in range(K)], [yh[i % 2] for i in range(K)],
                                        Xd, Yd, impl=impl)
    e1.record()
    barrier()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": tokens * K / (float(te.item()) / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": act_bytes,
           "d2h_bytes_per_step": act_bytes, "per_rank": True,
           "path": "dsp_st_block_forward_host_pipelined: pinned H2D / block / D2H per step, copies of adjacent "
                   "steps overlapped with the block (two staging buffers each way); no L2 flush"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            frames, cols, toks = sample_sizes(sh, "baseline")
            v, secs = oracle_sample(sh, args.seed, frames, cols, toks)
            cpu = {"value": v, "unit": "tokens/s", "cores": oracle_threads(), "cpu_model": cpu_model(), "kind": "oracle",
                   "sample": f"float64 numpy oracle, stage-sampled: spatial stage on {frames} frames, temporal stage "
                             f"on {cols} columns, MLP stage on {toks} tokens ({secs:.1f} s); tokens/s = 1 / sum of "
                             f"per-token stage costs"}
        out = {"metric": "ST-block fwd tokens/s", "value": value, "unit": "tokens/s", "n_gpus": N, "steps": K,
               "warmup": args.warmup, "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": sh.dtype, "data": "synthetic",
               "config": {"workload": desc, "B": sh.B, "T": sh.T, "S": sh.S, "C": sh.C, "num_heads": sh.NH,
                          "global_tokens": tokens, "switch_impl": impl if N > 1 else "none (N=1)",
                          "schedule": ("ulysses" if ulysses else "dsp"),
                          "l2": "flushed between timed steps (256 MiB memset outside the events)",
                          "launch": graph_note, "weights": prep_note},
               "roofline": roof, "kernels": kernels, "block_roofline": block_roof, "stages": stages, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "launches_per_step": launches / K, "clocks": clocks.summary()}
        if switch:
            out["switch"] = switch
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def run_model(args):
    """configs[2]: the 28-layer ST-DiT-XL/2-shaped forward (28 blocks at the single-block shape with
    the cross stage of P:137, per-layer weights, prepared), one dsp_st_model_forward per step,
    CUDA-graph replay."""
    import torch
    import torch.distributed as dist

    import paper_2403_10266_b200 as dsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    sh, L, N = synth.CONFIGS["blk"], 28, world
    Tn = sh.T // N
    ctx = dsp.Context(pg=pg, device=dev)
    shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    Lc = 120  # synthetic caption tokens (T5 length of Open-Sora / PixArt), replicated on every rank
    ctx_tokens = to_dev(synth.make_context(sh, args.seed, Lc)).view(sh.B, Lc, sh.C)
    layers = []
    for layer in range(L):
        W = {k: to_dev(v) for k, v in synth.make_block_weights(sh, args.seed, layer=layer).items()}
        W.update({k: to_dev(v) for k, v in synth.make_cross_weights(sh, args.seed, layer=layer).items()})
        W["ctx_tokens"] = ctx_tokens
        W["prepared"] = ctx.prepare_block(shape, W)
        layers.append(W)
    bws = [ctx.block_weights(W) for W in layers]
    X = to_dev(synth.make_x(sh, args.seed, t_range=(rank * Tn, (rank + 1) * Tn)))
    Y = torch.empty_like(X)
    ctx.ensure_workspace(dsp.workspace_bytes(shape, N))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    step_eager = lambda: ctx.st_model_forward(shape, bws, X, Y, impl="nccl")
    for _ in range(args.warmup):
        step_eager()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    l0 = ctx.launch_count()
    with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
        step_eager()
    per_step = ctx.launch_count() - l0
    torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    tokens = sh.B * sh.T * sh.S
    P, _ = peaks()
    flops = L * (32 * tokens * sh.C ** 2 + 4 * sh.B * sh.T * sh.S ** 2 * sh.C + 4 * sh.B * sh.S * sh.T ** 2 * sh.C
                 + 4 * tokens * sh.C ** 2 + 4 * sh.B * Lc * sh.C ** 2 + 4 * tokens * Lc * sh.C)  # + cross stage
    t_roof = flops / N / (P["bf16_tflops"] * 1e12) * 1e3
    if rank == 0:
        print(json.dumps({"metric": "28-layer ST-DiT forward tokens/s", "value": tokens * K / (t_ms / 1e3),
                          "unit": "tokens/s", "n_gpus": N, "steps": K, "warmup": args.warmup, "ms_per_step": t_ms / K,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic",
                          "config": {"workload": "configs[2] ST-DiT-XL/2-shaped: 28 blocks (spatial, temporal, cross "
                                                 "attention to 120 caption tokens, MLP; 743M block parameters), B=1 "
                                                 "T=16 S=1024 C=1152 16 heads, per-layer weights, prepared (LN folded; "
                                                 "LN1 of blocks 1..27 from the previous FC2 epilogue at N=1)",
                                     "l2": "flushed between timed steps", "launch": "cuda graph replay"},
                          "block_equivalent_us": round(t_ms / K / L * 1e3, 1),
                          "roofline": {"t_roofline_ms": round(t_roof, 3), "frac": round(t_roof / (t_ms / K), 3),
                                       "basis": "28 x block FLOPs (incl. the cross stage) / N / measured bf16 peak"},
                          "gpu_launches": per_step * K, "clocks": clocks.summary()}), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def run_nd(args):
    """Multi-dimensional block (DSP schedule P:93): [B, T, H, W, C] = [1, 16, 32, 32, 1152]
    (the single-block config with S = 32 x 32 factored), attention along W, H, T, sharded on T,
    16 heads, bf16, raw weights; one dsp_nd_block_forward per step, CUDA-graph replay."""
    import torch
    import torch.distributed as dist

    import paper_2403_10266_b200 as dsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    N = world
    dims, NH, order, shard = (1, 16, 32, 32, 1152), 16, (3, 2, 1), 1
    C = dims[-1]
    ctx = dsp.Context(pg=pg, device=dev)
    g = torch.Generator(device="cpu").manual_seed(args.seed)
    u = lambda *sh, sc=1.0: ((torch.rand(*sh, generator=g) * 2 - 1) * sc).to(torch.bfloat16).to(dev)
    stages = [dict(ln_w=1 + u(C, sc=0.1), ln_b=u(C, sc=0.1), w_qkv=u(3 * C, C, sc=(3 / C) ** 0.5),
                   w_o=u(C, C, sc=(3 / C) ** 0.5)) for _ in order]
    mlp = dict(ln_w=1 + u(C, sc=0.1), ln_b=u(C, sc=0.1), w_fc1=u(4 * C, C, sc=(3 / C) ** 0.5),
               w_fc2=u(C, 4 * C, sc=0.5 * (3 / (4 * C)) ** 0.5))
    for st_ in stages:
        st_["ln_w"] = st_["ln_w"].contiguous()
    mlp["ln_w"] = mlp["ln_w"].contiguous()
    loc = list(dims)
    loc[shard] //= N
    X = u(*loc)
    ws_bytes = dsp.nd_workspace_bytes(dims, "bf16", N)
    ctx.ensure_workspace(ws_bytes)
    Y = torch.empty_like(X)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    step = lambda: ctx.nd_block_forward(dims, NH, order, stages, mlp, shard, X, Y, impl="nccl")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    l0 = ctx.launch_count()
    with torch.cuda.stream(cap), torch.cuda.graph(gr, stream=cap):
        step()
    per_step = ctx.launch_count() - l0
    torch.cuda.synchronize()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record()
            gr.replay()
            b.record()
        torch.cuda.synchronize()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    tokens = int(np.prod(dims[:-1]))
    P, _ = peaks()
    flops = 40 * tokens * C * C + 4 * tokens * C * sum(dims[k] for k in order)
    t_roof = flops / N / (P["bf16_tflops"] * 1e12) * 1e6
    if rank == 0:
        print(json.dumps({"metric": "N-D block fwd tokens/s", "value": tokens * K / (t_ms / 1e3), "unit": "tokens/s",
                          "n_gpus": N, "steps": K, "warmup": args.warmup, "ms_per_step": t_ms / K,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic",
                          "config": {"workload": "multi-dimensional block [B,T,H,W,C]=[1,16,32,32,1152], attention "
                                                 "along W, H, T, 16 heads, sharded on T (P:44-46, P:93)",
                                     "l2": "flushed between timed steps", "launch": "cuda graph replay"},
                          "roofline": {"t_roofline_us": round(t_roof, 1), "frac": round(t_roof / (t_ms / K * 1e3), 3),
                                       "basis": "block FLOPs / N / measured bf16 peak"},
                          "gpu_launches": per_step * K, "clocks": clocks.summary()}), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def train_flops(sh) -> float:
    """Algorithmic FLOPs of one training step of the block (forward + backward): GEMMs
    32 tok C^2 forward and twice that backward (dgrad + wgrad); attention 4 B T S^2 C + 4 B S T^2 C
    forward (QK^T, PV) and 2.5x that backward (S, dP, dV, dK, dQ)."""
    tok = sh.B * sh.T * sh.S
    attn = 4 * sh.B * sh.T * sh.S ** 2 * sh.C + 4 * sh.B * sh.S * sh.T ** 2 * sh.C
    return 96 * tok * sh.C ** 2 + 3.5 * attn


def run_train(args):
    """one training step of the single ST block (configs[1] shape) = forward_train
    (activations kept) + backward (dx and the twelve fp32 weight gradients) + at N > 1 the ZeRO
    reduce-scatter of the gradients; CUDA-graph replay, L2 flushed between steps."""
    import torch
    import torch.distributed as dist

    import paper_2403_10266_b200 as dsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    sh, N = synth.CONFIGS["blk"], world
    Tn = sh.T // N
    ctx = dsp.Context(pg=pg, device=dev)
    shape = dsp.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    W = {k: to_dev(v) for k, v in synth.make_block_weights(sh, args.seed).items()}
    X = to_dev(synth.make_x(sh, args.seed, t_range=(rank * Tn, (rank + 1) * Tn)))
    gen = torch.Generator(device="cpu").manual_seed(args.seed + 1)
    dY = ((torch.rand(X.shape, generator=gen) * 2 - 1)).to(torch.bfloat16).to(dev)
    Y, dX = torch.empty_like(X), torch.empty_like(X)
    ctx.ensure_workspace(dsp.train_workspace_bytes(shape, N))
    saved = torch.empty(dsp.train_saved_layout(shape, N)["total"], dtype=torch.uint8, device=dev)
    sizes = [W[n].numel() for n in dsp.GRAD_NAMES]
    ntot = (sum(sizes) + N - 1) // N * N
    flat = torch.zeros(ntot, dtype=torch.float32, device=dev)
    shard = torch.zeros(ntot // N, dtype=torch.float32, device=dev)
    G, o = {}, 0
    for n, k in zip(dsp.GRAD_NAMES, sizes):
        G[n] = flat[o:o + k].view(W[n].shape)
        o += k
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def fwd():
        ctx.block_forward_train(shape, W, X, Y, saved, impl="nccl")

    def bwd():
        flat.zero_()
        ctx.block_backward(shape, W, saved, X, dY, dX, G, impl="nccl")
        if N > 1:
            ctx.grads_reduce(flat, zero_shard=True, out=shard)

    def step():
        fwd()
        bwd()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graphs = {}
    for name, fn_ in (("step", step), ("fwd", fwd), ("bwd", bwd)):
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        l0 = ctx.launch_count()
        with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
            fn_()
        graphs[name] = (g, ctx.launch_count() - l0)
    torch.cuda.synchronize()
    K = args.steps

    def timed(g):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(local) as clocks:
        t_ms = timed(graphs["step"][0])
    t_f, t_b = timed(graphs["fwd"][0]), timed(graphs["bwd"][0])
    tokens = sh.B * sh.T * sh.S
    P, _ = peaks()
    flops = train_flops(sh)
    t_roof = flops / N / (P["bf16_tflops"] * 1e12) * 1e3
    if rank == 0:
        print(json.dumps({"metric": "ST-block train step (fwd+bwd) tokens/s", "value": tokens * K / (t_ms / 1e3),
                          "unit": "tokens/s", "n_gpus": N, "steps": K, "warmup": args.warmup, "ms_per_step": t_ms / K,
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic",
                          "config": {"workload": "configs[1] single ST block training step: forward_train + backward "
                                                 "(dx, 12 fp32 weight gradients)" + (" + ZeRO reduce-scatter" if N > 1 else "")
                                                 + ", B=1 T=16 S=1024 C=1152 16 heads, raw weights",
                                     "l2": "flushed between timed steps", "launch": "cuda graph replay"},
                          "breakdown_ms": {"forward_train": round(t_f / K, 4), "backward": round(t_b / K, 4)},
                          "roofline": {"bound": "tensor", "achieved": round(flops / N / (t_ms / K / 1e3) / 1e12, 1),
                                       "peak": P["bf16_tflops"], "unit": "TFLOP/s",
                                       "frac": round(t_roof / (t_ms / K), 3), "traffic": None,
                                       "t_roofline_ms": round(t_roof, 4), "flops_per_step": flops,
                                       "basis": "whole training step: train FLOPs (bench.train_flops) / N over the "
                                                "device-timed step, against the measured bf16 peak (per-kernel "
                                                "shares: profiles/r02/train/launches_train_step.txt)"},
                          "gpu_launches": graphs["step"][1] * K, "clocks": clocks.summary()}), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(gpus: int, argv: list) -> int:
    """`python bench.py --gpus N` outside torchrun: re-launch this script as N ranks through
    torch.distributed.run on 127.0.0.1 (one process per GPU, RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_* set by the launcher); rank 0's JSON line reaches our stdout.  Returns the exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def launcher_check(args):
    """CPU check of the multi-rank launch (no GPU): every rank joins a gloo group and rank 0
    prints the ranks it saw."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.zeros(world, dtype=torch.int64)
    t[rank] = rank + 1
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launcher_check": True, "world": world, "gpus": args.gpus,
                          "ranks": [int(v) - 1 for v in t.tolist()],
                          "local_ranks_env": os.environ.get("LOCAL_RANK")}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dsp", choices=["dsp", "reference"])
    ap.add_argument("--config", default="blk", choices=list(CONFIGS) + ["model28", "nd", "train"])
    ap.add_argument("--switch", default="nccl", choices=["nccl", "p2p", "fused"])
    ap.add_argument("--schedule", default="dsp", choices=["dsp", "ulysses"],
                    help="ulysses: DeepSpeed-Ulysses on the same kernels (4 all-to-alls per attention stage)")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prepare", dest="prepare", action="store_false",
                    help="raw weights: LayerNorm kernels inside the block instead of the folded path")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="eager launches instead of graph replay")
    ap.add_argument("--launcher-check", action="store_true",
                    help="CPU-only: spawn --gpus ranks, join a gloo group, print the ranks (tests the launcher)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "RANK" not in os.environ and args.impl != "reference":
        raise SystemExit(spawn_ranks(args.gpus, sys.argv[1:]))
    if args.launcher_check:
        return launcher_check(args)
    if args.impl == "reference":
        if args.config == "model28":  # 28 blocks of the blk shape: the oracle's block cost x 28
            args.config, args.layers = "blk", 28
        elif args.config == "nd":
            return print(json.dumps({"impl": "reference", "unavailable": "no oracle timing leg for the N-D block"}))
        elif args.config == "train":
            return print(json.dumps({"impl": "reference", "unavailable": "no oracle timing leg for the training step"}))
        run_reference(args)
    elif args.config == "model28":
        run_model(args)
    elif args.config == "nd":
        run_nd(args)
    elif args.config == "train":
        run_train(args)
    else:
        run_dsp(args)


if __name__ == "__main__":
    main()
