"""Switch-only sweep (BASELINE.json configs[4]): the dynamic switch T->S and
S->T of a [B, T, S, C] bf16 activation from 1 MiB to 4 GiB global, bus bandwidth against
NVLink, plus the model-shaped points (blk, long video).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/switch_sweep.py [--impl nccl,p2p]
      N GPUs, one rank per GPU: dsp_switch through NCCL (pack -> ncclAlltoAll -> unpack) and
      through direct NVLink stores into the peers' symmetric buffers (P2P); the NCCL ceiling
      (torch all_to_all_single on the same bytes, nothing to pack) beside it.
  python scripts/switch_sweep.py --vranks N
      ONE GPU: N virtual ranks (N contexts, peer buffers are N local allocations, one stream
      each) through the real P2P kernels.  Peer stores stay in local HBM, so this measures the
      switch kernels' own cost (HBM GB/s), not NVLink.

Sizes: B=1, C=1024, T=16, S = 32 * 2^k (k = 0..12) -> global 2^20 .. 2^32 bytes exactly.
Per point: warm-up 5, then 200 (shard < 16 MiB) or 20 timed switches, CUDA events per call,
median; multi-GPU: max over ranks.  busbw = off-rank bytes sent per rank / t = (N-1)/N *
shard / t (nccl-tests convention); algbw = shard / t.  Every point is checked
bit-exact once against slices of the global tensor (pattern = hash of the global index).
One JSON line per point on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # virtual ranks spin on each other (see tests/conftest.py)

import torch  # noqa: E402

import paper_2403_10266_b200 as dsp  # noqa: E402

NVLINK_GBS = 900.0


def sweep_shapes(max_gib: float):
    pts = []
    for k in range(13):
        S = 32 << k
        if 16 * S * 1024 * 2 > max_gib * (1 << 30):
            break
        pts.append((f"sweep_{16 * S * 1024 * 2 >> 20}MiB", 1, 16, S, 1024))
    pts.append(("blk_C1152", 1, 16, 1024, 1152))
    if max_gib >= 1.2:
        pts.append(("long_C1152", 1, 128, 4096, 1152))
    return pts


def pattern_global(B, T, S, C, dev):
    """int16 view of a [B, T, S, C] tensor whose every element is a hash of its global index."""
    n = B * T * S * C
    i = torch.arange(n, device=dev, dtype=torch.int64)
    v = ((i * 2654435761) >> 7) & 0xFFFF
    return (v - 32768).to(torch.int16).view(B, T, S, C)


def time_calls(fn, iters, streams=None):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[len(t) // 2] * 1e-3  # seconds, median


def run_multi(args):
    import torch.distributed as dist
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ctx = dsp.Context(pg=dist.group.WORLD, device=dev)
    impls = args.impl.split(",")
    for name, B, T, S, C in sweep_shapes(args.max_gib):
        shape = dsp.make_shape(B, T, S, C, 1, "bf16")
        Tn, Sn = T // world, S // world
        shard = B * Tn * S * C * 2
        G = pattern_global(B, T, S, C, dev) if shard * world <= (256 << 20) else None
        iters = 200 if shard < (16 << 20) else 20
        for impl in impls:
            if impl == "p2p":
                import torch.distributed._symmetric_memory as symm
                buf = symm.empty(2 * shard, dtype=torch.uint8, device=dev)
                hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
                ctx.set_peer_buffers(hdl.buffer_ptrs, hdl.signal_pad_ptrs, 2 * shard)
                xT, yS = buf[:shard].view(torch.bfloat16), buf[shard:].view(torch.bfloat16)
            else:
                ctx.ensure_workspace(2 * shard)
                xT = torch.empty(shard // 2, dtype=torch.bfloat16, device=dev)
                yS = torch.empty_like(xT)
            ok = None
            if G is not None:
                xT.view(torch.int16).copy_(G[:, rank * Tn:(rank + 1) * Tn].reshape(-1))
                ctx.switch(shape, "T", "S", xT, yS, impl=impl)
                torch.cuda.synchronize()
                ok = bool(torch.equal(yS.view(torch.int16), G[:, :, rank * Sn:(rank + 1) * Sn].reshape(-1)))
            for direction, (a, b, src, dst) in {"T->S": ("T", "S", xT, yS), "S->T": ("S", "T", yS, xT)}.items():
                t = time_calls(lambda: ctx.switch(shape, a, b, src, dst, impl=impl), iters)
                tt = torch.tensor([t], dtype=torch.float64, device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt.item())
                sent = (world - 1) * shard // world
                if rank == 0:
                    print(json.dumps({"point": name, "global_bytes": shard * world, "n_gpus": world, "impl": impl,
                                      "direction": direction, "us": round(t * 1e6, 2),
                                      "busbw_GBps": round(sent / t / 1e9, 1), "algbw_GBps": round(shard / t / 1e9, 1),
                                      "nvlink_frac": round(sent / t / 1e9 / NVLINK_GBS, 3),
                                      "bitexact": ok}), flush=True)
            del xT, yS
        # NCCL ceiling: all_to_all_single on the same bytes (already packed: nothing to do)
        inp = torch.empty(shard, dtype=torch.uint8, device=dev)
        out = torch.empty_like(inp)
        t = time_calls(lambda: dist.all_to_all_single(out, inp), iters)
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        if rank == 0:
            sent = (world - 1) * shard // world
            print(json.dumps({"point": name, "global_bytes": shard * world, "n_gpus": world,
                              "impl": "torch.all_to_all_single (NCCL ceiling, pre-packed)", "us": round(t * 1e6, 2),
                              "busbw_GBps": round(sent / t / 1e9, 1), "nvlink_frac": round(sent / t / 1e9 / NVLINK_GBS, 3)}),
                  flush=True)
        del inp, out
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()


def run_virtual(args):
    N = args.vranks
    dev = torch.device("cuda", 0)
    ctxs = [dsp.Context(rank=r, world=N) for r in range(N)]
    streams = [torch.cuda.Stream() for _ in range(N)]
    for name, B, T, S, C in sweep_shapes(args.max_gib):
        shape = dsp.make_shape(B, T, S, C, 1, "bf16")
        Tn, Sn = T // N, S // N
        shard = B * Tn * S * C * 2
        region = [torch.empty(2 * shard, dtype=torch.uint8, device=dev) for _ in range(N)]
        sig = [torch.zeros(dsp.SIGNAL_PAD_BYTES // 8, dtype=torch.int64, device=dev) for _ in range(N)]
        for c in ctxs:
            c.set_peer_buffers([t.data_ptr() for t in region], [t.data_ptr() for t in sig], 2 * shard)
        xT = [region[r][:shard].view(torch.bfloat16) for r in range(N)]
        yS = [region[r][shard:].view(torch.bfloat16) for r in range(N)]

        def group(a, b, src, dst):
            cur = torch.cuda.current_stream()
            for s in streams:
                s.wait_stream(cur)
            for r in range(N):
                with torch.cuda.stream(streams[r]):
                    ctxs[r].switch(shape, a, b, src[r], dst[r], impl="p2p")
            for s in streams:
                cur.wait_stream(s)

        ok = None
        if shard * N <= (256 << 20):
            G = pattern_global(B, T, S, C, dev)
            for r in range(N):
                xT[r].view(torch.int16).copy_(G[:, r * Tn:(r + 1) * Tn].reshape(-1))
            group("T", "S", xT, yS)
            torch.cuda.synchronize()
            ok = all(torch.equal(yS[r].view(torch.int16), G[:, :, r * Sn:(r + 1) * Sn].reshape(-1)) for r in range(N))
            del G
        iters = 200 if shard < (16 << 20) else 20
        for direction, (a, b, src, dst) in {"T->S": ("T", "S", xT, yS), "S->T": ("S", "T", yS, xT)}.items():
            # one CUDA graph per point: the N ranks' launches become parallel graph branches, so
            # the time is the device's (host launch cost of N Python-driven ranks excluded)
            group(a, b, src, dst)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap), torch.cuda.graph(g, stream=cap):
                group(a, b, src, dst)
            torch.cuda.synchronize()
            t = time_calls(g.replay, iters)
            moved = N * shard * 2  # every rank reads its shard and writes its shard (local HBM)
            print(json.dumps({"point": name, "global_bytes": shard * N, "virtual_ranks": N, "impl": "p2p (virtual ranks, graph)",
                              "direction": direction, "us": round(t * 1e6, 2),
                              "hbm_GBps": round(moved / t / 1e9, 1), "bitexact": ok,
                              "note": "peer stores land in local HBM: kernel cost, not NVLink"}), flush=True)
        del region, sig, xT, yS
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="nccl,p2p")
    ap.add_argument("--vranks", type=int, default=0)
    ap.add_argument("--max-gib", type=float, default=4.0)
    args = ap.parse_args()
    if args.vranks:
        run_virtual(args)
    else:
        run_multi(args)


if __name__ == "__main__":
    main()
