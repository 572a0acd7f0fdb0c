"""World-size-2 multi-process test of the N>1 switch path on CPU (gloo).

Each process is one rank.  It asks the C ABI for its switch plan (dsp_switch_plan, the
host logic both GPU transports execute), packs its T-shard into per-peer chunks in the
plan's chunk order [peer][b][t'][s'][c], exchanges them with a real gloo all_to_all
(the collective the NCCL transport issues), unpacks with the plan's destination
strides, and checks the result against the oracle's S-shard bit-exactly; then back.
"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _switch_via_plan(m, shape, N, rank, frm, to, x_local: np.ndarray) -> np.ndarray:
    plan = m.switch_plan(shape, N, rank, frm, to)
    n0, n1, n2, run = plan.n[0], plan.n[1], plan.n[2], plan.run_bytes
    chunk = n1 * n2 * run
    xb = x_local.view(np.uint8).reshape(-1)
    send = np.empty(N * chunk, dtype=np.uint8)
    for q in range(n0):
        for b in range(n1):
            for t in range(n2):
                s = q * plan.src_stride[0] + b * plan.src_stride[1] + t * plan.src_stride[2]
                d = q * chunk + (b * n2 + t) * run
                send[d:d + run] = xb[s:s + run]
    recv = torch.empty(N * chunk, dtype=torch.uint8)
    dist.all_to_all_single(recv, torch.from_numpy(send))
    rb = recv.numpy()
    y = np.empty(x_local.nbytes, dtype=np.uint8)
    for src in range(n0):
        for b in range(n1):
            for t in range(n2):
                s = src * chunk + (b * n2 + t) * run
                d = src * plan.dst_stride[0] + b * plan.dst_stride[1] + t * plan.dst_stride[2]
                y[d:d + run] = rb[s:s + run]
    return y.view(x_local.dtype)


def _worker(rank, world, port, B, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import paper_2403_10266_b200 as m
        import synth
        from oracle import switch as osw
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sh = synth.BlockShape(B, 8, 16, 16, 1, "bf16")
        shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, 1, "bf16")
        x = synth.make_index_tagged(sh, 21)
        tsh = osw.split(x, osw.DIM_T, world)
        want_s = osw.switch(tsh, osw.DIM_T, osw.DIM_S)[rank]
        y = _switch_via_plan(m, shape, world, rank, osw.DIM_T, osw.DIM_S, tsh[rank]).reshape(want_s.shape)
        ok1 = np.array_equal(y, want_s)
        back = _switch_via_plan(m, shape, world, rank, osw.DIM_S, osw.DIM_T, y).reshape(tsh[rank].shape)
        ok2 = np.array_equal(back, tsh[rank])
        sent, _ = m.switch_volume(shape, world)
        q.put((rank, ok1, ok2, sent))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), False, 0))


@pytest.mark.parametrize("B", [1, 2])
def test_switch_world2_gloo(B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok1, ok2, sent in res:
        assert ok1 is True, (rank, ok1)
        assert ok2 is True
        assert sent == (world - 1) * B * (8 // world) * (16 // world) * 16 * 2


@pytest.mark.parametrize("n", [2, 4])
def test_bench_self_spawns_n_ranks(n):
    """`python bench.py --gpus N` started WITHOUT torchrun re-launches itself as N ranks (one
    process per GPU on a GPU box) through torch.distributed.run on 127.0.0.1; here every rank
    joins a gloo group and rank 0 alone prints the ranks it saw."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launcher-check"],
                       capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    out = json.loads(lines[0])
    assert out["world"] == n and out["ranks"] == list(range(n))


def _bwd_worker(rank, world, port, q):
    """One rank of the DSP backward (f4) on CPU: the oracle's per-stage backward pieces run on this rank's
    shards; the two switches of the backward go through the library's plan (dsp_switch_plan) and a real
    gloo all_to_all, T->S for dy (the adjoint of the forward's S->T) and S->T for dy1 (adjoint of T->S);
    the weight gradients are all-reduced (the sum ZeRO reduce-scatters)."""
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import paper_2403_10266_b200 as m
        import synth
        from oracle import backward as bw
        from oracle import block as ob
        from oracle import switch as osw
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sh = synth.BlockShape(1, 4, 8, 16, 2, "f32")
        shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "f32")
        W = {k: synth.to_f64(v, "f32") for k, v in synth.make_block_weights(sh, 5).items()}
        x = synth.to_f64(synth.make_x(sh, 5), "f32")
        dy = np.random.default_rng(9).standard_normal(x.shape)
        dx_ref, g_ref = bw.st_block_bwd(x, W, sh.NH, dy)
        xs = osw.split(x, osw.DIM_T, world)[rank]
        y1 = ob.spatial_stage(xs, W, sh.NH)                                       # forward on this rank
        y1s = _switch_via_plan(m, shape, world, rank, osw.DIM_T, osw.DIM_S, y1.astype(np.float32)).astype(np.float64)
        y1s = y1s.reshape(sh.B, sh.T, sh.S // world, sh.C)
        y2 = ob.temporal_stage(y1s, W, sh.NH)
        dys = osw.split(dy, osw.DIM_T, world)[rank].astype(np.float32)
        dz = _switch_via_plan(m, shape, world, rank, osw.DIM_T, osw.DIM_S, dys).astype(np.float64)
        dz = dz.reshape(y2.shape)
        dy2, gm = bw.mlp_stage_bwd(y2, W, dz)
        dy1s, gt = bw.temporal_stage_bwd(y1s, W, sh.NH, dy2)
        dy1 = _switch_via_plan(m, shape, world, rank, osw.DIM_S, osw.DIM_T, dy1s.astype(np.float32)).astype(np.float64)
        dx, gs = bw.spatial_stage_bwd(xs, W, sh.NH, dy1.reshape(xs.shape))
        ok_dx = np.allclose(dx, osw.split(dx_ref, osw.DIM_T, world)[rank], rtol=1e-5, atol=1e-5)
        worst = 0.0
        for n, v in {**gm, **gt, **gs}.items():
            t = torch.from_numpy(np.ascontiguousarray(v))
            dist.all_reduce(t)
            worst = max(worst, float(np.abs(t.numpy() - g_ref[n]).max() / max(np.abs(g_ref[n]).max(), 1e-30)))
        q.put((rank, bool(ok_dx), worst))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), 1.0))


def test_backward_schedule_world2_gloo():
    """The DSP backward over two processes (library switch plans + gloo all_to_all + all_reduce of the
    weight gradients) equals the unsharded oracle backward (the f32 wire format rounds the exchanged
    activations: 1e-5)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bwd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, worst in res:
        assert ok is True, (rank, ok)
        assert worst < 1e-4, (rank, worst)
