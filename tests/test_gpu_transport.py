"""GPU tests of the switch / split / gather transports against the oracle (bit-exact).

The NCCL transport of dsp_switch is pack -> ncclAlltoAll -> unpack (include/dsp_kernels.h).
NCCL cannot put two ranks on one GPU, so these tests run the library's own pack and unpack
kernels (dsp_switch_pack / dsp_switch_unpack) for every virtual rank and emulate the
all-to-all between them in NCCL's chunk order (recv_q[r] = send_r[q]); the gather's unpack
(dsp_gather_unpack) is tested the same way.  Everything is compared bitwise with
oracle.switch / oracle.split / oracle.gather on index-tagged inputs (every token row carries
its global index), at the configs[1] shape.  The P2P barrier tests check the device-resident
epoch under CUDA-graph replay and the timeout path (§3.1, §3.2).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import switch as osw
from tests.test_gpu_block import VirtualGroup, _run_block_n1, _setup
from tests.gpu_util import bits16, to_dev, weights_dev

pytestmark = pytest.mark.gpu

BLK = synth.CONFIGS["blk"]
DIMS = {"T": osw.DIM_T, "S": osw.DIM_S}


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _tagged(B):
    sh = synth.BlockShape(B, BLK.T, BLK.S, BLK.C, BLK.NH, "bf16")
    return sh, synth.make_index_tagged(sh, 11)


def _dev16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16).reshape(-1)).cuda()


def _host16(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 2])
@pytest.mark.parametrize("direction", ["TS", "ST"])
def test_switch_nccl_transport_pack_a2a_unpack_bitexact(N, B, direction):
    """dsp_switch's NCCL transport piece by piece at the blk shape: every rank packs its shard
    into per-peer chunks (checked against the oracle's outbox: chunk q of rank r is exactly the
    message r sends q), the all-to-all is emulated in chunk order, every rank unpacks; the
    result equals oracle.switch bitwise."""
    m = dsp()
    sh, x = _tagged(B)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    fr, to = (direction[0], direction[1])
    src = osw.split(x, DIMS[fr], N)
    want = osw.switch(src, DIMS[fr], DIMS[to])
    ctx = [m.Context(rank=r, world=N) for r in range(N)]
    nb = sh.M // N  # int16 elements per shard
    chunk = nb // N
    xs = [_dev16(src[r]) for r in range(N)]
    send = [torch.empty(nb, dtype=torch.int16, device="cuda") for _ in range(N)]
    for r in range(N):
        ctx[r].switch_pack(shape, fr, to, xs[r].view(torch.bfloat16), send[r].view(torch.bfloat16))
    torch.cuda.synchronize()
    n_to = (sh.S if to == "S" else sh.T) // N
    for r in range(N):
        got = _host16(send[r])
        for q in range(N):
            sl = [slice(None)] * 4
            sl[DIMS[to]] = slice(q * n_to, (q + 1) * n_to)
            assert np.array_equal(got[q * chunk:(q + 1) * chunk], src[r][tuple(sl)].reshape(-1)), (r, q)
    recv = [torch.cat([send[r][q * chunk:(q + 1) * chunk] for r in range(N)]) for q in range(N)]
    ys = [torch.empty(nb, dtype=torch.int16, device="cuda") for _ in range(N)]
    for q in range(N):
        ctx[q].switch_unpack(shape, fr, to, recv[q].view(torch.bfloat16), ys[q].view(torch.bfloat16))
    torch.cuda.synchronize()
    for q in range(N):
        assert np.array_equal(_host16(ys[q]), want[q].reshape(-1)), f"rank {q}"


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("dim", ["T", "S"])
@pytest.mark.parametrize("B", [1, 2])
def test_split_bitexact(N, dim, B):
    """dsp_split: rank r's chunk of the global tensor, bitwise = oracle.split."""
    m = dsp()
    sh, x = _tagged(B)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    want = osw.split(x, DIMS[dim], N)
    X = _dev16(x).view(torch.bfloat16)
    for r in range(N):
        c = m.Context(rank=r, world=N)
        out = torch.empty(sh.M // N, dtype=torch.bfloat16, device="cuda")
        c.split(shape, dim, X, out)
        torch.cuda.synchronize()
        assert np.array_equal(_host16(out), want[r].reshape(-1)), f"rank {r}"


@pytest.mark.parametrize("dim", ["T", "S"])
def test_gather_n1_bitexact(dim):
    """dsp_gather at N = 1 (the collective's single-rank case): a copy of the shard."""
    m = dsp()
    sh, x = _tagged(2)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    c = m.Context()
    out = torch.empty(sh.M, dtype=torch.bfloat16, device="cuda")
    c.gather(shape, dim, _dev16(x).view(torch.bfloat16), out)
    torch.cuda.synchronize()
    assert np.array_equal(_host16(out), osw.gather([x], DIMS[dim]).reshape(-1))


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("dim", ["T", "S"])
@pytest.mark.parametrize("B", [1, 2])
def test_gather_unpack_bitexact(N, dim, B):
    """dsp_gather at N > 1 = ncclAllGather (rank-major [N][local]) + dsp_gather_unpack; the
    all-gather is emulated by concatenating the shards in rank order."""
    m = dsp()
    sh, x = _tagged(B)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    shards = osw.split(x, DIMS[dim], N)
    gathered = torch.cat([_dev16(s) for s in shards])
    out = torch.empty(sh.M, dtype=torch.bfloat16, device="cuda")
    m.Context(rank=1, world=N).gather_unpack(shape, dim, gathered.view(torch.bfloat16), out)
    torch.cuda.synchronize()
    assert np.array_equal(_host16(out), osw.gather(shards, DIMS[dim]).reshape(-1))


def test_switch_pack_validation():
    m = dsp()
    sh, x = _tagged(1)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    c = m.Context(rank=0, world=2)
    a = torch.empty(sh.M // 2, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(m.DSPError) as e:
        c.switch_pack(shape, "T", "T", a, torch.empty_like(a))
    assert e.value.name == "DSP_ERR_SAME_DIM"
    with pytest.raises(m.DSPError) as e:
        c.switch_pack(shape, "T", "S", a, a)
    assert e.value.name == "DSP_ERR_ALIAS"


# ------------------------------------------------------------------ P2P barrier
def _epoch(g, r):
    return int(g.sig[r][8].item())


def test_p2p_switch_graph_replay_device_epoch():
    """The P2P barrier's epoch lives in device memory: two virtual ranks capture
    their switch into CUDA graphs; every replay advances each rank's device counter by the two
    barriers of a switch, and every replay on fresh inputs is bit-exact."""
    m = dsp()
    N = 2
    sh = synth.BlockShape(1, 16, 256, 256, 4, "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    nb = sh.M * 2 // N
    g = VirtualGroup(N, 2 * nb)
    xin = [g.view(r, 0, nb, torch.int16) for r in range(N)]
    ys = [g.view(r, nb, nb, torch.int16) for r in range(N)]
    graphs = [torch.cuda.CUDAGraph() for _ in range(N)]
    for r in range(N):  # capture does not execute: the device counters stay at 0
        with torch.cuda.graph(graphs[r], stream=g.streams[r]):
            g.ctx[r].switch(shape, "T", "S", xin[r].view(torch.bfloat16), ys[r].view(torch.bfloat16), impl="p2p")
    torch.cuda.synchronize()
    assert _epoch(g, 0) == 0 and _epoch(g, 1) == 0
    for it in range(5):
        x = synth.make_index_tagged(sh, 100 + it)
        tsh = osw.split(x, osw.DIM_T, N)
        for r in range(N):
            xin[r].copy_(_dev16(tsh[r]))
        torch.cuda.synchronize()
        g.run(lambda r: graphs[r].replay())
        want = osw.switch(tsh, osw.DIM_T, osw.DIM_S)
        for r in range(N):
            assert np.array_equal(_host16(ys[r]), want[r].reshape(-1)), f"replay {it} rank {r}"
            assert _epoch(g, r) == 2 * (it + 1)
    for c in g.ctx:
        c.check_errors()


@pytest.mark.parametrize("prepared", [False, True])
@pytest.mark.parametrize("impl", ["p2p", "fused"])
def test_block_graph_replay_virtual_ranks_bitwise(impl, prepared):
    """The bench's launch mode for P2P / fused at N > 1: each virtual rank's block captured in a
    CUDA graph and replayed three times equals the N = 1 block bitwise every time.  Prepared +
    fused runs the split T->S barrier (PROJ_S's last CTA arrives, the LN2 partials pass waits per
    sending rank): its epochs must advance exactly like the barrier kernel's under replay."""
    m = dsp()
    N = 2
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = _setup(sh)
    ref1 = bits16(_run_block_n1(sh, xs, Ws, prepared=prepared))
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    W = weights_dev(Ws, "bf16")
    if prepared:
        W["prepared"] = g.ctx[0].prepare_block(shape, W)
        torch.cuda.synchronize()
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    graphs = [torch.cuda.CUDAGraph() for _ in range(N)]
    for r in range(N):
        with torch.cuda.graph(graphs[r], stream=g.streams[r]):
            g.ctx[r].st_block_forward(shape, W, X[r], Y[r], impl=impl)
    torch.cuda.synchronize()
    per_block = _epoch(g, 0)
    assert per_block == 0
    for it in range(3):
        for r in range(N):
            Y[r].zero_()
        torch.cuda.synchronize()
        g.run(lambda r: graphs[r].replay())
        got = np.concatenate([bits16(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
        assert np.array_equal(got.reshape(-1), ref1.reshape(-1)), f"replay {it}"
    assert _epoch(g, 0) == _epoch(g, 1) > 0
    for c in g.ctx:
        c.check_errors()


def test_p2p_barrier_timeout_is_reported_not_trapped():
    """A peer that never arrives: the barrier gives up after the wall-clock timeout, records
    (epoch, peer) in the pad and returns (no __trap, the CUDA context survives);
    dsp_ctx_check_errors raises DSP_ERR_PEER_TIMEOUT naming the peer."""
    m = dsp()
    N = 2
    sh = synth.BlockShape(1, 4, 64, 64, 1, "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, 1, "bf16")
    nb = sh.M * 2 // N
    g = VirtualGroup(N, 2 * nb)
    g.ctx[0].set_barrier_timeout(0.05)
    g.ctx[0].check_errors()
    g.ctx[0].switch(shape, "T", "S", g.view(0, 0, nb, torch.bfloat16), g.view(0, nb, nb, torch.bfloat16), impl="p2p")
    torch.cuda.synchronize()  # returns: both barriers timed out instead of hanging
    with pytest.raises(m.DSPError) as e:
        g.ctx[0].check_errors()
    assert e.value.name == "DSP_ERR_PEER_TIMEOUT" and "rank 1" in str(e.value)
    assert _epoch(g, 0) == 2
    t = torch.arange(10, device="cuda").sum()  # the context is alive
    assert int(t.item()) == 45
    g.ctx[1].check_errors()  # the peer itself saw nothing


# ------------------------------------------------------------------ NCCL code path, emulated
def _emulated_group(N, region_bytes):
    g = VirtualGroup(N, region_bytes)
    for c in g.ctx:
        c.set_collective_emulation(True)
    return g


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 2])
@pytest.mark.parametrize("direction", ["TS", "ST"])
def test_switch_nccl_code_path_emulated_bitexact(N, B, direction):
    """dsp_switch(impl = NCCL) end to end over N virtual ranks at the blk shape: the library's own
    NCCL branch (pack into the workspace unless identity, all-to-all, unpack unless identity) with
    only the ncclAlltoAll call replaced by the emulated collective (barrier + pull + barrier)."""
    m = dsp()
    sh, x = _tagged(B)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    fr, to = direction[0], direction[1]
    src = osw.split(x, DIMS[fr], N)
    want = osw.switch(src, DIMS[fr], DIMS[to])
    nb = sh.M * 2 // N  # bytes per shard
    g = _emulated_group(N, 4 * nb)  # x | y | workspace (send + recv staging)
    for r in range(N):
        g.view(r, 0, nb, torch.int16).copy_(_dev16(src[r]))
        g.ctx[r].set_workspace(g.region[r][2 * nb:])
    xs = [g.view(r, 0, nb, torch.bfloat16) for r in range(N)]
    ys = [g.view(r, nb, nb, torch.bfloat16) for r in range(N)]
    g.run(lambda r: g.ctx[r].switch(shape, fr, to, xs[r], ys[r], impl="nccl"))
    for r in range(N):
        assert np.array_equal(_host16(ys[r]), want[r].reshape(-1)), f"rank {r}"
    for c in g.ctx:
        c.check_errors()


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("dim", ["T", "S"])
@pytest.mark.parametrize("B", [1, 2])
def test_gather_nccl_code_path_emulated_bitexact(N, dim, B):
    """dsp_gather at N > 1 end to end (all-gather into x_global or the workspace + the unpack kernel)
    with the ncclAllGather call emulated; every rank's x_global equals oracle.gather bitwise."""
    m = dsp()
    sh, x = _tagged(B)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    shards = osw.split(x, DIMS[dim], N)
    nb = sh.M * 2 // N
    g = _emulated_group(N, nb + sh.M * 2)  # x_local | workspace
    for r in range(N):
        g.view(r, 0, nb, torch.int16).copy_(_dev16(shards[r]))
        g.ctx[r].set_workspace(g.region[r][nb:])
    outs = [torch.empty(sh.M, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    g.run(lambda r: g.ctx[r].gather(shape, dim, g.view(r, 0, nb, torch.bfloat16), outs[r]))
    want = osw.gather(shards, DIMS[dim]).reshape(-1)
    for r in range(N):
        assert np.array_equal(_host16(outs[r]), want), f"rank {r}"


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("prepared", [False, True])
def test_block_nccl_code_path_emulated_n_invariant(N, prepared):
    """The block with impl = NCCL (bench.py's default transport at N > 1) over N virtual ranks at
    the blk shape, collectives emulated: bitwise equal to the N = 1 block (raw and prepared)."""
    m = dsp()
    sh = synth.CONFIGS["blk"]
    xs, Ws = _setup(sh)
    ref1 = bits16(_run_block_n1(sh, xs, Ws, prepared=prepared))
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = _emulated_group(N, ws + act)
    W = weights_dev(Ws, "bf16")
    if prepared:
        W["prepared"] = g.ctx[0].prepare_block(shape, W)
        torch.cuda.synchronize()
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, X[r], Y[r], impl="nccl"))
    got = np.concatenate([bits16(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref1.reshape(-1))
