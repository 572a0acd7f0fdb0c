"""GPU parity of the public stages and the ST block vs the float64 oracle.

Multi-rank paths are exercised on ONE GPU with "virtual ranks": N contexts (rank r of
world N) whose peer buffers are N local allocations, running concurrently on N
streams, with the P2P switch transport (direct stores + signal-pad barriers).  The
kernel logic is identical to the multi-GPU case; only the peer addresses are local.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import block as ob
from oracle import switch as osw
from tests.gpu_util import assert_block_close, bits16, to_dev, to_f64, weights_dev, weights_f64

pytestmark = pytest.mark.gpu


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _setup(sh: synth.BlockShape, seed=7, kappa=1.0):
    Ws = synth.make_block_weights(sh, seed, kappa=kappa)
    xs = synth.make_x(sh, seed)
    return xs, Ws


def _run_block_n1(sh, xs, Ws, prepared=False):
    m = dsp()
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, sh.dtype)
    Y = torch.empty_like(X)
    W = weights_dev(Ws, sh.dtype)
    if prepared:
        W["prepared"] = ctx.prepare_block(shape, W)
    ctx.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    return Y


def test_block_tiny_f32_check_path():
    """configs[0]: tiny ST block (T=4, S=16, C=64, 4 heads) fp32 check path, gate 1e-4."""
    sh = synth.CONFIGS["tiny"]
    xs, Ws = _setup(sh)
    Y = _run_block_n1(sh, xs, Ws)
    ref = ob.st_block(synth.to_f64(xs, "f32"), weights_f64(Ws, "f32"), sh.NH)
    np.testing.assert_allclose(to_f64(Y), ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("sh", [synth.BlockShape(1, 16, 256, 1152, 16, "bf16"),
                                synth.BlockShape(2, 8, 128, 256, 4, "bf16"),
                                synth.BlockShape(1, 4, 128, 1152, 16, "bf16")])
def test_block_bf16_full_oracle(sh):
    xs, Ws = _setup(sh)
    Y = _run_block_n1(sh, xs, Ws)
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    print(assert_block_close(to_f64(Y), ref))


@pytest.mark.parametrize("sh", [synth.BlockShape(1, 16, 256, 1152, 16, "bf16"),
                                synth.BlockShape(2, 8, 128, 256, 4, "bf16")])
def test_block_bf16_prepared_layernorm_folded(sh):
    """Prepared weights (dsp_st_block_prepare, R30): every LayerNorm folded into the GEMM that
    consumes it -- LN1 from row statistics, LN2/LN3 from the out-projection epilogues' per-row
    partials -- against the same oracle block."""
    xs, Ws = _setup(sh)
    Y = _run_block_n1(sh, xs, Ws, prepared=True)
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    print(assert_block_close(to_f64(Y), ref))


def test_block_bf16_blk_sampled():
    """configs[1] single ST block at full size (T=16, S=1024, C=1152) in the bench's launch
    configuration: the oracle computes the spatial stage for every frame and the temporal
    stage + MLP for 24 sampled spatial columns (slice independence)."""
    sh = synth.CONFIGS["blk"]
    xs, Ws = _setup(sh)
    Y = to_f64(_run_block_n1(sh, xs, Ws))
    W = weights_f64(Ws, "bf16")
    y1 = ob.spatial_stage(synth.to_f64(xs, "bf16"), W, sh.NH)
    cols = np.array(sorted(set([0, 1, 127, 128, 511, 1023] + list(np.random.default_rng(0).choice(1024, 18, replace=False)))))
    y = ob.mlp_stage(ob.temporal_stage(y1[:, :, cols], W, sh.NH), W)
    print(assert_block_close(Y[:, :, cols], y))


@pytest.mark.parametrize("dim", ["S", "T"])
def test_stage_attn_public(dim):
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = _setup(sh, seed=3)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, "bf16")
    Out = torch.empty_like(X)
    W = weights_dev(Ws, "bf16")
    st = "s" if dim == "S" else "t"
    fn = ctx.spatial_attn if dim == "S" else ctx.temporal_attn
    fn(shape, X, W[f"w_qkv_{st}"], W[f"w_o_{st}"], X, Out)
    torch.cuda.synchronize()
    Wf = weights_f64(Ws, "bf16")
    x = synth.to_f64(xs, "bf16")
    f = ob.mha_spatial if dim == "S" else ob.mha_temporal
    ref = x + f(x, Wf[f"w_qkv_{st}"], Wf[f"w_o_{st}"], sh.NH)
    print(assert_block_close(to_f64(Out), ref))


def test_block_repeat_run_bitwise():
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = _setup(sh)
    a = bits16(_run_block_n1(sh, xs, Ws))
    b = bits16(_run_block_n1(sh, xs, Ws))
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ virtual ranks
class VirtualGroup:
    """N contexts on one device, each with a private 'symmetric' buffer + signal pad."""

    def __init__(self, N, region_bytes):
        m = dsp()
        self.N = N
        self.ctx = [m.Context(rank=r, world=N) for r in range(N)]
        self.region = [torch.zeros(region_bytes, dtype=torch.uint8, device="cuda") for _ in range(N)]
        self.sig = [torch.zeros(m.SIGNAL_PAD_BYTES // 8, dtype=torch.int64, device="cuda") for _ in range(N)]
        base = [t.data_ptr() for t in self.region]
        sigp = [t.data_ptr() for t in self.sig]
        for c in self.ctx:
            c.set_peer_buffers(base, sigp, region_bytes)
        self.streams = [torch.cuda.Stream() for _ in range(N)]

    def view(self, r, offset, nbytes, dtype):
        return self.region[r][offset:offset + nbytes].view(dtype)

    def run(self, fn):
        cur = torch.cuda.current_stream()
        for s in self.streams:
            s.wait_stream(cur)
        for r in range(self.N):
            with torch.cuda.stream(self.streams[r]):
                fn(r)
        for s in self.streams:
            cur.wait_stream(s)
        torch.cuda.synchronize()


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 2])
def test_switch_p2p_virtual_ranks_bitexact(N, B):
    m = dsp()
    sh = synth.BlockShape(B, 16, 64, 64, 1, "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, 1, "bf16")
    x = synth.make_index_tagged(sh, 9)
    nb = sh.M * 2 // N
    g = VirtualGroup(N, 2 * nb)
    tsh = osw.split(x, osw.DIM_T, N)
    want_s = osw.switch(tsh, osw.DIM_T, osw.DIM_S)
    for r in range(N):
        g.view(r, 0, nb, torch.int16).copy_(torch.from_numpy(tsh[r].view(np.int16).reshape(-1)))
    xin = [g.view(r, 0, nb, torch.bfloat16) for r in range(N)]
    ys = [g.view(r, nb, nb, torch.bfloat16) for r in range(N)]
    g.run(lambda r: g.ctx[r].switch(shape, "T", "S", xin[r], ys[r], impl="p2p"))
    for r in range(N):
        assert np.array_equal(bits16(ys[r]), want_s[r].view(np.int16).reshape(-1)), f"T->S rank {r}"
    # and back: S -> T into the first half
    g.run(lambda r: g.ctx[r].switch(shape, "S", "T", ys[r], xin[r], impl="p2p"))
    for r in range(N):
        assert np.array_equal(bits16(xin[r]), tsh[r].view(np.int16).reshape(-1)), f"S->T rank {r}"


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("impl", ["p2p", "fused"])
@pytest.mark.parametrize("sh", [synth.BlockShape(1, 16, 256, 1152, 16, "bf16"),
                                synth.BlockShape(2, 8, 128, 256, 4, "bf16")])
def test_block_p2p_virtual_ranks_n_invariant(N, impl, sh):
    """DSP block over N virtual ranks == N=1 block bitwise (no reductions cross ranks,
    no split-K: each output's reduction order is independent of N).  `fused`: the switch is
    done by the out-projection / FC2 epilogues storing rows at their owner rank.  B = 2
    exercises the strided (non-identity) row runs of the switch."""
    m = dsp()
    xs, Ws = _setup(sh)
    ref1 = bits16(_run_block_n1(sh, xs, Ws))
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = m.workspace_bytes(shape, N)
    ws = (ws + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    W = weights_dev(Ws, "bf16")
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, X[r], Y[r], impl=impl))
    got = np.concatenate([bits16(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref1.reshape(-1))


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("impl", ["p2p", "fused"])
def test_block_prepared_virtual_ranks_vs_oracle(N, impl):
    """Prepared (LayerNorm-folded) block over N virtual ranks: LN2 statistics are recomputed
    after the switch (rows moved), LN3 from partials; checked against the oracle."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = _setup(sh)
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    W = weights_dev(Ws, "bf16")
    W["prepared"] = g.ctx[0].prepare_block(shape, W)
    torch.cuda.synchronize()
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, X[r], Y[r], impl=impl))
    got = np.concatenate([to_f64(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    print(assert_block_close(got, ref))


def test_block_host_pipelined_equals_device_path():
    """dsp_st_block_forward_host_pipelined (e2e serving path: H2D / block / D2H of adjacent steps
    overlapped on three streams, two staging buffers each way) returns, for every one of five
    different inputs, exactly the bytes of dsp_st_block_forward on device-resident input."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    Ws = synth.make_block_weights(sh, 7)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    W = weights_dev(Ws, sh.dtype)
    W["prepared"] = ctx.prepare_block(shape, W)
    xs = [synth.make_x(sh, 100 + i) for i in range(5)]
    want = []
    for x in xs:
        X = to_dev(x, sh.dtype)
        Y = torch.empty_like(X)
        ctx.st_block_forward(shape, W, X, Y)
        want.append(Y.view(torch.int16).cpu())
    xh = [to_dev(x, sh.dtype).view(torch.int16).cpu().pin_memory() for x in xs]
    yh = [torch.empty_like(t).pin_memory() for t in xh]
    ref = to_dev(xs[0], sh.dtype)
    xd = [torch.empty_like(ref) for _ in range(2)]
    yd = [torch.empty_like(ref) for _ in range(2)]
    ctx.st_block_forward_host_pipelined(shape, W, xh, yh, xd, yd)
    torch.cuda.current_stream().synchronize()
    for i in range(5):
        assert torch.equal(yh[i], want[i]), f"step {i}"
    with pytest.raises(m.DSPError):  # staging buffers must not overlap
        ctx.st_block_forward_host_pipelined(shape, W, xh[:2], yh[:2], [xd[0], xd[1]], [xd[0], yd[1]])


@pytest.mark.parametrize("N", [2, 4])
def test_switch_nd_p2p_virtual_ranks_bitexact(N):
    """dsp_switch_nd through the P2P kernels (virtual ranks) on a 5-D [B, T, H, W, C] activation,
    every ordered pair of sequence dims, bit-exact against the oracle's N-D switch; round trip."""
    m = dsp()
    dims = (2, 8, 8, 16, 64)
    g = (np.arange(int(np.prod(dims)), dtype=np.int64) * 2654435761 % 65521).astype(np.int16).reshape(dims)
    nb = g.nbytes // N
    grp = VirtualGroup(N, 2 * nb)
    for a in range(1, 4):
        for b in range(1, 4):
            if a == b:
                continue
            sh = osw.split_nd(g, a, N)
            want = osw.switch_nd(sh, a, b)
            for r in range(N):
                grp.view(r, 0, nb, torch.int16).copy_(torch.from_numpy(sh[r].reshape(-1)))
            xin = [grp.view(r, 0, nb, torch.int16) for r in range(N)]
            ys = [grp.view(r, nb, nb, torch.int16) for r in range(N)]
            grp.run(lambda r: grp.ctx[r].switch_nd(dims, a, b, xin[r], ys[r], impl="p2p"))
            for r in range(N):
                assert np.array_equal(ys[r].cpu().numpy(), want[r].reshape(-1)), (a, b, r)
            grp.run(lambda r: grp.ctx[r].switch_nd(dims, b, a, ys[r], xin[r], impl="p2p"))
            for r in range(N):
                assert np.array_equal(xin[r].cpu().numpy(), sh[r].reshape(-1)), ("back", a, b, r)


# ------------------------------------------------------------------ N-D block
def _nd_weights(C, nstages, seed, dtype="bf16"):
    """Seeded stage / MLP weights (bf16-representable) as host f64 and device tensors."""
    rng = np.random.default_rng(seed)
    def mk(shape, sc):
        v = rng.uniform(-1, 1, size=shape) * sc
        bits = synth.round_to_bf16_bits(v)
        return synth.bf16_bits_to_f64(bits), to_dev(bits, "bf16")
    st_h, st_d = [], []
    for _ in range(nstages):
        parts = dict(ln_w=mk((C,), 0.1), ln_b=mk((C,), 0.1), w_qkv=mk((3 * C, C), np.sqrt(3 / C)),
                     w_o=mk((C, C), np.sqrt(3 / C)))
        parts["ln_w"] = (parts["ln_w"][0] + 1.0, to_dev(synth.round_to_bf16_bits(parts["ln_w"][0] + 1.0), "bf16"))
        st_h.append({k: v[0] for k, v in parts.items()})
        st_d.append({k: v[1] for k, v in parts.items()})
    m = dict(ln_w=mk((C,), 0.1), ln_b=mk((C,), 0.1), w_fc1=mk((4 * C, C), np.sqrt(3 / C)),
             w_fc2=mk((C, 4 * C), 0.5 * np.sqrt(3 / (4 * C))))
    m["ln_w"] = (m["ln_w"][0] + 1.0, to_dev(synth.round_to_bf16_bits(m["ln_w"][0] + 1.0), "bf16"))
    return st_h, st_d, {k: v[0] for k, v in m.items()}, {k: v[1] for k, v in m.items()}


def test_nd_block_4d_equals_st_block():
    """[B, T, S, C] with attention along S then T, sharded on T: dsp_nd_block_forward is the ST block
    (raw weights), bitwise."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = _setup(sh)
    ref = bits16(_run_block_n1(sh, xs, Ws))
    W = weights_dev(Ws, "bf16")
    stages = [dict(ln_w=W["ln1_w"], ln_b=W["ln1_b"], w_qkv=W["w_qkv_s"], w_o=W["w_o_s"]),
              dict(ln_w=W["ln2_w"], ln_b=W["ln2_b"], w_qkv=W["w_qkv_t"], w_o=W["w_o_t"])]
    mlp = dict(ln_w=W["ln3_w"], ln_b=W["ln3_b"], w_fc1=W["w_fc1"], w_fc2=W["w_fc2"])
    dims = (sh.B, sh.T, sh.S, sh.C)
    ctx = m.Context()
    ctx.ensure_workspace(m.nd_workspace_bytes(dims, "bf16", 1))
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    ctx.nd_block_forward(dims, sh.NH, (2, 1), stages, mlp, 1, X, Y)
    torch.cuda.synchronize()
    assert np.array_equal(bits16(Y), ref)


@pytest.mark.parametrize("axis", [3, 2, 1])
def test_nd_block_5d_single_stage_vs_oracle(axis):
    """[B, T, H, W, C] = [1, 8, 16, 32, 256]: one attention stage along W (spatial-mode packing,
    4 sequences per tile), H (strided, 8 per tile) or T (strided, 16 per tile) + MLP, against
    the float64 oracle at the block gate (R22)."""
    from oracle import block_nd as obn
    m = dsp()
    dims, NH = (1, 8, 16, 32, 256), 4
    st_h, st_d, mlp_h, mlp_d = _nd_weights(dims[-1], 1, 20 + axis)
    xbits = synth.round_to_bf16_bits(np.random.default_rng(axis).uniform(-1, 1, size=dims))
    ctx = m.Context()
    ctx.ensure_workspace(m.nd_workspace_bytes(dims, "bf16", 1))
    X = to_dev(xbits, "bf16")
    Y = torch.empty_like(X)
    ctx.nd_block_forward(dims, NH, (axis,), st_d, mlp_d, 0 if axis != 0 else 1, X, Y)
    torch.cuda.synchronize()
    ref = obn.nd_block(synth.bf16_bits_to_f64(xbits), (axis,), st_h, mlp_h, NH)
    print(assert_block_close(to_f64(Y), ref))


@pytest.mark.parametrize("dims,axis", [((1, 6, 12, 20, 256), 3), ((1, 6, 12, 20, 256), 2), ((2, 51, 4, 4, 256), 1)])
def test_nd_block_ragged_axes_vs_oracle(dims, axis):
    """N-D block stages along axes whose lengths neither divide nor are a multiple of 128
    (W = 20, H = 12, T = 51; R33) + MLP, against the float64 oracle at the block gate."""
    from oracle import block_nd as obn
    m = dsp()
    NH = 4
    st_h, st_d, mlp_h, mlp_d = _nd_weights(dims[-1], 1, 40 + axis)
    xbits = synth.round_to_bf16_bits(np.random.default_rng(axis + 7).uniform(-1, 1, size=dims))
    ctx = m.Context()
    ctx.ensure_workspace(m.nd_workspace_bytes(dims, "bf16", 1))
    X = to_dev(xbits, "bf16")
    Y = torch.empty_like(X)
    ctx.nd_block_forward(dims, NH, (axis,), st_d, mlp_d, 1 if axis != 1 else 2, X, Y)
    torch.cuda.synchronize()
    ref = obn.nd_block(synth.bf16_bits_to_f64(xbits), (axis,), st_h, mlp_h, NH)
    print(assert_block_close(to_f64(Y), ref))


def test_nd_block_5d_vs_oracle_and_virtual_ranks():
    """[B, T, H, W, C] = [1, 8, 16, 32, 256], attention along W, H, T (3 stages), sharded on T:
    N = 1 against the float64 oracle (rel-L2 gate: four residual-stream roundings instead of the
    ST block's three, R32); N = 2, 4 virtual ranks (P2P N-D switches) bitwise equal to N = 1."""
    from oracle import block_nd as obn
    m = dsp()
    dims, NH, order, shard = (1, 8, 16, 32, 256), 4, (3, 2, 1), 1
    C = dims[-1]
    st_h, st_d, mlp_h, mlp_d = _nd_weights(C, 3, 11)
    rng = np.random.default_rng(12)
    xbits = synth.round_to_bf16_bits(rng.uniform(-1, 1, size=dims))
    x64 = synth.bf16_bits_to_f64(xbits)
    ctx = m.Context()
    ctx.ensure_workspace(m.nd_workspace_bytes(dims, "bf16", 1))
    X = to_dev(xbits, "bf16")
    Y = torch.empty_like(X)
    ctx.nd_block_forward(dims, NH, order, st_d, mlp_d, shard, X, Y)
    torch.cuda.synchronize()
    ref = obn.nd_block(x64, order, st_h, mlp_h, NH)
    g = to_f64(Y)
    l2 = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    print(f"3-stage N-D block vs oracle: rel-L2 {l2:.3e}, max-abs {np.abs(g - ref).max():.3e}")
    assert l2 <= 1e-2
    y1 = bits16(Y).reshape(dims)
    for N in (2, 4, 8):
        ws = (m.nd_workspace_bytes(dims, "bf16", N) + 1023) // 1024 * 1024
        act = X.numel() * 2 // N
        g = VirtualGroup(N, ws + act)
        xsh = osw.split_nd(xbits.view(np.int16).reshape(dims), shard, N)
        Xr = [torch.from_numpy(np.ascontiguousarray(xsh[r]).reshape(-1)).cuda().view(torch.bfloat16) for r in range(N)]
        Yr = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
        for r in range(N):
            g.ctx[r].set_workspace(g.region[r][:ws])
        g.run(lambda r: g.ctx[r].nd_block_forward(dims, NH, order, st_d, mlp_d, shard, Xr[r], Yr[r], impl="p2p"))
        got = np.concatenate([bits16(Yr[r]).reshape(osw.split_nd(y1, shard, N)[0].shape) for r in range(N)], axis=shard)
        assert np.array_equal(got, y1), N


# ------------------------------------------------------------------ ST-DiT cross stage
def _cross_setup(sh, Lc, seed=7):
    xs, Ws = _setup(sh, seed)
    Wc = synth.make_cross_weights(sh, seed)
    cx = synth.make_context(sh, seed, Lc)
    W = weights_dev(Ws, "bf16")
    W.update(weights_dev(Wc, "bf16"))
    W["ctx_tokens"] = to_dev(cx, "bf16").view(sh.B, Lc, sh.C)
    Wf = weights_f64(Ws, "bf16")
    Wf.update(weights_f64(Wc, "bf16"))
    return xs, W, Wf, synth.to_f64(cx, "bf16")


@pytest.mark.parametrize("prepared", [False, True])
@pytest.mark.parametrize("Lc", [120, 77])
def test_block_with_cross_stage_vs_oracle(prepared, Lc):
    """The ST-DiT block (SA -> switch -> TA -> cross attention to Lc caption tokens -> MLP -> switch,
    P:137) at N = 1 against the float64 oracle, raw and LayerNorm-folded weights."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, W, Wf, cx = _cross_setup(sh, Lc)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    if prepared:
        W["prepared"] = ctx.prepare_block(shape, W)
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    ctx.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    ref = ob.st_block(synth.to_f64(xs, "bf16"), Wf, sh.NH, cx)
    print(assert_block_close(to_f64(Y), ref))


@pytest.mark.parametrize("prepared", [False, True])
def test_block_with_cross_stage_ragged_lengths(prepared):
    """Block with S = 200 (ragged spatial tiles, R33) and a cross stage whose T * S = 3200
    queries per sample are 25 query tiles (odd: the single-tile kernel on separate views)."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 200, 256, 4, "bf16")
    xs, W, Wf, cx = _cross_setup(sh, 77)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    if prepared:
        W["prepared"] = ctx.prepare_block(shape, W)
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    ctx.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    ref = ob.st_block(synth.to_f64(xs, "bf16"), Wf, sh.NH, cx)
    print(assert_block_close(to_f64(Y), ref))


@pytest.mark.parametrize("N", [2, 4])
def test_block_with_cross_stage_virtual_ranks_n_invariant(N):
    """Cross stage under DSP sharding (local on the S-shards, context replicated): N virtual ranks
    with the fused switch == N = 1, bitwise."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, W, _, _ = _cross_setup(sh, 120)
    ctx1 = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx1.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    ctx1.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    ref1 = bits16(Y)
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    xsh = osw.split(xs, osw.DIM_T, N)
    Xr = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Yr = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, Xr[r], Yr[r], impl="fused"))
    got = np.concatenate([bits16(Yr[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref1.reshape(-1))


@pytest.mark.parametrize("impl", ["p2p", "fused"])
def test_model_prepared_cross_virtual_ranks_n_invariant(impl):
    """dsp_st_model_forward (prepared weights + cross stage, 3 layers) over 2 virtual ranks equals
    the N = 1 model bitwise: at N = 1 LN1 of layers 1.. is folded from the previous FC2 epilogue's
    partials, at N = 2 the same partial bits are recomputed after the S->T switch."""
    m = dsp()
    N, L, Lc = 2, 3, 120
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    prep_ctx = m.Context()
    ctxt = to_dev(synth.make_context(sh, 7, Lc), "bf16").view(sh.B, Lc, sh.C)
    layers = []
    for layer in range(L):
        Ws = synth.make_block_weights(sh, 7, layer=layer)
        Ws.update(synth.make_cross_weights(sh, 7, layer=layer))
        W = weights_dev(Ws, "bf16")
        W["ctx_tokens"] = ctxt
        W["prepared"] = prep_ctx.prepare_block(shape, W)
        layers.append(W)
    xs = synth.make_x(sh, 7)
    c1 = m.Context()
    c1.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, "bf16")
    Y1 = torch.empty_like(X)
    c1.st_model_forward(shape, layers, X, Y1)
    torch.cuda.synchronize()
    ref = bits16(Y1)
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    xsh = osw.split(xs, osw.DIM_T, N)
    Xr = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Yr = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_model_forward(shape, layers, Xr[r], Yr[r], impl=impl))
    got = np.concatenate([bits16(Yr[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref.reshape(-1))


# ---------------------------------------------------------------- temporal TSEQ layout (T >= 64)
TSEQ_SHAPE = synth.BlockShape(1, 64, 128, 1152, 16, "bf16")  # T >= 64, S_loc % 128 == 0, Dh = 72


@pytest.mark.parametrize("prepared", [False, True])
def test_block_tseq_vs_oracle(prepared):
    """T = 64, S = 128: the temporal stage runs on the sequence-major q | k | v layout (the
    temporal QKV GEMM's per-head TMA-box epilogue + contiguous FMHA tiles); full block against
    the float64 oracle at the block gate (R22)."""
    sh = TSEQ_SHAPE
    xs, Ws = _setup(sh)
    got = to_f64(_run_block_n1(sh, xs, Ws, prepared=prepared))
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    print(assert_block_close(got.reshape(ref.shape), ref))


@pytest.mark.parametrize("prepared", [False, True])
def test_block_tseq_equals_token_major_bitwise(prepared):
    """The TSEQ temporal stage (N = 1, S_loc = 128) and the token-major one (N = 2 virtual ranks,
    S_loc = 64 < 128) compute every output with the same arithmetic: the whole blocks are bitwise
    equal (R35: the QKV tile width does not change any bit; the FMHA tiles hold the same rows)."""
    m = dsp()
    sh, N = TSEQ_SHAPE, 2
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
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, X[r], Y[r], impl="p2p"))
    got = np.concatenate([bits16(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref1.reshape(-1))
