"""GPU coverage of the other BASELINE.json configs:

* configs[3] long video (T=128, S=4096): kernel-level parity at the long shapes (spatial
  attention over S=4096 = 32 KV tiles through the two-tile kernel; temporal attention over
  T=128, one sequence per tile) against the oracle's attention on the GPU's own q/k/v, and
  the full-size block forward (1.2 GB activation) run to completion with finite output and
  repeat-run determinism;
* configs[2] 28-layer ST-DiT-XL/2 shape: 28 blocks with per-layer weights (tensor ids
  16*l + 1 + k), checked per layer teacher-forced at l = 0, 13, 27 (oracle block applied to
  the GPU's layer-l input, spatial stage for all frames, temporal stage + MLP on sampled
  columns), end-to-end drift reported.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import block as ob
from tests.gpu_util import assert_block_close, bits16, to_dev, to_f64, weights_dev, weights_f64

pytestmark = pytest.mark.gpu


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _attn_ref_rows(qkv, B, T, S, C, NH, dim, seqs):
    """oracle.attention_core for the listed sequences only (slice independence)."""
    g = qkv.reshape(B, T, S, 3 * C)
    out = {}
    for sq in seqs:
        seq = g[0, sq] if dim == "S" else g[0, :, sq]
        q, k, v = ob.split_heads(seq, C, NH)
        out[sq] = ob.attention_core(q, k, v).transpose(1, 0, 2).reshape(seq.shape[0], C)
    return out


@pytest.mark.parametrize("dim,T,S,seqs", [("S", 2, 4096, [0, 1]), ("T", 128, 64, [0, 17, 63])])
def test_attention_core_long_video_shapes(dim, T, S, seqs):
    m = dsp()
    C, NH = 1152, 16
    tok = T * S
    rng = np.random.default_rng(11)
    v = rng.uniform(-1, 1, size=(tok, 3 * C))
    v[:, :C] *= np.sqrt(3.0)
    v[:, C:2 * C] *= np.sqrt(3.0)
    bits = synth.round_to_bf16_bits(v)
    qkv = synth.bf16_bits_to_f64(bits)
    ctx = m.Context()
    Q = to_dev(bits, "bf16")
    O = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
    ctx.attention_core(1, T, S, C, NH, dim, Q, O)
    torch.cuda.synchronize()
    got = to_f64(O).reshape(1, T, S, C)
    ref = _attn_ref_rows(qkv, 1, T, S, C, NH, dim, seqs)
    for sq, r in ref.items():
        g = got[0, sq] if dim == "S" else got[0, :, sq]
        assert_block_close(g, r, atol=1e-2, rtol=1e-2, rel_l2=1e-2)


def test_block_long_video_full_size_runs():
    """configs[3] at N=1: the whole 1.2 GB activation through the block; finite and repeatable."""
    m = dsp()
    sh = synth.CONFIGS["long"]
    x = to_dev(synth.make_x(sh, 7), "bf16")
    W = weights_dev(synth.make_block_weights(sh, 7), "bf16")
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    y1 = torch.empty_like(x)
    y2 = torch.empty_like(x)
    ctx.st_block_forward(shape, W, x, y1)
    ctx.st_block_forward(shape, W, x, y2)
    torch.cuda.synchronize()
    assert torch.isfinite(y1.float()).all()
    assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))
    assert 0.2 < float(y1.float().std()) < 5.0


def test_28_layer_teacher_forced():
    """configs[2] shape: 28 blocks, per-layer parity teacher-forced at l = 0, 13, 27."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 1024, 1152, 16, "bf16")
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    x = to_dev(synth.make_x(sh, 7), "bf16")
    check = {0, 13, 27}
    inputs = {}
    layers_w = {}
    cur = x
    for layer in range(28):
        Ws = synth.make_block_weights(sh, 7, layer=layer)
        if layer in check:
            inputs[layer] = cur.clone()
            layers_w[layer] = Ws
        nxt = torch.empty_like(cur)
        ctx.st_block_forward(shape, weights_dev(Ws, "bf16"), cur, nxt)
        cur = nxt
    torch.cuda.synchronize()
    assert torch.isfinite(cur.float()).all()
    cols = np.array([0, 5, 511, 1023])
    for layer in sorted(check):
        xin = to_f64(inputs[layer])
        W = weights_f64(layers_w[layer], "bf16")
        y1 = ob.spatial_stage(xin, W, sh.NH)
        want = ob.mlp_stage(ob.temporal_stage(y1[:, :, cols], W, sh.NH), W)
        # the GPU's output of this layer = input of the next (or the final output)
        got_t = inputs[layer + 1] if layer + 1 in inputs else None
        if got_t is None:
            # recompute this layer's GPU output from its GPU input
            out = torch.empty_like(inputs[layer])
            ctx.st_block_forward(shape, weights_dev(layers_w[layer], "bf16"), inputs[layer], out)
            torch.cuda.synchronize()
            got_t = out
        print(f"layer {layer}:", assert_block_close(to_f64(got_t)[:, :, cols], want))


def test_model_forward_chained_layernorm():
    """dsp_st_model_forward over L = 3 prepared blocks (LN1 of blocks 1, 2 folded from the previous
    block's FC2 partials): L = 1 equals the block bitwise; L = 3 against the float64 oracle chained
    over the same three layers' weights."""
    m = dsp()
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    xs = synth.make_x(sh, 7)
    x = to_dev(xs, "bf16")
    layers = [synth.make_block_weights(sh, 7, layer=l) for l in range(3)]
    W = []
    for Ws in layers:
        w = weights_dev(Ws, "bf16")
        w["prepared"] = ctx.prepare_block(shape, w)
        W.append(w)
    y_model, y_block = torch.empty_like(x), torch.empty_like(x)
    ctx.st_model_forward(shape, W[:1], x, y_model)
    ctx.st_block_forward(shape, W[0], x, y_block)
    torch.cuda.synchronize()
    assert torch.equal(y_model.view(torch.int16), y_block.view(torch.int16))
    y = torch.empty_like(x)
    ctx.st_model_forward(shape, W, x, y)
    # the same three blocks as separate calls (LN1 statistics from the row-statistics pass)
    cur = x
    for w in W:
        nxt = torch.empty_like(x)
        ctx.st_block_forward(shape, w, cur, nxt)
        cur = nxt
    torch.cuda.synchronize()
    # only the LN1 statistics' source differs (fp32 combination of per-tile partials vs a two-pass
    # sum, equal to ~1e-6 relative); the bf16 pipeline re-rounds downstream, so the two outputs
    # differ at the level of the bf16 noise itself (measured rel-L2 2.7e-3), not bitwise
    g, c = to_f64(y), to_f64(cur)
    l2 = np.linalg.norm(g - c) / np.linalg.norm(c)
    print(f"model vs 3 block calls: rel-L2 {l2:.3e}")
    assert l2 <= 1e-2
    # against the oracle: bf16 storage error compounds over layers (multi-layer
    # drift is reported, the gate is per layer), so only the rel-L2 gate applies here
    ref = synth.to_f64(xs, "bf16")
    for Ws in layers:
        ref = ob.st_block(ref, weights_f64(Ws, "bf16"), sh.NH)
    g = to_f64(y)
    l2 = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    print(f"3 layers vs oracle: rel-L2 {l2:.3e}, max-abs {np.abs(g - ref).max():.3e}")
    assert l2 <= 1e-2


def test_block_long_video_virtual_ranks_n_invariant():
    """configs[3] at full size (T=128, S=4096, 1.2 GB activation) over N = 2 virtual ranks with the
    fused switch: bitwise equal to the N = 1 block (the long-video shapes through every kernel,
    incl. the 32-tile spatial sequences and one-tile temporal sequences)."""
    from tests.test_gpu_block import VirtualGroup
    from oracle import switch as osw
    m = dsp()
    sh = synth.CONFIGS["long"]
    xs = synth.make_x(sh, 7)
    W = weights_dev(synth.make_block_weights(sh, 7), "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx = m.Context()
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, "bf16")
    Y1 = torch.empty_like(X)
    ctx.st_block_forward(shape, W, X, Y1)
    torch.cuda.synchronize()
    ref1 = bits16(Y1).reshape(-1)
    del ctx, X, Y1
    torch.cuda.empty_cache()
    N = 2
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
    assert np.array_equal(got.reshape(-1), ref1)


@pytest.mark.parametrize("N,impl", [(8, "fused"), (8, "p2p"), (4, "fused")])
def test_blk_full_shape_virtual_ranks_n_invariant(N, impl):
    """configs[1] (the bench's single block, S = 1024) at the N = 4 / 8 shard shapes the north star
    targets (tok_r = 4096 / 2048), N virtual ranks, prepared weights, against the N = 1 prepared
    block: LN2 statistics are recomputed after the switch at N > 1 (partials at N = 1), so the
    comparison is within the block gate (measured rel-L2 8.6e-4) rather than bitwise; the raw
    path's bitwise N-invariance is covered at S = 256 in test_gpu_block.py."""
    from tests.test_gpu_block import VirtualGroup
    from oracle import switch as osw
    m = dsp()
    sh = synth.CONFIGS["blk"]
    xs = synth.make_x(sh, 7)
    W = weights_dev(synth.make_block_weights(sh, 7), "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx = m.Context()
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    W["prepared"] = ctx.prepare_block(shape, W)
    X = to_dev(xs, "bf16")
    Y1 = torch.empty_like(X)
    ctx.st_block_forward(shape, W, X, Y1)
    torch.cuda.synchronize()
    ref = to_f64(Y1)
    ws = (m.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    xsh = osw.split(xs, osw.DIM_T, N)
    Xr = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Yr = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, W, Xr[r], Yr[r], impl=impl))
    got = np.concatenate([to_f64(Yr[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    print(assert_block_close(got, ref.reshape(got.shape), atol=2e-2, rtol=1e-2, rel_l2=5e-3))
