"""GPU parity of the building blocks vs the float64 oracle (through the C ABI)."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import block as ob
from tests.gpu_util import assert_block_close, to_dev, to_f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2403_10266_b200 as dsp
    c = dsp.Context()
    c.ensure_workspace(1 << 20)
    return c


def _rand_bf16(shape, seed, scale=1.0, tid=1):
    n = int(np.prod(shape))
    v = synth.uniform_pm1(seed, tid, np.arange(n, dtype=np.uint64)).reshape(shape) * scale
    bits = synth.round_to_bf16_bits(v)
    return bits, synth.bf16_bits_to_f64(bits)


@pytest.mark.parametrize("M,N,K", [(128, 192, 64), (300, 1152, 1152), (16384, 3456, 1152), (2048, 4608, 1152),
                                   (2048, 1152, 4608), (77, 96, 72), (256, 32, 16), (1000, 256, 520),
                                   (333, 288, 200)])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_linear_bf16(ctx, M, N, K, epi):
    import paper_2403_10266_b200 as dsp
    a_bits, a = _rand_bf16((M, K), 1, 1.0, 1)
    w_bits, w = _rand_bf16((N, K), 2, math.sqrt(3.0 / K), 2)
    r_bits, r = _rand_bf16((M, N), 3, 1.0, 3)
    A, W, R = to_dev(a_bits, "bf16"), to_dev(w_bits, "bf16"), to_dev(r_bits, "bf16")
    D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ctx.linear(A, W, D, R if epi == 1 else None, epi)
    torch.cuda.synchronize()
    ref = ob.linear(a, w)
    if epi == 1:
        ref = r + ref
    elif epi == 2:
        ref = ob.gelu_tanh(ref)
    # bf16 output rounding (2^-9 rel) + fp32 accumulation over K
    assert_block_close(to_f64(D), ref, atol=1e-2, rtol=8e-3, rel_l2=5e-3)


def test_linear_f32(ctx):
    M, N, K = 70, 96, 40
    rng = np.random.default_rng(1)
    a, w, r = rng.standard_normal((M, K)), rng.standard_normal((N, K)) / 6, rng.standard_normal((M, N))
    A, W, R = (torch.tensor(t, dtype=torch.float32, device="cuda") for t in (a, w, r))
    for epi in (0, 1, 2):
        D = torch.empty(M, N, dtype=torch.float32, device="cuda")
        ctx.linear(A, W, D, R if epi == 1 else None, epi)
        a32, w32, r32 = (t.astype(np.float32).astype(np.float64) for t in (a, w, r))
        ref = ob.linear(a32, w32)
        ref = r32 + ref if epi == 1 else (ob.gelu_tanh(ref) if epi == 2 else ref)
        np.testing.assert_allclose(to_f64(D), ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("dt,C", [("bf16", 1152), ("bf16", 64), ("f32", 64), ("bf16", 200)])
def test_layer_norm(ctx, dt, C):
    rows = 333
    rng = np.random.default_rng(2)
    x = rng.standard_normal((rows, C)) * 2 + 0.5
    g, b = 1 + 0.1 * rng.standard_normal(C), 0.1 * rng.standard_normal(C)
    if dt == "bf16":
        xs, gs, bs = (synth.round_to_bf16_bits(t) for t in (x, g, b))
        x, g, b = (synth.bf16_bits_to_f64(t) for t in (xs, gs, bs))
    else:
        xs, gs, bs = (t.astype(np.float32) for t in (x, g, b))
        x, g, b = (t.astype(np.float64) for t in (xs, gs, bs))
    X, G, Bt = (to_dev(t, dt) for t in (xs, gs, bs))
    Y = torch.empty_like(X)
    ctx.layer_norm(X, G, Bt, 1e-5, Y)
    torch.cuda.synchronize()
    ref = ob.layer_norm(x, g, b)
    if dt == "bf16":
        assert_block_close(to_f64(Y), ref, atol=1e-2, rtol=8e-3, rel_l2=5e-3)
    else:
        np.testing.assert_allclose(to_f64(Y), ref, rtol=1e-4, atol=1e-4)


def _qkv_case(B, T, S, C, NH, kappa, seed=5):
    """qkv [tok, 3C] bf16 with q scaled so the score std ~ kappa."""
    tok = B * T * S
    _, v = _rand_bf16((tok, 3 * C), seed, 1.0, 4)
    sc = np.ones(3 * C)
    sc[:C] = math.sqrt(3.0) * kappa      # std(q) = kappa
    sc[C:2 * C] = math.sqrt(3.0)         # std(k) = 1  -> std(q.k / sqrt(Dh)) = kappa
    bits = synth.round_to_bf16_bits(v * sc)
    return bits, synth.bf16_bits_to_f64(bits)


def _attn_ref(qkv, B, T, S, C, NH, dim):
    """oracle.attention_core applied to every sequence of the local layout."""
    Dh = C // NH
    g = qkv.reshape(B, T, S, 3 * C)
    out = np.empty((B, T, S, C))
    def run(seq):  # seq [L, 3C]
        q, k, v = ob.split_heads(seq, C, NH)
        return ob.attention_core(q, k, v).transpose(1, 0, 2).reshape(seq.shape[0], C)
    if dim == "S":
        for b in range(B):
            for t in range(T):
                out[b, t] = run(g[b, t])
    else:
        for b in range(B):
            for s in range(S):
                out[b, :, s] = run(g[b, :, s])
    return out.reshape(B * T * S, C)


@pytest.mark.parametrize("B,T,S,C,NH,dim,kappa", [
    (1, 2, 1024, 1152, 16, "S", 1.0),     # spatial blk frame, 8 kv tiles
    (1, 1, 256, 1152, 16, "S", 4.0),      # peaky softmax, lazy rescale path
    (1, 1, 256, 1152, 16, "S", 300.0),    # extreme logits: exp2 arguments far below -126 (poly clamp)
    (2, 3, 128, 256, 4, "S", 1.0),        # Dh=64, one tile
    (1, 5, 16, 128, 8, "S", 1.0),         # S<128: 8 frames per tile, ragged frame count
    (1, 16, 64, 1152, 16, "T", 1.0),      # temporal T=16, 8 columns per tile
    (2, 16, 12, 1152, 16, "T", 4.0),      # ragged column tail, B=2, peaky
    (1, 128, 8, 1152, 16, "T", 1.0),      # long-video T=128, one sequence per tile
    (1, 4, 32, 64, 4, "T", 1.0),          # Dh=16, T=4 -> 32 columns per tile
    (1, 64, 8, 1152, 16, "T", 1.0),       # T=64: two sequences per tile, 64-key windows (two P stores)
    (1, 32, 9, 256, 4, "T", 4.0),         # T=32: four per tile, ragged column tail, peaky
    (1, 3, 64, 256, 4, "S", 1.0),         # S=64 spatial: two frames per tile
    (1, 2, 70, 128, 2, "T", 1.0),         # T=2: 64 sequences per tile (window 32 keys, 2 valid)
])
def test_attention_core_bf16(ctx, B, T, S, C, NH, dim, kappa):
    bits, qkv = _qkv_case(B, T, S, C, NH, kappa)
    Q = to_dev(bits, "bf16")
    O = torch.full((B * T * S, C), float("nan"), dtype=torch.bfloat16, device="cuda")
    ctx.attention_core(B, T, S, C, NH, dim, Q, O)
    torch.cuda.synchronize()
    ref = _attn_ref(qkv, B, T, S, C, NH, dim)
    assert_block_close(to_f64(O), ref, atol=1e-2, rtol=1e-2, rel_l2=1e-2)


@pytest.mark.parametrize("dim", ["S", "T"])
def test_attention_core_f32(ctx, dim):
    B, T, S, C, NH = 1, 4, 16, 64, 4
    rng = np.random.default_rng(3)
    qkv = rng.standard_normal((B * T * S, 3 * C)).astype(np.float32)
    Q = torch.tensor(qkv, device="cuda")
    O = torch.empty(B * T * S, C, dtype=torch.float32, device="cuda")
    ctx.attention_core(B, T, S, C, NH, dim, Q, O)
    torch.cuda.synchronize()
    np.testing.assert_allclose(to_f64(O), _attn_ref(qkv.astype(np.float64), B, T, S, C, NH, dim), rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("B,T,S,Lc,kappa", [(2, 4, 128, 120, 1.0), (1, 2, 256, 77, 1.0), (2, 2, 128, 128, 4.0),
                                             (1, 4, 64, 300, 1.0), (1, 1, 256, 1, 1.0),
                                             (2, 1, 200, 120, 1.0), (1, 3, 128, 77, 1.0), (1, 1, 40, 50, 4.0)])
def test_cross_attention_bf16(ctx, B, T, S, Lc, kappa):
    """dsp_cross_attn vs the oracle: caption-like context lengths 120 / 77 (masked tail
    keys), exactly one tile, three tiles with a ragged last one, a single context token; peaky
    scores at kappa = 4; query counts per sample that are not a multiple of 256 (200: a
    clipped second query tile; 384: an odd tile count, single-tile kernel; 40)."""
    import paper_2403_10266_b200 as dsp
    C, NH = 1152, 16
    tok = B * T * S
    h_bits, h = _rand_bf16((tok, C), 31, 1.0, 1)
    c_bits, cx = _rand_bf16((B * Lc, C), 32, 1.0, 2)
    wq_bits, wq = _rand_bf16((C, C), 33, math.sqrt(3.0 * kappa / C), 3)
    wkv_bits, wkv = _rand_bf16((2 * C, C), 34, math.sqrt(3.0 / C), 4)
    wkv[:C] *= 1.0  # k rows carry the kappa scale through q
    wo_bits, wo = _rand_bf16((C, C), 35, math.sqrt(3.0 / C), 5)
    r_bits, r = _rand_bf16((tok, C), 36, 1.0, 6)
    shape = dsp.make_shape(B, T, S, C, NH, "bf16")
    ctx.ensure_workspace(dsp.cross_workspace_bytes(shape, 1, Lc))
    H, CX, R = to_dev(h_bits, "bf16"), to_dev(c_bits, "bf16"), to_dev(r_bits, "bf16")
    WQ, WKV, WO = to_dev(wq_bits, "bf16"), to_dev(wkv_bits, "bf16"), to_dev(wo_bits, "bf16")
    OUT = torch.empty_like(H)
    ctx.cross_attn(shape, H, CX.view(B, Lc, C), WQ, WKV, WO, R, OUT)
    torch.cuda.synchronize()
    Lq = T * S
    ref = r.copy()
    for b in range(B):
        ref[b * Lq:(b + 1) * Lq] += ob.cross_attention(h[b * Lq:(b + 1) * Lq], cx[b * Lc:(b + 1) * Lc], wq, wkv, wo, NH)
    print(assert_block_close(to_f64(OUT), ref))
