"""Pins for oracle/block.py and oracle/sharded.py against things other than themselves.

* torch.nn library modules in float64 (LayerNorm, GELU(tanh), MultiheadAttention,
  scaled_dot_product_attention) — independent code with the same definitions;
* brute-force scalar loops from the formulas on tiny shapes;
* closed forms (extent-1 attention, uniform softmax, zero weights);
* invariants (permutation equivariance, slice independence — the DSP premise P:93,
  sharded == unsharded, MLP/switch commutation R14).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import block as ob
from oracle import sharded
from oracle.switch import DIM_S, DIM_T, split, switch

rng = np.random.default_rng(0)


def _w(sh, seed=7, kappa=1.0):
    return {k: synth.to_f64(v, sh.dtype) for k, v in synth.make_block_weights(sh, seed, kappa=kappa).items()}


def _x(sh, seed=7):
    return synth.to_f64(synth.make_x(sh, seed), sh.dtype)


def test_layer_norm_vs_torch():
    z = rng.standard_normal((5, 7, 33)) * 3 + 1
    g, b = rng.standard_normal(33), rng.standard_normal(33)
    ref = F.layer_norm(torch.from_numpy(z), (33,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5).numpy()
    np.testing.assert_allclose(ob.layer_norm(z, g, b), ref, rtol=0, atol=1e-12)
    n = ob.layer_norm(z, np.ones(33), np.zeros(33))
    np.testing.assert_allclose(n.mean(-1), 0, atol=1e-12)
    np.testing.assert_allclose(n.var(-1), 1, atol=1e-4)       # var/(var+eps)


def test_gelu_vs_torch_and_closed_form():
    u = np.linspace(-8, 8, 1001)
    ref = F.gelu(torch.from_numpy(u), approximate="tanh").numpy()
    np.testing.assert_allclose(ob.gelu_tanh(u), ref, rtol=0, atol=1e-14)
    assert ob.gelu_tanh(np.array([0.0]))[0] == 0.0
    assert abs(ob.gelu_tanh(np.array([20.0]))[0] - 20.0) < 1e-12


def test_attention_core_vs_sdpa_and_bruteforce():
    q, k, v = (rng.standard_normal((3, 9, 8)) for _ in range(3))
    got = ob.attention_core(q, k, v)
    ref = F.scaled_dot_product_attention(*(torch.from_numpy(t) for t in (q, k, v))).numpy()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    # brute force scalar loops
    H, L, D = q.shape
    for h in range(H):
        for i in range(L):
            s = [sum(q[h, i, d] * k[h, j, d] for d in range(D)) / math.sqrt(D) for j in range(L)]
            m = max(s)
            e = [math.exp(x - m) for x in s]
            z = sum(e)
            for d in range(D):
                o = sum(e[j] / z * v[h, j, d] for j in range(L))
                assert abs(o - got[h, i, d]) < 1e-12


def test_mha_sequence_vs_torch_multiheadattention():
    """nn.MultiheadAttention with in_proj_weight = w_qkv ([q|k|v] rows, R8), out_proj = w_o."""
    L, C, NH = 11, 24, 3
    h = rng.standard_normal((L, C))
    wqkv = rng.standard_normal((3 * C, C)) / math.sqrt(C)
    wo = rng.standard_normal((C, C)) / math.sqrt(C)
    m = torch.nn.MultiheadAttention(C, NH, bias=False, batch_first=True, dtype=torch.float64)
    with torch.no_grad():
        m.in_proj_weight.copy_(torch.from_numpy(wqkv))
        m.out_proj.weight.copy_(torch.from_numpy(wo))
        th = torch.from_numpy(h)[None]
        ref = m(th, th, th, need_weights=False)[0][0].numpy()
    np.testing.assert_allclose(ob.mha_sequence(h, wqkv, wo, NH), ref, rtol=0, atol=1e-12)


def test_mha_bruteforce_tiny():
    L, C, NH = 3, 4, 2
    Dh = C // NH
    h = rng.standard_normal((L, C))
    wqkv = rng.standard_normal((3 * C, C))
    wo = rng.standard_normal((C, C))
    G = [[sum(h[i, c] * wqkv[o, c] for c in range(C)) for o in range(3 * C)] for i in range(L)]
    O = [[0.0] * C for _ in range(L)]
    for j in range(NH):
        for i in range(L):
            s = [sum(G[i][j * Dh + d] * G[kk][C + j * Dh + d] for d in range(Dh)) / math.sqrt(Dh) for kk in range(L)]
            m = max(s)
            e = [math.exp(a - m) for a in s]
            z = sum(e)
            for d in range(Dh):
                O[i][j * Dh + d] = sum(e[kk] / z * G[kk][2 * C + j * Dh + d] for kk in range(L))
    want = [[sum(O[i][c] * wo[o, c] for c in range(C)) for o in range(C)] for i in range(L)]
    np.testing.assert_allclose(ob.mha_sequence(h, wqkv, wo, NH), np.array(want), rtol=0, atol=1e-11)


def test_extent1_and_uniform_softmax_closed_forms():
    C, NH = 16, 4
    wqkv = rng.standard_normal((3 * C, C))
    wo = rng.standard_normal((C, C))
    h1 = rng.standard_normal((1, C))
    # L = 1: softmax of one score is 1 -> output = (h Wv^T) Wo^T
    np.testing.assert_allclose(ob.mha_sequence(h1, wqkv, wo, NH), h1 @ wqkv[2 * C:].T @ wo.T, atol=1e-12)
    # Wk = 0: all scores equal -> each head outputs the sequence mean of V
    w0 = wqkv.copy()
    w0[C:2 * C] = 0
    h = rng.standard_normal((7, C))
    vmean = (h @ wqkv[2 * C:].T).mean(0, keepdims=True)
    np.testing.assert_allclose(ob.mha_sequence(h, w0, wo, NH), np.repeat(vmean @ wo.T, 7, 0), atol=1e-12)


def test_permutation_equivariance():
    C, NH, L = 16, 2, 9
    wqkv, wo = rng.standard_normal((3 * C, C)), rng.standard_normal((C, C))
    h = rng.standard_normal((L, C))
    p = rng.permutation(L)
    np.testing.assert_allclose(ob.mha_sequence(h[p], wqkv, wo, NH), ob.mha_sequence(h, wqkv, wo, NH)[p], atol=1e-12)


def test_slice_independence_dsp_premise():
    """spatial computation is independent of the temporal dim (and vice versa)."""
    sh = synth.BlockShape(1, 4, 8, 16, 2, "f32")
    W = _w(sh)
    x = _x(sh)
    y = ob.spatial_stage(x, W, sh.NH)
    x2 = x.copy()
    x2[:, 1:] = rng.standard_normal(x2[:, 1:].shape)
    assert np.array_equal(ob.spatial_stage(x2, W, sh.NH)[:, 0], y[:, 0])
    yt = ob.temporal_stage(x, W, sh.NH)
    x3 = x.copy()
    x3[:, :, 1:] = rng.standard_normal(x3[:, :, 1:].shape)
    assert np.array_equal(ob.temporal_stage(x3, W, sh.NH)[:, :, 0], yt[:, :, 0])


def test_zero_weights_identity_and_shape():
    sh = synth.BlockShape(1, 4, 8, 16, 2, "f32")
    W = {k: synth.to_f64(v, "f32") for k, v in synth.zero_block_weights(sh).items()}
    x = _x(sh)
    assert np.array_equal(ob.st_block(x, W, sh.NH), x)


def test_block_vs_torch_composition():
    """Whole block vs torch.nn modules in float64 (independent library code)."""
    sh = synth.BlockShape(2, 4, 8, 24, 3, "f32")
    W = _w(sh)
    x = _x(sh)
    C = sh.C
    tx = torch.from_numpy(x)
    T = {k: torch.from_numpy(v) for k, v in W.items()}

    def mha(h, wqkv, wo):
        m = torch.nn.MultiheadAttention(C, sh.NH, bias=False, batch_first=True, dtype=torch.float64)
        with torch.no_grad():
            m.in_proj_weight.copy_(wqkv)
            m.out_proj.weight.copy_(wo)
            return m(h, h, h, need_weights=False)[0]

    with torch.no_grad():
        B, Tt, S = sh.B, sh.T, sh.S
        h = F.layer_norm(tx, (C,), T["ln1_w"], T["ln1_b"], 1e-5).reshape(B * Tt, S, C)
        y1 = tx + mha(h, T["w_qkv_s"], T["w_o_s"]).reshape(B, Tt, S, C)
        h = F.layer_norm(y1, (C,), T["ln2_w"], T["ln2_b"], 1e-5).permute(0, 2, 1, 3).reshape(B * S, Tt, C)
        y2 = y1 + mha(h, T["w_qkv_t"], T["w_o_t"]).reshape(B, S, Tt, C).permute(0, 2, 1, 3)
        h = F.layer_norm(y2, (C,), T["ln3_w"], T["ln3_b"], 1e-5)
        y = y2 + F.linear(F.gelu(F.linear(h, T["w_fc1"]), approximate="tanh"), T["w_fc2"])
    np.testing.assert_allclose(ob.st_block(x, W, sh.NH), y.numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("N", [1, 2, 4])
def test_sharded_equals_unsharded_bitexact(N):
    """simulate_sharded(x, W, N) == st_block(x, W) (same per-sequence code on the same bytes)."""
    sh = synth.BlockShape(1, 8, 16, 32, 4, "f32")
    W, x = _w(sh), _x(sh)
    ref = ob.st_block(x, W, sh.NH)
    got, _ = sharded.simulate_sharded(x, W, sh.NH, N, elem_bytes=4)
    # Attention stages are bit-exact (identical per-sequence code on identical bytes);
    # the position-wise MLP goes through BLAS with a different row count per call, which
    # changes the last bit only.
    np.testing.assert_allclose(got, ref, rtol=4e-16 * 8, atol=4e-16 * 8)
    y1 = ob.spatial_stage(x, W, sh.NH)
    assert np.array_equal(np.concatenate([ob.spatial_stage(s, W, sh.NH) for s in split(x, DIM_T, N)], 1), y1)
    y2 = ob.temporal_stage(y1, W, sh.NH)
    assert np.array_equal(np.concatenate([ob.temporal_stage(s, W, sh.NH) for s in split(y1, DIM_S, N)], 2), y2)


def test_mlp_switch_commutation_R14():
    sh = synth.BlockShape(1, 4, 8, 16, 2, "f32")
    W, x = _w(sh), _x(sh)
    a, _ = sharded.simulate_sharded(x, W, sh.NH, 2, mlp_before_switch=True)
    b, _ = sharded.simulate_sharded(x, W, sh.NH, 2, mlp_before_switch=False)
    assert np.array_equal(a, b)


def test_acceptance_grid_tiny():
    """SPEC acceptance-style grid at the tiny config shape (T=4,S=16,C=64,NH=4), N in {1,2,4}."""
    sh = synth.CONFIGS["tiny"]
    W, x = _w(sh), _x(sh)
    ref = ob.st_block(x, W, sh.NH)
    for N in (1, 2, 4):
        got, _ = sharded.simulate_sharded(x, W, sh.NH, N, elem_bytes=4)
        np.testing.assert_allclose(got, ref, rtol=1e-14, atol=1e-14)
