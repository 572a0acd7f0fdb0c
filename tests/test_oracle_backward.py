"""Pins of oracle/backward.py — CPU only.

Each pin is independent of the oracle's own arithmetic: torch.autograd through a torch.nn
composition in float64 (library code), central finite differences of the forward oracle,
the adjoint identity of the switch (a permutation), and sharded == unsharded.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import backward as bw
from oracle import block as ob
from oracle.switch import DIM_S, DIM_T, split, switch

rng = np.random.default_rng(3)


def _w(sh, seed=7, kappa=1.0):
    return {k: synth.to_f64(v, sh.dtype) for k, v in synth.make_block_weights(sh, seed, kappa=kappa).items()}


def _x(sh, seed=7):
    return synth.to_f64(synth.make_x(sh, seed), sh.dtype)


def _torch_block(tx, T, NH):
    """The block as torch.nn modules (same composition as test_oracle_block's forward pin)."""
    B, Tt, S, C = tx.shape

    def mha(h, wqkv, wo):
        # torch's functional MHA (the nn.MultiheadAttention forward), so wqkv / wo stay autograd leaves
        return F.multi_head_attention_forward(h.transpose(0, 1), h.transpose(0, 1), h.transpose(0, 1), C, NH,
                                              wqkv, None, None, None, False, 0.0, wo, None,
                                              training=False, need_weights=False)[0].transpose(0, 1)

    h = F.layer_norm(tx, (C,), T["ln1_w"], T["ln1_b"], 1e-5).reshape(B * Tt, S, C)
    y1 = tx + mha(h, T["w_qkv_s"], T["w_o_s"]).reshape(B, Tt, S, C)
    h = F.layer_norm(y1, (C,), T["ln2_w"], T["ln2_b"], 1e-5).permute(0, 2, 1, 3).reshape(B * S, Tt, C)
    y2 = y1 + mha(h, T["w_qkv_t"], T["w_o_t"]).reshape(B, S, Tt, C).permute(0, 2, 1, 3)
    h = F.layer_norm(y2, (C,), T["ln3_w"], T["ln3_b"], 1e-5)
    return y2 + F.linear(F.gelu(F.linear(h, T["w_fc1"]), approximate="tanh"), T["w_fc2"])


def test_torch_composition_is_the_forward_oracle():
    sh = synth.BlockShape(1, 4, 8, 24, 3, "f32")
    W, x = _w(sh), _x(sh)
    T = {k: torch.from_numpy(v) for k, v in W.items()}
    with torch.no_grad():
        y = _torch_block(torch.from_numpy(x), T, sh.NH)
    np.testing.assert_allclose(ob.st_block(x, W, sh.NH), y.numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("shape", [(2, 4, 8, 24, 3), (1, 3, 5, 16, 2)])
def test_block_bwd_vs_torch_autograd(shape):
    """dx and all twelve weight gradients vs torch.autograd in float64 (incl. ragged T=3, S=5)."""
    sh = synth.BlockShape(*shape, "f32")
    W, x = _w(sh, kappa=1.5), _x(sh)
    dy = rng.standard_normal(x.shape)
    tx = torch.from_numpy(x).requires_grad_(True)
    T = {k: torch.from_numpy(v.copy()).requires_grad_(True) for k, v in W.items()}
    y = _torch_block(tx, T, sh.NH)
    y.backward(torch.from_numpy(dy))
    dx, grads = bw.st_block_bwd(x, W, sh.NH, dy)
    np.testing.assert_allclose(dx, tx.grad.numpy(), rtol=1e-10, atol=1e-11)
    assert set(grads) == set(bw.GRAD_NAMES)
    for n in bw.GRAD_NAMES:
        np.testing.assert_allclose(grads[n], T[n].grad.numpy(), rtol=1e-10, atol=1e-11, err_msg=n)


def test_pieces_vs_autograd():
    """layer_norm / gelu / attention backward pieces vs torch.autograd (independent library)."""
    z = rng.standard_normal((6, 5, 33)) * 2 + 0.5
    g, b = rng.standard_normal(33), rng.standard_normal(33)
    dy = rng.standard_normal(z.shape)
    tz, tg, tb = (torch.from_numpy(a.copy()).requires_grad_(True) for a in (z, g, b))
    F.layer_norm(tz, (33,), tg, tb, 1e-5).backward(torch.from_numpy(dy))
    dz, dg_, db_ = bw.layer_norm_bwd(z, g, dy)
    for a, t in ((dz, tz), (dg_, tg), (db_, tb)):
        np.testing.assert_allclose(a, t.grad.numpy(), rtol=1e-11, atol=1e-12)
    u = rng.standard_normal(1000) * 4
    du = rng.standard_normal(1000)
    tu = torch.from_numpy(u.copy()).requires_grad_(True)
    F.gelu(tu, approximate="tanh").backward(torch.from_numpy(du))
    np.testing.assert_allclose(bw.gelu_tanh_bwd(u, du), tu.grad.numpy(), rtol=1e-12, atol=1e-13)
    q, k, v, do = (rng.standard_normal((3, 17, 8)) for _ in range(4))
    tq, tk, tv = (torch.from_numpy(a.copy()).requires_grad_(True) for a in (q, k, v))
    F.scaled_dot_product_attention(tq, tk, tv).backward(torch.from_numpy(do))
    for a, t in zip(bw.attention_core_bwd(q, k, v, do), (tq, tk, tv)):
        np.testing.assert_allclose(a, t.grad.numpy(), rtol=1e-11, atol=1e-12)
    # log-sum-exp vs torch.logsumexp of the scaled scores
    a = torch.from_numpy(q) @ torch.from_numpy(k).transpose(-1, -2) / np.sqrt(8)
    np.testing.assert_allclose(bw.attention_lse(q, k), torch.logsumexp(a, -1).numpy(), rtol=1e-13)


def test_block_bwd_finite_differences():
    """Central differences of the FORWARD oracle along random directions (no autograd)."""
    sh = synth.BlockShape(1, 2, 4, 8, 2, "f32")
    W, x = _w(sh, kappa=1.2), _x(sh)
    dy = rng.standard_normal(x.shape)
    dx, grads = bw.st_block_bwd(x, W, sh.NH, dy)
    f = lambda xx, WW: float((ob.st_block(xx, WW, sh.NH) * dy).sum())
    h = 1e-5
    for _ in range(3):
        e = rng.standard_normal(x.shape)
        fd = (f(x + h * e, W) - f(x - h * e, W)) / (2 * h)
        assert abs(fd - (dx * e).sum()) < 1e-7 * max(1.0, abs(fd))
    for n in bw.GRAD_NAMES:
        e = rng.standard_normal(W[n].shape)
        Wp, Wm = dict(W), dict(W)
        Wp[n], Wm[n] = W[n] + h * e, W[n] - h * e
        fd = (f(x, Wp) - f(x, Wm)) / (2 * h)
        assert abs(fd - (grads[n] * e).sum()) < 1e-7 * max(1.0, abs(fd)), n


@pytest.mark.parametrize("N", [2, 4])
def test_switch_adjoint_is_inverse_switch(N):
    """<switch_{T->S}(a), b> = <a, switch_{S->T}(b)>: the switch is a permutation, so the
    backward of a switch is the opposite switch."""
    a = rng.standard_normal((2, 8, 12, 5))
    b = rng.standard_normal((2, 8, 12, 5))
    sa = switch(split(a, DIM_T, N), DIM_T, DIM_S)
    bs = split(b, DIM_S, N)
    lhs = sum(float((sa[r] * bs[r]).sum()) for r in range(N))
    tb = switch(bs, DIM_S, DIM_T)
    at = split(a, DIM_T, N)
    rhs = sum(float((at[r] * tb[r]).sum()) for r in range(N))
    assert abs(lhs - rhs) < 1e-10


@pytest.mark.parametrize("N", [1, 2, 4])
def test_sharded_bwd_equals_unsharded(N):
    """The DSP backward schedule over N ranks (switch adjoints + summed weight gradients)
    equals the unsharded backward."""
    sh = synth.BlockShape(1, 8, 8, 16, 2, "f32")
    W, x = _w(sh), _x(sh)
    dy = rng.standard_normal(x.shape)
    dx_ref, g_ref = bw.st_block_bwd(x, W, sh.NH, dy)
    dx, g, _ = bw.simulate_sharded_bwd(x, W, sh.NH, N, dy)
    np.testing.assert_allclose(dx, dx_ref, rtol=1e-12, atol=1e-13)
    for n in bw.GRAD_NAMES:
        np.testing.assert_allclose(g[n], g_ref[n], rtol=1e-12, atol=1e-13, err_msg=n)


def test_zero_dy_and_zero_weights():
    """dy = 0 gives zero gradients; with zero weights the block is the identity, so dx = dy."""
    sh = synth.BlockShape(1, 2, 4, 8, 2, "f32")
    W, x = _w(sh), _x(sh)
    dx, g = bw.st_block_bwd(x, W, sh.NH, np.zeros_like(x))
    assert not dx.any() and not any(v.any() for v in g.values())
    Z = {k: synth.to_f64(v, "f32") for k, v in synth.zero_block_weights(sh).items()}
    dy = rng.standard_normal(x.shape)
    dx, _ = bw.st_block_bwd(x, Z, sh.NH, dy)
    np.testing.assert_array_equal(dx, dy)
