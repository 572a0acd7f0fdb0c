"""Pins for oracle/block_nd.py (the multi-dimensional block, and its DSP schedule)."""
import numpy as np
import pytest

import synth
from oracle import block as ob
from oracle import block_nd as obn
from oracle import switch as osw


def _weights(C, nstages, seed=3):
    rng = np.random.default_rng(seed)
    u = lambda *s, sc=1.0: rng.uniform(-1, 1, size=s) * sc
    stages = [dict(ln_w=1 + 0.1 * u(C), ln_b=0.1 * u(C), w_qkv=u(3 * C, C, sc=np.sqrt(3 / C)),
                   w_o=u(C, C, sc=np.sqrt(3 / C))) for _ in range(nstages)]
    Wm = dict(ln_w=1 + 0.1 * u(C), ln_b=0.1 * u(C), w_fc1=u(4 * C, C, sc=np.sqrt(3 / C)),
              w_fc2=u(C, 4 * C, sc=0.5 * np.sqrt(3 / (4 * C))))
    return stages, Wm


def test_nd_block_with_two_dims_is_the_st_block():
    """order = (S, T) on [B, T, S, C] reproduces the (separately pinned) ST block exactly."""
    sh = synth.BlockShape(2, 4, 8, 16, 2, "f32")
    x = synth.to_f64(synth.make_x(sh, 4), "f32")
    W = {k: synth.to_f64(v, "f32") for k, v in synth.make_block_weights(sh, 4).items()}
    stages = [dict(ln_w=W["ln1_w"], ln_b=W["ln1_b"], w_qkv=W["w_qkv_s"], w_o=W["w_o_s"]),
              dict(ln_w=W["ln2_w"], ln_b=W["ln2_b"], w_qkv=W["w_qkv_t"], w_o=W["w_o_t"])]
    Wm = dict(ln_w=W["ln3_w"], ln_b=W["ln3_b"], w_fc1=W["w_fc1"], w_fc2=W["w_fc2"])
    assert np.array_equal(obn.nd_block(x, (2, 1), stages, Wm, sh.NH), ob.st_block(x, W, sh.NH))


def test_mha_along_brute_force_axis():
    """mha_along(axis=2) on [B, T, H, W, C] == explicit loops over (b, t, w) of mha_sequence."""
    C, NH = 8, 2
    x = np.random.default_rng(1).normal(size=(1, 2, 4, 3, C))
    stages, _ = _weights(C, 1)
    got = obn.mha_along(x, stages[0]["w_qkv"], stages[0]["w_o"], NH, 2)
    for t in range(2):
        for w in range(3):
            want = ob.mha_sequence(x[0, t, :, w], stages[0]["w_qkv"], stages[0]["w_o"], NH)
            assert np.allclose(got[0, t, :, w], want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("N", [1, 2, 4])
def test_nd_dsp_schedule_equals_unsharded(N):
    """[B, T, H, W, C], attention along W, H, T; sharded on T: the DSP schedule over N simulated
    ranks (two N-D switches) equals the unsharded block (same per-sequence function on the same
    bytes; the MLP's BLAS row blocking may differ in the last bit, R27)."""
    C, NH = 16, 2
    dims = (1, 4, 4, 8, C)
    x = np.random.default_rng(2).uniform(-1, 1, size=dims)
    stages, Wm = _weights(C, 3)
    order = (3, 2, 1)
    want = obn.nd_block(x, order, stages, Wm, NH)
    led = osw.Ledger()
    got = obn.simulate_sharded_nd(x, order, stages, Wm, NH, N, 1, led)
    np.testing.assert_allclose(np.concatenate(got, axis=1), want, rtol=0, atol=1e-12)
    M = int(np.prod(dims))
    for r in range(N):
        assert led.ops(r) == 2                             # two switches per block
        assert led.sent(r) == 2 * (N - 1) * M // (N * N)


def test_nd_slice_independence():
    """Stage along axis k: perturbing the input at other positions of the OTHER dims does not change
    the output of an untouched sequence (the DSP premise P:93)."""
    C, NH = 8, 2
    x = np.random.default_rng(5).normal(size=(1, 3, 4, 4, C))
    stages, _ = _weights(C, 1)
    y = obn.attn_stage(x, stages[0], NH, 2)
    x2 = x.copy()
    x2[0, 1] += 1.0        # another T index
    x2[0, :, :, 3] -= 2.0  # another W index
    y2 = obn.attn_stage(x2, stages[0], NH, 2)
    assert np.array_equal(y[0, 0, :, :3], y2[0, 0, :, :3])
