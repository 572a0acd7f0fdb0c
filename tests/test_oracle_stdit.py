"""Pins for oracle.stdit (the rest of P:137's ST-DiT block, R36-R38): each reading is
checked against a special case the definition reduces to, an invariant it must have, or the
sharded schedule -- never against a retyped copy of its own formula."""
import numpy as np
import pytest

import synth
from oracle import block as ob
from oracle import stdit as osd
from oracle import volume as ov

SH = synth.BlockShape(2, 4, 16, 64, 4, "f32")


def _inputs(latte=False, seed=3):
    x = synth.to_f64(synth.make_x(SH, seed), "f32")
    W = {k: synth.to_f64(v, "f32") for k, v in synth.make_block_weights(SH, seed).items()}
    if latte:
        W.update({k: synth.to_f64(v, "f32") for k, v in synth.make_latte_weights(SH, seed).items()})
    return x, W


def _mod(sublayers=("s", "t", "m"), seed=3):
    return {k: tuple(a.astype(np.float64) for a in v) for k, v in synth.make_modulation(SH, seed, sublayers=sublayers).items()}


def test_no_extras_is_the_st_block():
    x, W = _inputs()
    np.testing.assert_array_equal(osd.stdit_block(x, W, SH.NH), ob.st_block(x, W, SH.NH))


def test_neutral_modulation_is_the_st_block():
    """shift = scale = 0, gate = 1: adaLN-Zero reduces to the unconditioned block exactly (R36)."""
    x, W = _inputs()
    z = np.zeros((SH.B, SH.C))
    mod = {k: (z, z, np.ones((SH.B, SH.C))) for k in ("s", "t", "m")}
    np.testing.assert_array_equal(osd.stdit_block(x, W, SH.NH, mod=mod), ob.st_block(x, W, SH.NH))


def test_zero_gates_are_the_identity():
    """The "-Zero" of adaLN-Zero (DiT): with every gate 0 the block returns its input."""
    x, W = _inputs(latte=True)
    mod = {k: (v[0], v[1], np.zeros_like(v[2])) for k, v in _mod(("s", "t", "m", "ms")).items()}
    np.testing.assert_array_equal(osd.stdit_block(x, W, SH.NH, mod=mod), x)


def test_gate_scales_the_branch_linearly():
    """y - x of one sublayer is linear in its gate: gate * 3 -> three times the update."""
    x, W = _inputs()
    m = _mod()
    one = {"s": m["s"]}
    three = {"s": (m["s"][0], m["s"][1], 3.0 * m["s"][2])}
    d1 = osd.spatial_part(x, W, SH.NH, one) - x
    d3 = osd.spatial_part(x, W, SH.NH, three) - x
    np.testing.assert_allclose(d3, 3.0 * d1, rtol=1e-12, atol=1e-13)


def test_modulation_is_per_sample():
    """Sample b's output depends only on sample b's modulation (and input)."""
    x, W = _inputs()
    m = _mod()
    m2 = {k: tuple(a.copy() for a in v) for k, v in m.items()}
    for k in m2:
        for a in m2[k]:
            a[1] += 0.5  # change sample 1 only
    y, y2 = osd.stdit_block(x, W, SH.NH, mod=m), osd.stdit_block(x, W, SH.NH, mod=m2)
    np.testing.assert_array_equal(y[0], y2[0])
    assert not np.allclose(y[1], y2[1])


def test_modulation_folds_into_the_weights():
    """The B = 1 fold (R36): the conditioned block of sample b equals the plain block with
    gamma (1 + scale), beta (1 + scale) + shift and gate-scaled output rows."""
    x, W = _inputs(latte=True)
    m = _mod(("s", "t", "m", "ms"))
    want = osd.stdit_block(x, W, SH.NH, mod=m)
    for b in range(SH.B):
        got = osd.stdit_block(x[b:b + 1], osd.fold_modulation(W, m, b), SH.NH)
        np.testing.assert_allclose(got[0], want[b], rtol=1e-12, atol=1e-12)


def test_zero_latte_mlp_is_the_st_block():
    """R38: with w_fc2_s = 0 the spatial MLP adds nothing."""
    x, W = _inputs(latte=True)
    W["w_fc2_s"] = np.zeros_like(W["w_fc2_s"])
    np.testing.assert_array_equal(osd.stdit_block(x, W, SH.NH), ob.st_block(x, W, SH.NH))


def test_latte_spatial_mlp_is_position_wise():
    """The spatial MLP touches each token alone: permuting the tokens of a frame before the
    spatial MLP permutes its output (no positional terms, R7)."""
    x, W = _inputs(latte=True)
    perm = np.random.default_rng(0).permutation(SH.S)
    f = lambda z: z + ob.mlp(ob.layer_norm(z, W["ln_m_w"], W["ln_m_b"]), W["w_fc1_s"], W["w_fc2_s"])
    np.testing.assert_allclose(f(x[:, :, perm]), f(x)[:, :, perm], rtol=0, atol=1e-13)


def test_zero_pe_is_the_st_block():
    x, W = _inputs()
    np.testing.assert_array_equal(osd.stdit_block(x, W, SH.NH, pe=np.zeros((SH.T, SH.C))), ob.st_block(x, W, SH.NH))


def test_pe_breaks_and_restores_frame_permutation_equivariance():
    """Without pe, permuting the frames permutes the block's output (no positional terms);
    with pe it does so only if the pe rows are permuted along (R37 is a per-frame table)."""
    x, W = _inputs()
    pe = synth.to_f64(synth.make_temporal_pe(SH), "f32")
    perm = np.array([2, 0, 3, 1])
    np.testing.assert_allclose(ob.st_block(x[:, perm], W, SH.NH), ob.st_block(x, W, SH.NH)[:, perm], rtol=0, atol=1e-12)
    y = osd.stdit_block(x, W, SH.NH, pe=pe)
    np.testing.assert_allclose(osd.stdit_block(x[:, perm], W, SH.NH, pe=pe[perm]), y[:, perm], rtol=0, atol=1e-12)
    assert not np.allclose(osd.stdit_block(x[:, perm], W, SH.NH, pe=pe), y[:, perm], atol=1e-6)


def test_pe_table_is_sinusoidal():
    pe = synth.to_f64(synth.make_temporal_pe(SH), "f32")
    np.testing.assert_allclose(pe[0, 0::2], 0.0, atol=0)
    np.testing.assert_allclose(pe[0, 1::2], 1.0, atol=0)
    np.testing.assert_allclose(pe[:, 0], np.sin(np.arange(SH.T)), rtol=1e-6)  # frequency 1 column


@pytest.mark.parametrize("N", [2, 4])
def test_sharded_equals_unsharded_with_everything(N):
    """The DSP schedule with adaLN-Zero, pe and the Latte pair: split -> spatial part on
    the T-shards -> switch -> + pe, temporal, MLP on the S-shards -> switch -> gather equals the
    unsharded block (R27: only BLAS row blocking of the projections may differ)."""
    x, W = _inputs(latte=True)
    m = _mod(("s", "t", "m", "ms"))
    pe = synth.to_f64(synth.make_temporal_pe(SH), "f32")
    np.testing.assert_allclose(osd.simulate_sharded(x, W, SH.NH, N, mod=m, pe=pe),
                               osd.stdit_block(x, W, SH.NH, mod=m, pe=pe), rtol=1e-13, atol=1e-13)


def test_latte_pair_gives_table1_megatron_row():
    """Table 1: Megatron-SP moves 8M per Latte pair (two attention + two MLP layers,
    AG + RS each), DSP 2M/N: the pair does not change DSP's two switches."""
    M, N = 2 ** 20, 8
    assert ov.predict_volume("megatron", M, N, n_attn=2, n_mlp=2) == 2 * 4 * (N - 1) * M // N
    assert ov.predict_volume("dsp", M, N) == 2 * (N - 1) * M // (N * N)
