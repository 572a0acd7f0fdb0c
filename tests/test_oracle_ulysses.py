"""Pins for oracle/ulysses.py: the DeepSpeed-Ulysses schedule of the ST block (Table 1).

Pinned against things other than the module itself: the unsharded block (its own pins are
torch.nn and brute force), the element-wise index map of the sequence <-> head exchange written
out on index-tagged inputs, the round trip, SPEC's worked ledger number (256 elements at
M = 128, N = 2) and the closed form 8 (N-1) M / N^2 = 4 x DSP (Table 1: 8M/N vs 2M/N).
"""
import numpy as np
import pytest

import synth
from oracle import block as ob
from oracle import sharded, volume
from oracle import ulysses as ou
from oracle.switch import DIM_T, Ledger, split


def _w(sh):
    return {k: synth.to_f64(v, sh.dtype) for k, v in synth.make_block_weights(sh, 7).items()}


def _x(sh):
    return synth.to_f64(synth.make_x(sh, 7), sh.dtype)


@pytest.mark.parametrize("N", [1, 2, 4])
def test_ulysses_equals_unsharded_block(N):
    """Same per-head arithmetic on the same values: equal to st_block up to BLAS row blocking of the
    projections (R27)."""
    sh = synth.BlockShape(1, 8, 16, 32, 4, "f32")
    W, x = _w(sh), _x(sh)
    got, _ = ou.simulate_ulysses(x, W, sh.NH, N, elem_bytes=4)
    np.testing.assert_allclose(got, ob.st_block(x, W, sh.NH), rtol=4e-16 * 16, atol=4e-16 * 16)


def test_ulysses_equals_dsp_schedule():
    sh = synth.BlockShape(2, 4, 8, 16, 4, "f32")
    W, x = _w(sh), _x(sh)
    a, _ = ou.simulate_ulysses(x, W, sh.NH, 2, elem_bytes=4)
    b, _ = sharded.simulate_sharded(x, W, sh.NH, 2, elem_bytes=4)
    np.testing.assert_allclose(a, b, rtol=4e-16 * 16, atol=4e-16 * 16)


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("B", [1, 2])
def test_seq_to_head_index_map_and_round_trip(N, B):
    """Rank g after the exchange holds x[b, t, s, g*C/N + c'] for EVERY token (b, t, s) -- written
    as explicit loops over a sample of the global tensor -- and head_to_seq inverts it."""
    sh = synth.BlockShape(B, 8, 6, 16, 4, "bf16")
    x = synth.make_index_tagged(sh, 3).astype(np.int64)
    C, cn = sh.C, sh.C // N
    parts = split(x, DIM_T, N)
    led = Ledger()
    heads = ou.seq_to_head(parts, sh.NH, led, "q")
    for g in range(N):
        assert heads[g].shape == (B, sh.T, sh.S, cn)
        for b in range(B):
            for t in range(sh.T):
                for s in range(0, sh.S, 2):
                    for c in range(0, cn, 3):
                        assert heads[g][b, t, s, c] == x[b, t, s, g * cn + c]
    back = ou.head_to_seq(heads, led, "o")
    for r in range(N):
        assert np.array_equal(back[r], parts[r])
    per = volume.per_switch_elements(sh.M, N)            # (N-1) M / N^2 per all-to-all
    for r in range(N):
        assert led.sent(r) == 2 * per


def test_ledger_matches_spec_S303_and_table1():
    """B=1, T=4, S=4, D=8 (M = 128), N = 2: 256 elements sent per rank per block, 8
    all-to-alls, and 4x the DSP ledger measured on the same block (64)."""
    sh = synth.BlockShape(1, 4, 4, 8, 2, "f32")
    W, x = _w(sh), _x(sh)
    led = Ledger()
    ou.simulate_ulysses(x, W, sh.NH, 2, led, elem_bytes=4)
    assert led.sent(0) == 256 and led.sent(1) == 256
    assert led.ops(0, "AllToAll") == 8
    led_dsp = Ledger()
    sharded.simulate_sharded(x, W, sh.NH, 2, led_dsp, elem_bytes=4)
    assert led.sent(0) == 4 * led_dsp.sent(0)


@pytest.mark.parametrize("N", [2, 4, 8])
def test_ledger_closed_form(N):
    sh = synth.BlockShape(1, 8, 8, 16, 8, "f32")
    W, x = _w(sh), _x(sh)
    led = Ledger()
    ou.simulate_ulysses(x, W, sh.NH, N, led, elem_bytes=4)
    for r in range(N):
        assert led.sent(r) == volume.predict_volume("ulysses", sh.M, N) == 8 * (N - 1) * sh.M // (N * N)
        assert led.ops(r, "AllToAll") == volume.op_count("ulysses", N)


def test_ulysses_needs_n_dividing_heads():
    sh = synth.BlockShape(1, 4, 4, 12, 3, "f32")
    W, x = _w(sh), _x(sh)
    with pytest.raises(ValueError):
        ou.simulate_ulysses(x, W, sh.NH, 2)
