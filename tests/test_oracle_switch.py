"""Pins for oracle/switch.py: split, gather and the dynamic switch (§3.1)."""
import numpy as np
import pytest

import synth
from oracle import switch as osw
from oracle import volume
from oracle.switch import DIM_S, DIM_T


def _parse(lines):
    return {ln.split(":")[0]: [int(v) for v in ln.split(":")[1].split()] for ln in lines}


def test_spec_worked_example_S151(golden):
    g = _parse(golden("spec_a2a_example.txt"))
    x = np.array(g["global_TS"]).reshape(1, 2, 2, 1)          # [B, T, S, C]
    t = osw.split(x, DIM_T, 2)
    assert t[0].reshape(-1).tolist() == g["tshard_rank0"]
    assert t[1].reshape(-1).tolist() == g["tshard_rank1"]
    s = osw.switch(t, DIM_T, DIM_S)
    assert s[0].reshape(-1).tolist() == g["sshard_rank0"]
    assert s[1].reshape(-1).tolist() == g["sshard_rank1"]


@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("B", [1, 2])
def test_switch_closed_form_index_map(N, B):
    """T->S: XS_q[b, t, s', c] = x[b, t, q*Sn + s', c]; S->T inverse."""
    sh = synth.BlockShape(B, 16, 32, 4, 1, "bf16")
    x = synth.make_index_tagged(sh, 5)
    Tn, Sn = sh.T // N, sh.S // N
    led = osw.Ledger()
    t = osw.split(x, DIM_T, N)
    for r in range(N):
        assert np.array_equal(t[r], x[:, r * Tn:(r + 1) * Tn])
    s = osw.switch(t, DIM_T, DIM_S, led, "t2s")
    for q in range(N):
        # element-by-element closed form, written as explicit loops over a sample
        for b in range(B):
            for tt in range(0, sh.T, 5):
                for sp in range(0, Sn, 3):
                    assert np.array_equal(s[q][b, tt, sp], x[b, tt, q * Sn + sp])
    back = osw.switch(s, DIM_S, DIM_T, led, "s2t")
    for r in range(N):
        assert np.array_equal(back[r], t[r])
    assert np.array_equal(osw.gather(back, DIM_T), x)
    assert np.array_equal(osw.gather(s, DIM_S), x)          # gather agnostic of shard axis
    # ledger: exact per-switch volume, conservation, N=1 -> 0 bytes
    per = volume.per_switch_elements(sh.M, N)
    for r in range(N):
        assert led.sent(r) == 2 * per
    assert sum(e.elements_sent for e in led.entries) == sum(e.elements_recv for e in led.entries)
    if N == 1:
        assert led.sent() == 0


def test_switch_is_pure_permutation_on_multiset():
    sh = synth.BlockShape(1, 8, 8, 4, 1, "bf16")
    x = synth.make_x(sh, 11)
    s = osw.switch(osw.split(x, DIM_T, 4), DIM_T, DIM_S)
    a = np.sort(np.concatenate([v.reshape(-1) for v in s]))
    assert np.array_equal(a, np.sort(x.reshape(-1)))


def test_index_tagged_blk8():
    """Model-shaped switch at blk N=8 (index-only): every token row lands where the map says."""
    sh = synth.BlockShape(1, 16, 1024, 2, 1, "bf16")  # C reduced to the 2 tag channels
    N = 8
    x = synth.make_index_tagged(sh, 1)
    s = osw.switch(osw.split(x, DIM_T, N), DIM_T, DIM_S)
    Sn = sh.S // N
    for q in range(N):
        tag = s[q][..., 0].astype(np.int64) | (s[q][..., 1].astype(np.int64) << 16)
        t_idx = np.arange(sh.T)[:, None]
        s_idx = q * Sn + np.arange(Sn)[None, :]
        assert np.array_equal(tag[0], t_idx * sh.S + s_idx)


def test_errors():
    x = np.zeros((1, 4, 6, 2))
    with pytest.raises(osw.DSPOracleError):
        osw.split(x, DIM_T, 3)
    t = osw.split(x, DIM_T, 2)
    with pytest.raises(osw.DSPOracleError):
        osw.switch(t, DIM_T, DIM_T)
    with pytest.raises(osw.DSPOracleError):
        osw.switch(osw.split(np.zeros((1, 4, 6, 2)), DIM_T, 4), DIM_T, DIM_S)  # 4 does not divide S=6
    with pytest.raises(osw.DSPOracleError):
        osw.split(x, 3, 2)
