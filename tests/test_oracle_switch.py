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


# ---------------------------------------------------------------- N-D switch
def _tagged_nd(dims, seed=3):
    """int64 tensor whose every element holds its own global flat index (plus a seeded offset)."""
    return np.arange(int(np.prod(dims)), dtype=np.int64).reshape(dims) * 7 + seed


@pytest.mark.parametrize("dims", [(2, 4, 8, 4, 3), (1, 8, 4, 2, 4, 2), (4, 4, 4, 5)])
@pytest.mark.parametrize("N", [2, 4])
def test_switch_nd_closed_form_all_pairs(dims, N):
    """Every ordered pair (a, b) of non-channel dims: after switch_nd(a -> b), rank q holds exactly
    the elements whose index along b lies in [q*db/N, (q+1)*db/N), in their original relative order
    -- checked element by element from the index tag against the explicit index map."""
    x = _tagged_nd(dims)
    nd = len(dims)
    for a in range(nd - 1):
        for b in range(nd - 1):
            if a == b or dims[a] % N or dims[b] % N:
                continue
            sh = osw.split_nd(x, a, N)
            out = osw.switch_nd(sh, a, b)
            nb = dims[b] // N
            for q in range(N):
                got = out[q]
                exp_shape = list(dims)
                exp_shape[b] = nb
                assert list(got.shape) == exp_shape
                # decode every element's global index and compare with the map (i_b = q*nb + local i_b)
                flat = (got - 3) // 7
                idx = np.array(np.unravel_index(flat.reshape(-1), dims)).T.reshape(*got.shape, nd)
                loc = np.indices(got.shape).transpose(*range(1, nd + 1), 0)
                want = loc.copy()
                want[..., b] += q * nb
                assert np.array_equal(idx, want), (a, b, q)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_switch_nd_equals_4d_switch_and_round_trips(N):
    sh = synth.BlockShape(2, 16, 32, 4, 1, "bf16")
    x = synth.make_index_tagged(sh, 5)
    t = osw.split(x, DIM_T, N)
    assert all(np.array_equal(u, v) for u, v in zip(osw.switch_nd(t, 1, 2), osw.switch(t, DIM_T, DIM_S)))
    dims = (2, 8, 8, 8, 4)
    g = _tagged_nd(dims)
    if N > 8 or 8 % N:
        return
    s0 = osw.split_nd(g, 1, N)
    back = osw.switch_nd(osw.switch_nd(s0, 1, 3), 3, 1)
    assert all(np.array_equal(u, v) for u, v in zip(back, s0))
    # composition: 1 -> 2 -> 3 equals 1 -> 3
    via = osw.switch_nd(osw.switch_nd(s0, 1, 2), 2, 3)
    direct = osw.switch_nd(s0, 1, 3)
    assert all(np.array_equal(u, v) for u, v in zip(via, direct))


@pytest.mark.parametrize("N", [2, 4, 8])
def test_switch_nd_ledger_volume(N):
    """Off-rank elements sent per rank per switch = (N-1) M / N^2 for any pair of dims."""
    dims = (1, 8, 16, 8, 4)
    M = int(np.prod(dims))
    x = np.zeros(dims, dtype=np.int16)
    for a, b in [(1, 2), (3, 1), (2, 3)]:
        led = osw.Ledger()
        osw.switch_nd(osw.split_nd(x, a, N), a, b, led, "t")
        for r in range(N):
            assert led.sent(r) == (N - 1) * M // (N * N)


def test_switch_nd_errors():
    x = np.zeros((2, 4, 4, 3))
    with pytest.raises(osw.DSPOracleError):
        osw.split_nd(x, 3, 2)          # the channel dim is never sharded
    with pytest.raises(osw.DSPOracleError):
        osw.switch_nd(osw.split_nd(x, 1, 2), 1, 1)
    with pytest.raises(osw.DSPOracleError):
        osw.switch_nd(osw.split_nd(x, 1, 2), 1, 3)
