"""Pins for oracle.block.cross_attention / cross_stage (ST-DiT's cross attention)."""
import numpy as np
import pytest
import torch

from oracle import block as ob


def _w(C, seed):
    rng = np.random.default_rng(seed)
    s = np.sqrt(3.0 / C)
    return (rng.uniform(-1, 1, (C, C)) * s, rng.uniform(-1, 1, (2 * C, C)) * s, rng.uniform(-1, 1, (C, C)) * s)


@pytest.mark.parametrize("L,Lc,C,NH", [(16, 7, 32, 4), (5, 12, 24, 2)])
def test_cross_attention_vs_torch_mha(L, Lc, C, NH):
    """torch.nn.MultiheadAttention in float64 (in_proj = [w_q | w_k | w_v], no bias)."""
    wq, wkv, wo = _w(C, 1)
    rng = np.random.default_rng(2)
    h, ctx = rng.normal(size=(L, C)), rng.normal(size=(Lc, C))
    mha = torch.nn.MultiheadAttention(C, NH, bias=False, batch_first=True, dtype=torch.float64)
    with torch.no_grad():
        mha.in_proj_weight.copy_(torch.from_numpy(np.concatenate([wq, wkv])))
        mha.out_proj.weight.copy_(torch.from_numpy(wo))
        want = mha(torch.from_numpy(h)[None], torch.from_numpy(ctx)[None], torch.from_numpy(ctx)[None],
                   need_weights=False)[0][0].numpy()
    np.testing.assert_allclose(ob.cross_attention(h, ctx, wq, wkv, wo, NH), want, rtol=0, atol=1e-12)


def test_cross_attention_brute_force():
    C, NH, L, Lc = 8, 2, 3, 4
    wq, wkv, wo = _w(C, 3)
    rng = np.random.default_rng(4)
    h, ctx = rng.normal(size=(L, C)), rng.normal(size=(Lc, C))
    dh = C // NH
    out = np.zeros((L, C))
    for i in range(L):
        o = np.zeros(C)
        for j in range(NH):
            q = sum(h[i, c] * wq[j * dh:(j + 1) * dh, c] for c in range(C))
            sc = []
            for t in range(Lc):
                k = sum(ctx[t, c] * wkv[j * dh:(j + 1) * dh, c] for c in range(C))
                sc.append(float(np.dot(q, k)) / np.sqrt(dh))
            mx = max(sc)
            e = [np.exp(s - mx) for s in sc]
            for t in range(Lc):
                v = sum(ctx[t, c] * wkv[C + j * dh:C + (j + 1) * dh, c] for c in range(C))
                o[j * dh:(j + 1) * dh] += e[t] / sum(e) * v
        out[i] = wo @ o
    np.testing.assert_allclose(ob.cross_attention(h, ctx, wq, wkv, wo, NH), out, rtol=0, atol=1e-12)


def test_cross_attention_special_cases():
    """ctx = h reduces to self-attention (mha_sequence); one context token: softmax = 1, so every
    query gets (ctx w_v^T) w_o^T; permuting the context tokens changes nothing."""
    C, NH = 16, 4
    wq, wkv, wo = _w(C, 5)
    rng = np.random.default_rng(6)
    h = rng.normal(size=(9, C))
    np.testing.assert_allclose(ob.cross_attention(h, h, wq, wkv, wo, NH),
                               ob.mha_sequence(h, np.concatenate([wq, wkv]), wo, NH), rtol=0, atol=1e-12)
    one = rng.normal(size=(1, C))
    want = np.tile((one @ wkv[C:].T) @ wo.T, (9, 1))
    np.testing.assert_allclose(ob.cross_attention(h, one, wq, wkv, wo, NH), want, rtol=0, atol=1e-12)
    ctx = rng.normal(size=(6, C))
    perm = rng.permutation(6)
    np.testing.assert_allclose(ob.cross_attention(h, ctx, wq, wkv, wo, NH),
                               ob.cross_attention(h, ctx[perm], wq, wkv, wo, NH), rtol=0, atol=1e-12)


def test_cross_stage_is_per_sample_and_position_independent():
    """Sample b only sees ctx[b]; shuffling tokens inside a sample permutes the output identically
    (no positional terms), so the stage is local under any token sharding (DSP)."""
    C, NH = 16, 2
    rng = np.random.default_rng(7)
    wq, wkv, wo = _w(C, 8)
    Wc = dict(ln_w=1 + 0.1 * rng.normal(size=C), ln_b=0.1 * rng.normal(size=C), w_q=wq, w_kv=wkv, w_o=wo)
    x = rng.normal(size=(2, 3, 4, C))
    ctx = rng.normal(size=(2, 5, C))
    y = ob.cross_stage(x, ctx, Wc, NH)
    ctx2 = ctx.copy()
    ctx2[1] += 1.0
    y2 = ob.cross_stage(x, ctx2, Wc, NH)
    assert np.array_equal(y[0], y2[0]) and not np.allclose(y[1], y2[1])
    p = rng.permutation(12)
    xs = x[0].reshape(12, C)[p].reshape(3, 4, C)
    ys = ob.cross_stage(xs[None], ctx[:1], Wc, NH)[0].reshape(12, C)
    np.testing.assert_allclose(ys, y[0].reshape(12, C)[p], rtol=0, atol=1e-12)


@pytest.mark.parametrize("N", [1, 2, 4])
def test_st_block_with_cross_sharded_equals_unsharded(N):
    """The ST-DiT block with its cross stage under the DSP schedule (cross stage on S-shards, the
    context replicated) equals the unsharded block; without ctx it is the plain ST block."""
    import synth
    from oracle import sharded
    sh = synth.BlockShape(1, 4, 16, 32, 4, "f32")
    x = synth.to_f64(synth.make_x(sh, 3), "f32")
    W = {k: synth.to_f64(v, "f32") for k, v in synth.make_block_weights(sh, 3).items()}
    W.update({k: synth.to_f64(v, "f32") for k, v in synth.make_cross_weights(sh, 3).items()})
    ctx = synth.to_f64(synth.make_context(sh, 3, 7), "f32")
    want = ob.st_block(x, W, sh.NH, ctx)
    got, _ = sharded.simulate_sharded(x, W, sh.NH, N, ctx=ctx)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
    assert not np.allclose(want, ob.st_block(x, W, sh.NH))
