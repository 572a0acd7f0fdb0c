"""GPU parity of the training path (include/dsp_train.h) vs oracle/backward.py.

Building blocks (dgrad / wgrad GEMMs on MN-major tcgen05 operands, the GELU-backward and dual-store
epilogues, LayerNorm backward, attention lse and the tcgen05 attention backward) are compared with
the float64 oracle on the same bf16 inputs; then the block's forward_train + backward at N = 1 and
over virtual ranks (P2P switch, R39-R40 tolerances).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import backward as bw
from oracle import block as ob
from oracle import switch as osw
from tests.gpu_util import assert_block_close, bits16, to_dev, to_f64, weights_dev, weights_f64

pytestmark = pytest.mark.gpu

LOG2E = 1.4426950408889634


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _bf16(a: np.ndarray) -> torch.Tensor:
    """float64 array -> bf16 CUDA tensor (rounded once; read back exactly with to_f64)."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda()


def _rand(shape, scale, seed):
    return np.random.default_rng(seed).uniform(-1, 1, size=shape) * scale


def grad_close(got, ref, rel_l2=1e-2, rel_max=3e-2, name=""):
    """R40: a gradient is within tolerance when its relative L2 error is <= rel_l2 and every element is
    within rel_max * max|ref| (bf16 operands and bf16-stored intermediates; fp32 accumulation)."""
    err = np.abs(got - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    l2 = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    msg = f"{name}: rel-L2 {l2:.3e}, max-abs {err.max():.3e} (scale {scale:.3e})"
    assert l2 <= rel_l2 and err.max() <= rel_max * scale, msg
    return msg


# ----------------------------------------------------------------------- GEMMs
@pytest.mark.parametrize("M,N,K", [(1000, 1152, 4608), (4096, 4608, 1152), (300, 3456, 1152), (256, 1152, 128)])
@pytest.mark.parametrize("gelu", [False, True])
def test_linear_dgrad_vs_oracle(M, N, K, gelu):
    """dX = dY W (W [N, K] read MN-major), optionally * gelu'(u): ragged M, K = 128 / 1152 / 4608."""
    m = dsp()
    ctx = m.Context()
    dY = _bf16(_rand((M, N), 1.0, 1))
    W = _bf16(_rand((N, K), 1.0 / np.sqrt(N), 2))
    u = _bf16(_rand((M, K), 3.0, 3)) if gelu else None
    dX = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
    ctx.linear_dgrad(dY, W, dX, u=u)
    torch.cuda.synchronize()
    ref, _ = bw.linear_bwd(np.zeros((M, K)), to_f64(W), to_f64(dY))
    if gelu:
        ref = bw.gelu_tanh_bwd(to_f64(u), ref)
    print(assert_block_close(to_f64(dX), ref))


@pytest.mark.parametrize("M,N,K", [(16384, 1152, 1152), (2048, 3456, 1152), (16384, 4608, 1152),
                                   (16384, 1152, 4608), (384, 192, 256)])
def test_linear_wgrad_vs_oracle(M, N, K):
    """dW[N, K] = dY^T X in fp32 over M tokens (split-K partials summed in order), then accumulate."""
    m = dsp()
    ctx = m.Context()
    dY = _bf16(_rand((M, N), 1.0, 4))
    X = _bf16(_rand((M, K), 1.0, 5))
    dW = torch.empty(N, K, dtype=torch.float32, device="cuda")
    ctx.linear_wgrad(dY, X, dW)
    torch.cuda.synchronize()
    _, ref = bw.linear_bwd(to_f64(X), np.zeros((N, K)), to_f64(dY))
    got = to_f64(dW)
    # fp32 accumulation of exact bf16 products: relative error ~ sqrt(M) * 2^-24
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max() + 1e-4, np.abs(got - ref).max()
    ctx.linear_wgrad(dY, X, dW, accumulate=True)
    torch.cuda.synchronize()
    np.testing.assert_allclose(to_f64(dW), 2 * got, rtol=2e-5, atol=1e-4)  # slice sums re-rounded
    assert m.lib().dsp_wgrad_workspace_bytes(ctx.handle, M, N, K) >= N * K * 4


def test_linear_gelu_aux_vs_oracle_and_plain_gelu():
    """G = gelu(A W^T) and U = A W^T from one GEMM; G bitwise = the forward's GELU epilogue."""
    m = dsp()
    ctx = m.Context()
    M, N, K = 1000, 4608, 1152
    A = _bf16(_rand((M, K), 1.0, 6))
    W = _bf16(_rand((N, K), 1.0 / np.sqrt(K) * 2, 7))
    G = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    U = torch.empty_like(G)
    G2 = torch.empty_like(G)
    ctx.linear_gelu_aux(A, W, G, U)
    m_ = m
    m_.lib()
    ctx._call("dsp_linear", m.DSP_BF16, M, N, K, A.data_ptr(), W.data_ptr(), None, m.DSP_EPI_GELU, G2.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    u_ref = ob.linear(to_f64(A), to_f64(W))
    print(assert_block_close(to_f64(U), u_ref))
    print(assert_block_close(to_f64(G), ob.gelu_tanh(u_ref)))
    assert np.array_equal(bits16(G), bits16(G2))


# ------------------------------------------------------------------- LayerNorm
@pytest.mark.parametrize("rows,C", [(4096, 1152), (333, 1152), (64, 2048), (10, 64)])
@pytest.mark.parametrize("with_res", [True, False])
def test_layer_norm_bwd_vs_oracle(rows, C, with_res):
    m = dsp()
    ctx = m.Context()
    ctx.ensure_workspace(8 * rows + 2 * C * 4 * ((rows + 63) // 64) + 4096)
    x = _bf16(_rand((rows, C), 2.0, 8) + 0.3)
    gam = _bf16(1.0 + _rand((C,), 0.5, 9))
    dh = _bf16(_rand((rows, C), 1.0, 10))
    dres = _bf16(_rand((rows, C), 1.0, 11)) if with_res else None
    dx = torch.empty(rows, C, dtype=torch.bfloat16, device="cuda")
    gb = torch.zeros(2 * C, dtype=torch.float32, device="cuda")
    ctx.layer_norm_bwd(x, gam, dh, dres, dx, gb)
    torch.cuda.synchronize()
    dz, dg, db = bw.layer_norm_bwd(to_f64(x), to_f64(gam), to_f64(dh))
    if with_res:
        dz = dz + to_f64(dres)
    print(assert_block_close(to_f64(dx), dz))
    g = to_f64(gb)
    print(grad_close(g[:C], dg, rel_l2=1e-5, rel_max=1e-5, name="dgamma"))
    print(grad_close(g[C:], db, rel_l2=1e-5, rel_max=1e-5, name="dbeta"))


# ------------------------------------------------------------------- attention
def _attn_inputs(B, Tl, Sl, C, NH, seed, kappa=1.0):
    tok = B * Tl * Sl
    qkv = _bf16(_rand((tok, 3 * C), kappa, seed))
    dout = _bf16(_rand((tok, C), 1.0, seed + 1))
    return qkv, dout


def _oracle_attn(qkv, dout, B, Tl, Sl, C, NH, dim):
    """per-sequence oracle: o, lse (natural log) and dqkv in the token-major layouts."""
    g = to_f64(qkv).reshape(B, Tl, Sl, 3 * C)
    do = to_f64(dout).reshape(B, Tl, Sl, C)
    o = np.zeros((B, Tl, Sl, C))
    lse = np.zeros((B, Tl, Sl, NH))
    dg = np.zeros_like(g)
    seqs = [(b, t, slice(None)) for b in range(B) for t in range(Tl)] if dim == "S" else \
        [(b, slice(None), s) for b in range(B) for s in range(Sl)]
    for b, t, s in seqs:
        gs = g[b, t, s] if dim == "S" else g[b, :, s]
        L = gs.shape[0]
        q, k, v = ob.split_heads(gs, C, NH)
        oo = ob.attention_core(q, k, v).transpose(1, 0, 2).reshape(L, C)
        ll = bw.attention_lse(q, k).T
        dos = (do[b, t, s] if dim == "S" else do[b, :, s]).reshape(L, NH, C // NH).transpose(1, 0, 2)
        dq, dk, dv = bw.attention_core_bwd(q, k, v, dos)
        mg = lambda a: a.transpose(1, 0, 2).reshape(L, C)
        dgs = np.concatenate([mg(dq), mg(dk), mg(dv)], 1)
        if dim == "S":
            o[b, t], lse[b, t], dg[b, t] = oo, ll, dgs
        else:
            o[b, :, s], lse[b, :, s], dg[b, :, s] = oo, ll, dgs
    tok = B * Tl * Sl
    return o.reshape(tok, C), lse.reshape(tok, NH), dg.reshape(tok, 3 * C)


@pytest.mark.parametrize("B,Tl,Sl,dim", [(1, 2, 1024, "S"), (1, 2, 256, "S"), (1, 16, 64, "T"), (2, 16, 24, "T"),
                                         (1, 128, 8, "T"), (1, 32, 20, "T")])
def test_attention_lse_and_bwd_vs_oracle(B, Tl, Sl, dim):
    """Forward lse (log2 domain) and the tcgen05 attention backward: spatial L = 1024 / 256 (several
    key tiles: dQ by f32 reduce-add), temporal T = 16 / 32 (block-diagonal packing, partial last
    group) and T = 128 (one tile per sequence, direct dQ store)."""
    m = dsp()
    ctx = m.Context()
    C, NH = 1152, 16
    qkv, dout = _attn_inputs(B, Tl, Sl, C, NH, 20)
    tok = B * Tl * Sl
    o = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(tok, NH, dtype=torch.float32, device="cuda")
    ctx.attention_core_lse(B, Tl, Sl, C, NH, dim, qkv, o, lse)
    dqkv = torch.full((tok, 3 * C), float("nan"), dtype=torch.bfloat16, device="cuda")
    ctx.attention_core_bwd(B, Tl, Sl, C, NH, dim, qkv, o, dout, lse, dqkv)
    torch.cuda.synchronize()
    o_ref, lse_ref, dg_ref = _oracle_attn(qkv, dout, B, Tl, Sl, C, NH, dim)
    print(assert_block_close(to_f64(o), o_ref))
    np.testing.assert_allclose(to_f64(lse), lse_ref * LOG2E, rtol=0, atol=2e-3)
    got = to_f64(dqkv)
    assert np.isfinite(got).all()
    for i, nm in enumerate(("dq", "dk", "dv")):
        print(grad_close(got[:, i * C:(i + 1) * C], dg_ref[:, i * C:(i + 1) * C], name=nm))


def test_attention_bwd_peaky_softmax():
    """kappa = 4 scores (a peaky softmax): the recomputed P = exp2(s - lse) must stay consistent."""
    m = dsp()
    ctx = m.Context()
    B, Tl, Sl, C, NH, dim = 1, 1, 1024, 1152, 16, "S"
    qkv, dout = _attn_inputs(B, Tl, Sl, C, NH, 30, kappa=4.0)
    tok = B * Tl * Sl
    o = torch.empty(tok, C, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(tok, NH, dtype=torch.float32, device="cuda")
    ctx.attention_core_lse(B, Tl, Sl, C, NH, dim, qkv, o, lse)
    dqkv = torch.empty(tok, 3 * C, dtype=torch.bfloat16, device="cuda")
    ctx.attention_core_bwd(B, Tl, Sl, C, NH, dim, qkv, o, dout, lse, dqkv)
    torch.cuda.synchronize()
    _, _, dg_ref = _oracle_attn(qkv, dout, B, Tl, Sl, C, NH, dim)
    got = to_f64(dqkv)
    for i, nm in enumerate(("dq", "dk", "dv")):
        print(grad_close(got[:, i * C:(i + 1) * C], dg_ref[:, i * C:(i + 1) * C], rel_l2=2e-2, name=nm))


# ----------------------------------------------------------------------- block
def _train_n1(sh, xs, Ws, dys, reps=1):
    m = dsp()
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ctx.ensure_workspace(m.train_workspace_bytes(shape, 1))
    lay = m.train_saved_layout(shape, 1)
    saved = torch.empty(lay["total"], dtype=torch.uint8, device="cuda")
    W = weights_dev(Ws, "bf16")
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    dY = _bf16(dys)
    dX = torch.empty_like(X)
    G = {n: torch.zeros(W[n].shape, dtype=torch.float32, device="cuda") for n in m.GRAD_NAMES}
    for _ in range(reps):
        ctx.block_forward_train(shape, W, X, Y, saved)
        ctx.block_backward(shape, W, saved, X, dY, dX, G)
    torch.cuda.synchronize()
    return Y, dX, G


@pytest.mark.parametrize("sh", [synth.BlockShape(1, 16, 256, 1152, 16, "bf16"),
                                synth.BlockShape(2, 4, 128, 1152, 16, "bf16")])
def test_block_train_vs_oracle(sh):
    """forward_train == the oracle block; backward dx and all twelve weight gradients vs
    oracle/backward.st_block_bwd (R40)."""
    xs, Ws = synth.make_x(sh, 7), synth.make_block_weights(sh, 7)
    dys = _rand((sh.B, sh.T, sh.S, sh.C), 1.0, 40)
    Y, dX, G = _train_n1(sh, xs, Ws, dys)
    x64, W64 = synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16")
    dy64 = to_f64(_bf16(dys)).reshape(dys.shape)
    print(assert_block_close(to_f64(Y).reshape(xs.shape), ob.st_block(x64, W64, sh.NH)))
    dx_ref, g_ref = bw.st_block_bwd(x64, W64, sh.NH, dy64)
    print(grad_close(to_f64(dX).reshape(xs.shape), dx_ref, name="dx"))
    for n in bw.GRAD_NAMES:
        print(grad_close(to_f64(G[n]), g_ref[n], rel_l2=2e-2, rel_max=5e-2, name=n))


def test_block_train_deterministic_and_accumulating():
    """The backward is deterministic (no atomics in the reductions: dx and every gradient bitwise
    equal across runs), and a second pass accumulates (+=) the same gradient again."""
    sh = synth.BlockShape(1, 16, 128, 1152, 16, "bf16")
    xs, Ws = synth.make_x(sh, 3), synth.make_block_weights(sh, 3)
    dys = _rand((sh.B, sh.T, sh.S, sh.C), 1.0, 41)
    _, dx1, g1 = _train_n1(sh, xs, Ws, dys, reps=1)
    _, dx1b, g1b = _train_n1(sh, xs, Ws, dys, reps=1)
    _, dx2, g2 = _train_n1(sh, xs, Ws, dys, reps=2)
    assert np.array_equal(bits16(dx1), bits16(dx1b)) and np.array_equal(bits16(dx1), bits16(dx2))
    for n in g1:
        assert torch.equal(g1[n], g1b[n]), n
        torch.testing.assert_close(g2[n], 2 * g1[n], rtol=1e-5, atol=1e-5 * float(g1[n].abs().max()))


@pytest.mark.parametrize("N", [2, 4])
def test_block_train_virtual_ranks(N):
    """DSP training over N virtual ranks (P2P switches, the backward's switches in the opposite
    direction): y and dx bitwise equal to N = 1 (row-local dgrad / LN / per-sequence attention);
    the weight gradients summed over the ranks match N = 1 within fp32 reordering."""
    m = dsp()
    from tests.test_gpu_block import VirtualGroup
    sh = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")
    xs, Ws = synth.make_x(sh, 5), synth.make_block_weights(sh, 5)
    dys = _rand((sh.B, sh.T, sh.S, sh.C), 1.0, 42)
    Y1, dX1, G1 = _train_n1(sh, xs, Ws, dys)
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = (m.train_workspace_bytes(shape, N) + 1023) // 1024 * 1024
    sv = (m.train_saved_layout(shape, N)["total"] + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + sv + 4 * act)
    W = weights_dev(Ws, "bf16")
    xsh = osw.split(xs, osw.DIM_T, N)
    dysh = osw.split(to_f64(_bf16(dys)).reshape(dys.shape), osw.DIM_T, N)
    X = [g.view(r, ws + sv, act, torch.bfloat16) for r in range(N)]
    Y = [g.view(r, ws + sv + act, act, torch.bfloat16) for r in range(N)]
    dY = [g.view(r, ws + sv + 2 * act, act, torch.bfloat16) for r in range(N)]
    dX = [g.view(r, ws + sv + 3 * act, act, torch.bfloat16) for r in range(N)]
    saved = [g.region[r][ws:ws + sv] for r in range(N)]
    G = [{n: torch.zeros(W[n].shape, dtype=torch.float32, device="cuda") for n in m.GRAD_NAMES} for _ in range(N)]
    for r in range(N):
        X[r].copy_(to_dev(xsh[r], "bf16").reshape(-1))
        dY[r].copy_(_bf16(dysh[r]).reshape(-1))
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].block_forward_train(shape, W, X[r], Y[r], saved[r], impl="p2p"))
    g.run(lambda r: g.ctx[r].block_backward(shape, W, saved[r], X[r], dY[r], dX[r], G[r], impl="p2p"))
    cat = lambda ts: np.concatenate([bits16(t).reshape(sh.B, sh.T // N, sh.S, sh.C) for t in ts], 1).reshape(-1)
    assert np.array_equal(cat(Y), bits16(Y1).reshape(-1))
    assert np.array_equal(cat(dX), bits16(dX1).reshape(-1))
    for n in m.GRAD_NAMES:
        tot = sum(to_f64(G[r][n]) for r in range(N))
        ref = to_f64(G1[n])
        assert np.abs(tot - ref).max() <= 1e-4 * np.abs(ref).max() + 1e-5, n


def test_block_train_benchmarked_shape_vs_oracle():
    """The exact configuration `bench.py --config train` times (configs[1]: B=1 T=16 S=1024 C=1152,
    16 heads; the spatial attention backward on its multi-key-tile path with the f32 dQ reduce-add)
    against the float64 oracle backward: dx and all twelve weight gradients (R40)."""
    sh = synth.BlockShape(1, 16, 1024, 1152, 16, "bf16")
    xs, Ws = synth.make_x(sh, 7), synth.make_block_weights(sh, 7)
    dys = _rand((sh.B, sh.T, sh.S, sh.C), 1.0, 43)
    Y, dX, G = _train_n1(sh, xs, Ws, dys)
    x64, W64 = synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16")
    dy64 = to_f64(_bf16(dys)).reshape(dys.shape)
    dx_ref, g_ref = bw.st_block_bwd(x64, W64, sh.NH, dy64)
    print(grad_close(to_f64(dX).reshape(xs.shape), dx_ref, name="dx"))
    for n in bw.GRAD_NAMES:
        print(grad_close(to_f64(G[n]), g_ref[n], rel_l2=2e-2, rel_max=5e-2, name=n))


def test_training_path_rejects_what_it_does_not_support():
    """Documented limits (include/dsp_train.h) fail loudly with the right status, before any launch."""
    m = dsp()
    ctx = m.Context()
    ok = synth.BlockShape(1, 16, 128, 1152, 16, "bf16")
    Ws = weights_dev(synth.make_block_weights(ok, 1), "bf16")
    X = to_dev(synth.make_x(ok, 1), "bf16")
    Y = torch.empty_like(X)

    def call(shape, W=Ws, ws=True):
        if ws:
            ctx.ensure_workspace(m.train_workspace_bytes(shape, 1))
        saved = torch.empty(m.train_saved_layout(shape, 1)["total"] + 256, dtype=torch.uint8, device="cuda")
        with pytest.raises(m.DSPError) as e:
            ctx.block_forward_train(shape, W, X, Y, saved)
        return e.value.name

    assert call(m.make_shape(1, 16, 128, 1152, 12, "bf16")) == "DSP_ERR_UNSUPPORTED"   # Dh = 96
    assert call(m.make_shape(1, 16, 100, 1152, 16, "bf16")) == "DSP_ERR_UNSUPPORTED"   # S neither divides nor is a multiple of 128
    assert call(m.make_shape(1, 16, 128, 1152, 16, "f32")) == "DSP_ERR_UNSUPPORTED"    # f32
    W2 = dict(Ws)
    W2["pe_t"] = torch.zeros(16, 1152, dtype=torch.bfloat16, device="cuda")
    assert call(m.make_shape(1, 16, 128, 1152, 16, "bf16"), W=W2) == "DSP_ERR_UNSUPPORTED"  # forward-only extras
    shape = m.make_shape(1, 16, 128, 1152, 16, "bf16")
    saved = torch.empty(m.train_saved_layout(shape, 1)["total"] + 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(m.DSPError) as e:  # the fused switch epilogues are forward-only
        ctx.block_forward_train(shape, Ws, X, Y, saved, impl="fused")
    assert e.value.name == "DSP_ERR_UNSUPPORTED"
    ctx.set_workspace(torch.empty(1024, dtype=torch.uint8, device="cuda"))
    assert call(m.make_shape(1, 16, 128, 1152, 16, "bf16"), ws=False) == "DSP_ERR_WORKSPACE"
