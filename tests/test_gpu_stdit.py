"""GPU parity of the rest of P:137's ST-DiT block (R36-R38) against oracle.stdit:
the Latte pair's spatial MLP, the temporal positional embedding, adaLN-Zero through the B = 1
weight fold, all of them at once, and over virtual ranks (bitwise N-invariance)."""
import numpy as np
import pytest
import torch

import synth
from oracle import stdit as osd
from oracle import switch as osw
from tests.gpu_util import assert_block_close, bits16, to_dev, to_f64, weights_dev, weights_f64
from tests.test_gpu_block import VirtualGroup

pytestmark = pytest.mark.gpu

SH = synth.BlockShape(1, 16, 256, 1152, 16, "bf16")


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _host(latte=True, pe=True, mod=True, seed=7):
    W = synth.make_block_weights(SH, seed)
    if latte:
        W.update(synth.make_latte_weights(SH, seed))
    m = synth.make_modulation(SH, seed, sublayers=("s", "t", "m", "ms")) if mod else None
    p = synth.make_temporal_pe(SH) if pe else None
    return synth.make_x(SH, seed), W, m, p


def _oracle(xs, W, m, p):
    """The oracle block and the residual-stream values it passes through, each of which the GPU
    block stores in bf16 (R34's storage bound): after the spatial attention, the Latte MLP, pe,
    the temporal attention, and the output."""
    mod = None if m is None else {k: tuple(a.astype(np.float64) for a in v) for k, v in m.items()}
    pe = None if p is None else synth.to_f64(p, "bf16")
    x, Wf = synth.to_f64(xs, "bf16"), weights_f64(W, "bf16")
    ref = osd.stdit_block(x, Wf, SH.NH, mod=mod, pe=pe)
    Wa = {k: v for k, v in Wf.items() if k not in synth.LATTE_NAMES}
    stored = [osd.spatial_part(x, Wa, SH.NH, mod)]
    y1 = osd.spatial_part(x, Wf, SH.NH, mod)
    if "w_fc1_s" in Wf:
        stored.append(y1)
    y1 = osd.add_pe(y1, pe)
    if pe is not None:
        stored.append(y1)
    stored += [osd.temporal_part(y1, Wf, SH.NH, mod), ref]
    return ref, stored


def _device_weights(ctx, shape, W, m, p, prepared):
    Wd = weights_dev(W, "bf16")
    if p is not None:
        Wd["pe_t"] = to_dev(p, "bf16")
    if m is not None:
        mod = np.zeros((4, 3, SH.C), np.float32)
        for i, k in enumerate(dsp().ADALN_SUBLAYERS):
            if k in m:
                mod[i] = np.stack([a[0] for a in m[k]])
        Wd = ctx.adaln_fold(shape, Wd, torch.from_numpy(mod).cuda())
    if prepared:
        Wd["prepared"] = ctx.prepare_block(shape, Wd)
    torch.cuda.synchronize()
    return Wd


def _run_n1(xs, W, m, p, prepared):
    mm = dsp()
    ctx = mm.Context()
    shape = mm.make_shape(SH.B, SH.T, SH.S, SH.C, SH.NH, "bf16")
    ctx.ensure_workspace(mm.workspace_bytes(shape, 1))
    Wd = _device_weights(ctx, shape, W, m, p, prepared)
    X = to_dev(xs, "bf16")
    Y = torch.empty_like(X)
    ctx.st_block_forward(shape, Wd, X, Y)
    torch.cuda.synchronize()
    return Y


@pytest.mark.parametrize("prepared", [False, True])
@pytest.mark.parametrize("what", ["latte", "pe", "adaln", "all"])
def test_stdit_block_vs_oracle(what, prepared):
    """Each extra alone and all together, raw and prepared weights, against the float64 oracle
    at the block gate (R22, with R34's bf16 storage bound for the up to five residual-stream values
    the block stores; the adaLN fold adds one bf16 rounding of the modulated weights)."""
    xs, W, m, p = _host(latte=what in ("latte", "all"), pe=what in ("pe", "all"), mod=what in ("adaln", "all"))
    got = to_f64(_run_n1(xs, W, m, p, prepared)).reshape(SH.B, SH.T, SH.S, SH.C)
    ref, stored = _oracle(xs, W, m, p)
    print(assert_block_close(got, ref, stored=stored))


@pytest.mark.parametrize("prepared", [False, True])
@pytest.mark.parametrize("N", [2, 4])
def test_stdit_block_virtual_ranks_n_invariant(N, prepared):
    """Latte pair + pe + adaLN-folded weights over N virtual ranks (P2P switch) == the N = 1 block
    bitwise: the spatial MLP is local on the T-shards, pe is added on the S-shards."""
    mm = dsp()
    xs, W, m, p = _host()
    ref = bits16(_run_n1(xs, W, m, p, prepared))
    shape = mm.make_shape(SH.B, SH.T, SH.S, SH.C, SH.NH, "bf16")
    ws = (mm.workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = SH.M * 2 // N
    g = VirtualGroup(N, ws + act)
    Wd = _device_weights(g.ctx[0], shape, W, m, p, prepared)
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward(shape, Wd, X[r], Y[r], impl="p2p"))
    got = np.concatenate([bits16(Y[r]).reshape(SH.B, SH.T // N, SH.S, SH.C) for r in range(N)], axis=1)
    assert np.array_equal(got.reshape(-1), ref.reshape(-1))


def test_adaln_fold_rejects_batches():
    mm = dsp()
    ctx = mm.Context()
    sh2 = synth.BlockShape(2, 4, 128, 256, 4, "bf16")
    shape = mm.make_shape(sh2.B, sh2.T, sh2.S, sh2.C, sh2.NH, "bf16")
    Wd = weights_dev(synth.make_block_weights(sh2, 1), "bf16")
    with pytest.raises(mm.DSPError, match="UNSUPPORTED"):
        ctx.adaln_fold(shape, Wd, torch.zeros(4, 3, sh2.C, device="cuda"))


def test_latte_pair_rejects_fused_switch_and_ulysses():
    mm = dsp()
    xs, W, _, p = _host(mod=False)
    N = 2
    shape = mm.make_shape(SH.B, SH.T, SH.S, SH.C, SH.NH, "bf16")
    ws = (max(mm.workspace_bytes(shape, N), mm.ulysses_workspace_bytes(shape, N)) + 1023) // 1024 * 1024
    act = SH.M * 2 // N
    g = VirtualGroup(N, ws + act)
    Wd = weights_dev(W, "bf16")
    Wd["pe_t"] = to_dev(p, "bf16")
    g.ctx[0].set_workspace(g.region[0][:ws])
    X = to_dev(osw.split(xs, osw.DIM_T, N)[0], "bf16").reshape(-1)
    Y = g.view(0, ws, act, torch.bfloat16)
    with pytest.raises(mm.DSPError, match="UNSUPPORTED"):
        g.ctx[0].st_block_forward(shape, Wd, X, Y, impl="fused")
    with pytest.raises(mm.DSPError, match="UNSUPPORTED"):
        g.ctx[0].st_block_forward_ulysses(shape, Wd, X, Y, impl="p2p")
