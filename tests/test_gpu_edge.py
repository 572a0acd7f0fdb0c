"""GPU parity at the degenerate and ragged edges of the hot path (through the C ABI).

* length-1 attention (T = 1 for the temporal stage, S = 1 for the spatial stage): the softmax
  over one key is exactly 1, so each head's output is its value row -- a closed form the
  kernels must hit bit for bit (P = exp2(0) = 1 in bf16, O = V / 1);
* blocks whose temporal or spatial extent is 1 (one stage reduces to V·Wo), raw and prepared;
* sequence lengths that are neither a multiple nor a divisor of the 128-row tile (R33): the
  last query tile is clipped by the TMA store, keys past the end of the last key tile are
  masked before the row max.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import block as ob
from tests.gpu_util import assert_block_close, to_dev, to_f64, weights_dev, weights_f64

pytestmark = pytest.mark.gpu


def _dsp():
    import paper_2403_10266_b200 as m
    return m


def _qkv_bits(B, T, S, C, seed=11):
    n = B * T * S * 3 * C
    v = synth.uniform_pm1(seed, 5, np.arange(n, dtype=np.uint64)).reshape(B * T * S, 3 * C)
    return synth.round_to_bf16_bits(v)


@pytest.mark.parametrize("B,T,S,C,NH,dim", [
    (1, 1, 300, 1152, 16, "T"),   # temporal, one frame: 300 sequences of length 1 (128 per tile)
    (2, 1, 77, 256, 4, "T"),      # ragged tile count, B = 2
    (1, 40, 1, 1152, 16, "S"),    # spatial, one token per frame
    (1, 5, 1, 64, 4, "S"),        # Dh = 16
])
def test_length_one_attention_is_v(B, T, S, C, NH, dim):
    """softmax over a single key is 1: O must equal the value slice of QKV bit for bit."""
    m = _dsp()
    ctx = m.Context()
    ctx.ensure_workspace(1 << 20)
    bits = _qkv_bits(B, T, S, C)
    Q = to_dev(bits, "bf16")
    O = torch.full((B * T * S, C), float("nan"), dtype=torch.bfloat16, device="cuda")
    ctx.attention_core(B, T, S, C, NH, dim, Q, O)
    torch.cuda.synchronize()
    V = Q[:, 2 * C:]
    assert torch.equal(O.view(torch.int16), V.contiguous().view(torch.int16))


@pytest.mark.parametrize("B,T,S,C,NH,dim,kappa", [
    (1, 16, 200, 256, 4, "S", 1.0),    # S = 200: two query tiles per frame (pair kernel), 72 valid keys in the last
    (1, 3, 384, 1152, 16, "S", 1.0),   # S = 384: three full tiles, odd tile count (single-tile kernel)
    (1, 2, 300, 1152, 16, "S", 4.0),   # S = 300: three tiles, 44 valid in the last, peaky
    (2, 16, 48, 256, 4, "S", 1.0),     # S = 48 (not a divisor of 128): one masked tile per frame
    (1, 3, 576, 1152, 16, "S", 1.0),   # S = 576 = 24 x 24 latent: 4.5 tiles
    (1, 51, 40, 1152, 16, "T", 1.0),   # T = 51 frames: one masked tile per column
    (2, 100, 9, 256, 4, "T", 4.0),     # T = 100, B = 2, peaky
    (1, 200, 6, 256, 4, "T", 1.0),     # T = 200: two tiles per column (pair kernel)
])
def test_ragged_sequences(B, T, S, C, NH, dim, kappa):
    """Sequence lengths that neither divide 128 nor are a multiple of it (R33)."""
    m = _dsp()
    ctx = m.Context()
    ctx.ensure_workspace(1 << 20)
    n = B * T * S * 3 * C
    v = synth.uniform_pm1(13, 5, np.arange(n, dtype=np.uint64)).reshape(B * T * S, 3 * C)
    v[:, :2 * C] *= kappa
    bits = synth.round_to_bf16_bits(v)
    Q = to_dev(bits, "bf16")
    O = torch.full((B * T * S, C), float("nan"), dtype=torch.bfloat16, device="cuda")
    ctx.attention_core(B, T, S, C, NH, dim, Q, O)
    torch.cuda.synchronize()
    g = synth.bf16_bits_to_f64(bits).reshape(B, T, S, 3 * C)
    ref = np.empty((B, T, S, C))

    def run(seq):
        q, k, v = ob.split_heads(seq, C, NH)
        return ob.attention_core(q, k, v).transpose(1, 0, 2).reshape(seq.shape[0], C)
    for b in range(B):
        if dim == "S":
            for t in range(T):
                ref[b, t] = run(g[b, t])
        else:
            for s_ in range(S):
                ref[b, :, s_] = run(g[b, :, s_])
    assert_block_close(to_f64(O), ref.reshape(B * T * S, C), atol=1e-2, rtol=1e-2, rel_l2=1e-2)


@pytest.mark.parametrize("sh", [synth.BlockShape(1, 1, 256, 256, 4, "bf16"),    # T = 1
                                synth.BlockShape(1, 16, 1, 256, 4, "bf16"),     # S = 1
                                synth.BlockShape(2, 1, 128, 1152, 16, "bf16"),  # T = 1, B = 2, model width
                                synth.BlockShape(1, 51, 64, 256, 4, "bf16"),    # T = 51 (ragged temporal)
                                synth.BlockShape(1, 4, 200, 256, 4, "bf16")])   # S = 200 (ragged spatial)
@pytest.mark.parametrize("prepared", [False, True])
def test_block_degenerate_extent(sh, prepared):
    """A block whose temporal (or spatial) extent is 1, or ragged, against the oracle block."""
    m = _dsp()
    Ws = synth.make_block_weights(sh, 7)
    xs = synth.make_x(sh, 7)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, sh.dtype)
    Y = torch.empty_like(X)
    W = weights_dev(Ws, sh.dtype)
    if prepared:
        W["prepared"] = ctx.prepare_block(shape, W)
    ctx.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    print(assert_block_close(to_f64(Y), ref))


@pytest.mark.parametrize("sh,prepared", [
    (synth.BlockShape(1, 4, 128, 2048, 16, "bf16"), False),   # Dh = 128 (two 64-column TMA boxes)
    (synth.BlockShape(1, 4, 128, 2048, 16, "bf16"), True),    # 12-vector row statistics, 8 LN partials
    (synth.BlockShape(1, 8, 128, 1024, 16, "bf16"), False),   # Dh = 64
    (synth.BlockShape(1, 8, 128, 1024, 16, "bf16"), True),
    (synth.BlockShape(2, 4, 64, 768, 12, "bf16"), True),      # Dh = 64, C = 768 (DiT-B width)
])
def test_block_other_widths(sh, prepared):
    """Model widths other than the paper's 1152 / Dh = 72 against the oracle block."""
    m = _dsp()
    Ws = synth.make_block_weights(sh, 7)
    xs = synth.make_x(sh, 7)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    ctx.ensure_workspace(m.workspace_bytes(shape, 1))
    X = to_dev(xs, sh.dtype)
    Y = torch.empty_like(X)
    W = weights_dev(Ws, sh.dtype)
    if prepared:
        W["prepared"] = ctx.prepare_block(shape, W)
    ctx.st_block_forward(shape, W, X, Y)
    torch.cuda.synchronize()
    ref = ob.st_block(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH)
    print(assert_block_close(to_f64(Y), ref))


def test_prepared_path_rejects_wide_rows():
    """C > 3072 on the prepared (LayerNorm-folded) path is a documented UNSUPPORTED, not a
    wrong answer; the raw-weights path covers any width."""
    m = _dsp()
    sh = synth.BlockShape(1, 2, 16, 4096, 32, "bf16")
    Ws = synth.make_block_weights(sh, 7)
    ctx = m.Context()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    W = weights_dev(Ws, sh.dtype)
    with pytest.raises(m.DSPError, match="UNSUPPORTED"):
        ctx.prepare_block(shape, W)
