"""The rest of the ST-DiT block of the paper's experiments, float64 numpy (TEST INFRASTRUCTURE ONLY).

P:137 (§4, Models): "We choose spatial-temporal diffusion transformer (ST-DiT) [DiT, Latte] as our
experiment model ... Our model structure basically follows Latte."  The paper gives no block
formula beyond that citation; the readings adopted here (R36-R38) are the standard ones
of the two cited models, each switchable so that with all of them off this is `block.st_block`:

* R36 adaLN-Zero conditioning (DiT): each sublayer k (spatial attention "s", temporal attention
  "t", MLP "m", and the Latte pair's spatial MLP "ms") has per-sample shift_k, scale_k, gate_k
  [B, C] (the timestep / class embedding through SiLU + Linear, computed once per sampling step
  outside the per-token path): y = x + gate_k * F_k(LN_k(x) * (1 + scale_k) + shift_k).
  gate = 0 (the "-Zero" initialisation) makes the sublayer the identity.
* R37 temporal positional embedding (Latte): a table pe [T, C] added to the residual stream once,
  after the spatial sublayers and before the first temporal one: y1 <- y1 + pe[t].
* R38 Latte pair: the spatial sub-block carries its own position-wise MLP (LN_m, W1_s, W2_s)
  after the spatial attention, as Latte's spatial transformer block does; with it the block is
  Latte's (spatial block, temporal block) pair and Megatron-SP's volume is Table 1's 8M (P:112-115,
  `volume.predict_volume(..., n_mlp=2)`).

The sharded schedule is unchanged by any of them: the spatial MLP is position-wise (local on the
T-shards), the modulation vectors are per sample (every rank holds them), and pe[t] is added on
the S-shards, where every rank holds all T positions of its columns.
"""
from __future__ import annotations

import numpy as np

from . import block
from .switch import DIM_S, DIM_T, Ledger, gather, split, switch

SUBLAYERS = ("s", "t", "m", "ms")


def modulate(h: np.ndarray, shift: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """DiT's adaLN modulation of a LayerNorm output h [B, ..., C] with per-sample shift, scale
    [B, C]: h * (1 + scale) + shift."""
    sh = shift.reshape((shift.shape[0],) + (1,) * (h.ndim - 2) + (shift.shape[-1],))
    sc = scale.reshape(sh.shape)
    return h * (1.0 + sc) + sh


def _gate(y: np.ndarray, gate: np.ndarray | None) -> np.ndarray:
    if gate is None:
        return y
    return y * gate.reshape((gate.shape[0],) + (1,) * (y.ndim - 2) + (gate.shape[-1],))


def _sub(x, ln_w, ln_b, f, mod, k):
    """x + gate_k * f(modulate(LN(x)))  (R36); mod None: x + f(LN(x))."""
    h = block.layer_norm(x, ln_w, ln_b)
    if mod is not None and k in mod:
        shift, scale, gate = mod[k]
        return x + _gate(f(modulate(h, shift, scale)), gate)
    return x + f(h)


def spatial_part(x, W, num_heads, mod=None):
    """Spatial attention (+ the Latte pair's spatial MLP) on whole frames [B, T', S, C]."""
    y = _sub(x, W["ln1_w"], W["ln1_b"], lambda h: block.mha_spatial(h, W["w_qkv_s"], W["w_o_s"], num_heads), mod, "s")
    if "w_fc1_s" in W:  # R38
        y = _sub(y, W["ln_m_w"], W["ln_m_b"], lambda h: block.mlp(h, W["w_fc1_s"], W["w_fc2_s"]), mod, "ms")
    return y


def add_pe(y: np.ndarray, pe: np.ndarray | None, t0: int = 0) -> np.ndarray:
    """y [B, T', S', C] with frames t0..t0+T'-1: y + pe[t] (R37)."""
    if pe is None:
        return y
    return y + pe[t0:t0 + y.shape[1]][None, :, None, :]


def temporal_part(y1, W, num_heads, mod=None):
    """Temporal attention on whole columns [B, T, S', C]."""
    return _sub(y1, W["ln2_w"], W["ln2_b"], lambda h: block.mha_temporal(h, W["w_qkv_t"], W["w_o_t"], num_heads),
                mod, "t")


def mlp_part(y2, W, mod=None):
    return _sub(y2, W["ln3_w"], W["ln3_b"], lambda h: block.mlp(h, W["w_fc1"], W["w_fc2"]), mod, "m")


def stdit_block(x: np.ndarray, W: dict, num_heads: int, mod: dict | None = None, pe: np.ndarray | None = None,
                ctx: np.ndarray | None = None) -> np.ndarray:
    """The unsharded ST-DiT block on x [B, T, S, C]: spatial part, + pe, temporal attention,
    optional cross stage (block.cross_stage), MLP.  mod: {sublayer: (shift, scale, gate)}
    per-sample [B, C] arrays (R36); pe: [T, C] (R37); Latte pair if W has w_fc1_s (R38)."""
    y1 = add_pe(spatial_part(x, W, num_heads, mod), pe)
    y2 = temporal_part(y1, W, num_heads, mod)
    if ctx is not None:
        Wc = dict(ln_w=W["ln_c_w"], ln_b=W["ln_c_b"], w_q=W["w_q_c"], w_kv=W["w_kv_c"], w_o=W["w_o_c"])
        y2 = block.cross_stage(y2, ctx, Wc, num_heads)
    return mlp_part(y2, W, mod)


def simulate_sharded(x: np.ndarray, W: dict, num_heads: int, world: int, mod: dict | None = None,
                     pe: np.ndarray | None = None, ledger: Ledger | None = None, elem_bytes: int = 2):
    """The DSP schedule of `stdit_block` over `world` simulated ranks: spatial part on the
    T-shards, switch T->S, + pe on the S-shards (each holds every frame of its columns), temporal
    attention + MLP, switch S->T, gather.  Returns the gathered output."""
    shards = split(x, DIM_T, world)
    y1 = [spatial_part(s, W, num_heads, mod) for s in shards]
    y1s = switch(y1, DIM_T, DIM_S, ledger, "switch_T2S", elem_bytes)
    y2 = [temporal_part(add_pe(s, pe), W, num_heads, mod) for s in y1s]
    y = [mlp_part(s, W, mod) for s in y2]
    out = switch(y, DIM_S, DIM_T, ledger, "switch_S2T", elem_bytes)
    return gather(out, DIM_T, ledger, "epilogue", elem_bytes)


def fold_modulation(W: dict, mod: dict, b: int = 0) -> dict:
    """Sample b's modulation written into the weights (the algebra a B = 1 implementation may use):
    LN(x; g, be) * (1 + sc) + sh = LN(x; g * (1 + sc), be * (1 + sc) + sh) and
    gate * (h W^T) = h (diag(gate) W)^T.  Returns a weight dict for `block`/`stdit_block` with
    mod=None that computes the conditioned block of sample b exactly (in real arithmetic)."""
    out = dict(W)
    pairs = {"s": ("ln1", "w_o_s"), "t": ("ln2", "w_o_t"), "m": ("ln3", "w_fc2"), "ms": ("ln_m", "w_fc2_s")}
    for k, (ln, wo) in pairs.items():
        if k not in mod or f"{ln}_w" not in W:
            continue
        shift, scale, gate = (a[b] for a in mod[k])
        out[f"{ln}_w"] = W[f"{ln}_w"] * (1.0 + scale)
        out[f"{ln}_b"] = W[f"{ln}_b"] * (1.0 + scale) + shift
        out[wo] = W[wo] * gate[:, None]
    return out
