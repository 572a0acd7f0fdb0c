"""Unsharded spatial-temporal block, float64 numpy (TEST INFRASTRUCTURE ONLY).

Block (reading R1, SURVEY §8 "Block definition"):
    y1 = x  + MHA_S(LN1(x))     spatial: one sequence per (b, t), length S
    y2 = y1 + MHA_T(LN2(y1))    temporal: one sequence per (b, s), length T
    y  = y2 + MLP(LN3(y2))
P:40 ("Residual connections are used around the layers ... Layer normalization
is also applied before each layer"); P:17 and P:46 (attention "calculated
separately for the temporal and spatial dimensions"); P:137 (ST-DiT follows
Latte).  Readings where the paper is silent: LN eps 1e-5
with affine and biased variance (R3); no linear biases (R4); MLP ratio 4 with
tanh-GELU (R5); scale 1/sqrt(Dh) (R6); no masks / positional terms (R7);
w_qkv rows are [q | k | v], head j owns rows j*Dh..(j+1)*Dh-1 of each (R8).
"""
from __future__ import annotations

import numpy as np

LN_EPS = 1e-5


def linear(h: np.ndarray, w: np.ndarray) -> np.ndarray:
    """nn.Linear without bias: h @ w^T, w in [out, in] layout (R4, R8)."""
    return h @ w.T


def layer_norm(z: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float = LN_EPS) -> np.ndarray:
    """Per-token LayerNorm over the last (channel) axis (R3).

    mu = mean(z); var = mean((z - mu)^2) (biased); (z - mu)/sqrt(var + eps)*gamma + beta
    """
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    return (z - mu) / np.sqrt(var + eps) * gamma + beta


def gelu_tanh(u: np.ndarray) -> np.ndarray:
    """0.5 u (1 + tanh(sqrt(2/pi) (u + 0.044715 u^3)))  (R5)."""
    return 0.5 * u * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (u + 0.044715 * u ** 3)))


def attention_core(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Per-head softmax attention over one sequence (R6, R7).

    q, k, v: [NH, L, Dh].  A = q k^T / sqrt(Dh); P = softmax over keys (row max
    subtracted); O = P v.  Returns [NH, L, Dh].
    """
    dh = q.shape[-1]
    a = (q @ np.swapaxes(k, -1, -2)) / np.sqrt(dh)
    a = a - a.max(axis=-1, keepdims=True)
    p = np.exp(a)
    p = p / p.sum(axis=-1, keepdims=True)
    return p @ v


def split_heads(g: np.ndarray, C: int, num_heads: int):
    """G = H w_qkv^T of shape [L, 3C] -> q, k, v each [NH, L, Dh] (R8)."""
    L = g.shape[0]
    dh = C // num_heads
    q, k, v = g[:, :C], g[:, C:2 * C], g[:, 2 * C:]
    f = lambda t: t.reshape(L, num_heads, dh).transpose(1, 0, 2)
    return f(q), f(k), f(v)


def mha_sequence(h: np.ndarray, w_qkv: np.ndarray, w_o: np.ndarray, num_heads: int) -> np.ndarray:
    """Multi-head self-attention over ONE sequence h [L, C] -> [L, C].

    G = h w_qkv^T; split into q, k, v and heads; O_j = softmax(q_j k_j^T/sqrt(Dh)) v_j;
    O = [O_0 .. O_{NH-1}] (heads concatenated along channels); return O w_o^T.
    """
    L, C = h.shape
    q, k, v = split_heads(linear(h, w_qkv), C, num_heads)
    o = attention_core(q, k, v)                       # [NH, L, Dh]
    o = o.transpose(1, 0, 2).reshape(L, C)
    return linear(o, w_o)


def mha_spatial(h: np.ndarray, w_qkv, w_o, num_heads: int) -> np.ndarray:
    """Spatial attention on [B, T', S, C]: one sequence over S per (b, t)."""
    out = np.empty_like(h)
    for b in range(h.shape[0]):
        for t in range(h.shape[1]):
            out[b, t] = mha_sequence(h[b, t], w_qkv, w_o, num_heads)
    return out


def mha_temporal(h: np.ndarray, w_qkv, w_o, num_heads: int) -> np.ndarray:
    """Temporal attention on [B, T, S', C]: one sequence over T per (b, s)."""
    out = np.empty_like(h)
    for b in range(h.shape[0]):
        for s in range(h.shape[2]):
            out[b, :, s] = mha_sequence(h[b, :, s], w_qkv, w_o, num_heads)
    return out


def mlp(h: np.ndarray, w_fc1, w_fc2) -> np.ndarray:
    """Position-wise MLP gelu_tanh(h W1^T) W2^T (R5)."""
    return linear(gelu_tanh(linear(h, w_fc1)), w_fc2)


def spatial_stage(x, W, num_heads):
    """y1 = x + MHA_S(LN1 x) on a [B, T', S, C] array (whole frames)."""
    return x + mha_spatial(layer_norm(x, W["ln1_w"], W["ln1_b"]), W["w_qkv_s"], W["w_o_s"], num_heads)


def temporal_stage(y1, W, num_heads):
    """y2 = y1 + MHA_T(LN2 y1) on a [B, T, S', C] array (whole columns)."""
    return y1 + mha_temporal(layer_norm(y1, W["ln2_w"], W["ln2_b"]), W["w_qkv_t"], W["w_o_t"], num_heads)


def mlp_stage(y2, W):
    """y = y2 + MLP(LN3 y2), position-wise."""
    return y2 + mlp(layer_norm(y2, W["ln3_w"], W["ln3_b"]), W["w_fc1"], W["w_fc2"])


def st_block(x: np.ndarray, W: dict, num_heads: int, ctx: np.ndarray | None = None) -> np.ndarray:
    """The unsharded ST block on global x [B, T, S, C] (float64).  With `ctx` [B, Lc, C] and the
    cross weights in W (ln_c_w, ln_c_b, w_q_c, w_kv_c, w_o_c), the ST-DiT block of P:137: a cross
    stage y2' = y2 + CA(LN_c(y2), ctx) between the temporal stage and the MLP."""
    y2 = temporal_stage(spatial_stage(x, W, num_heads), W, num_heads)
    if ctx is not None:
        Wc = dict(ln_w=W["ln_c_w"], ln_b=W["ln_c_b"], w_q=W["w_q_c"], w_kv=W["w_kv_c"], w_o=W["w_o_c"])
        y2 = cross_stage(y2, ctx, Wc, num_heads)
    return mlp_stage(y2, W)


# --------------------------------------------------------------- cross-attention
def cross_attention(h: np.ndarray, ctx: np.ndarray, w_q, w_kv, w_o, num_heads: int) -> np.ndarray:
    """Multi-head cross-attention of ONE sample's tokens h [L, C] to its context tokens ctx [Lc, C]
    (ST-DiT "uses spatial-temporal and cross attention"; Latte/PixArt-style text
    conditioning).  q = h w_q^T, [k | v] = ctx w_kv^T (w_kv rows [k | v], head j owns rows
    j*Dh..(j+1)*Dh-1 of each, R8); O_j = softmax(q_j k_j^T / sqrt(Dh)) v_j; heads concatenated;
    return O w_o^T.  No mask, no bias (R4, R7)."""
    L, C = h.shape
    dh = C // num_heads
    q = linear(h, w_q).reshape(L, num_heads, dh).transpose(1, 0, 2)
    kv = linear(ctx, w_kv)
    Lc = ctx.shape[0]
    k = kv[:, :C].reshape(Lc, num_heads, dh).transpose(1, 0, 2)
    v = kv[:, C:].reshape(Lc, num_heads, dh).transpose(1, 0, 2)
    o = attention_core(q, k, v)                        # [NH, L, Dh]
    return linear(o.transpose(1, 0, 2).reshape(L, C), w_o)


def cross_stage(x: np.ndarray, ctx: np.ndarray, Wc: dict, num_heads: int) -> np.ndarray:
    """y = x + CA(LN(x), ctx) on x [B, ..., C] with ctx [B, Lc, C]: every token of sample b attends
    to sample b's context (position-independent: any sharding of the tokens is local)."""
    out = np.empty_like(x)
    for b in range(x.shape[0]):
        hb = layer_norm(x[b], Wc["ln_w"], Wc["ln_b"]).reshape(-1, x.shape[-1])
        out[b] = (x[b].reshape(-1, x.shape[-1]) +
                  cross_attention(hb, ctx[b], Wc["w_q"], Wc["w_kv"], Wc["w_o"], num_heads)).reshape(x[b].shape)
    return out
