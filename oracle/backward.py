"""Backward pass of the ST block and of its DSP schedule, float64 numpy (TEST INFRASTRUCTURE ONLY).

SURVEY §8(f) f4: "the switch's adjoint is the inverse switch, so it is reused unchanged; tcgen05
FMHA and GEMM backward; ZeRO-sharded weights".  The paper's throughput numbers are training
(§4.2: "scale the number of GPUs used for training"); P:125 (§3.3) combines DSP with ZeRO
for the parameters, whose gradients are the per-rank sums reduced over the ranks.

Everything here is the textbook chain rule of the forward in `block.py`, written out step by
step in the forward's own order and notation (reading R39 in DESIGN.md):
  linear        y = h W^T                 dh = dy W,  dW = dy^T h
  layer_norm    y = xhat*gamma + beta      dgamma = sum dy*xhat, dbeta = sum dy,
                                           dz = (dxhat - mean(dxhat) - xhat*mean(dxhat*xhat)) / sigma
  gelu_tanh     g = 0.5 u (1 + tanh w)     du = dg * d/du[g]
  attention     A = q k^T / sqrt(Dh), P = softmax(A), O = P v
                                           dv = P^T dO, dP = dO v^T,
                                           dA = P * (dP - rowsum(dP * P)), dq = dA k / sqrt(Dh),
                                           dk = dA^T q / sqrt(Dh)
Residuals pass the gradient through unchanged.  No blocking or fusion; the only library
primitives are matmuls and elementwise numpy.  Pinned (tests/test_oracle_backward.py) against
torch.autograd of an independent torch.nn composition in float64, central finite differences on
tiny shapes, the switch adjoint identity <switch(a), b> = <a, switch^-1(b)>, and sharded ==
unsharded.
"""
from __future__ import annotations

import numpy as np

from . import block
from .switch import DIM_S, DIM_T, gather, split, switch

GRAD_NAMES = (
    "ln1_w", "ln1_b", "w_qkv_s", "w_o_s",
    "ln2_w", "ln2_b", "w_qkv_t", "w_o_t",
    "ln3_w", "ln3_b", "w_fc1", "w_fc2",
)


def linear_bwd(h: np.ndarray, w: np.ndarray, dy: np.ndarray):
    """y = h w^T (w [out, in]) -> (dh = dy w, dw = dy^T h) over all leading axes of h."""
    h2 = h.reshape(-1, h.shape[-1])
    d2 = dy.reshape(-1, dy.shape[-1])
    return (d2 @ w).reshape(h.shape[:-1] + (w.shape[1],)), d2.T @ h2


def layer_norm_bwd(z: np.ndarray, gamma: np.ndarray, dy: np.ndarray, eps: float = block.LN_EPS):
    """Gradient of block.layer_norm (R3: biased variance, eps 1e-5, affine).

    Returns (dz, dgamma, dbeta); dgamma / dbeta summed over every token of z."""
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    sigma = np.sqrt(var + eps)
    xhat = (z - mu) / sigma
    C = z.shape[-1]
    dgamma = (dy * xhat).reshape(-1, C).sum(axis=0)
    dbeta = dy.reshape(-1, C).sum(axis=0)
    dxhat = dy * gamma
    dz = (dxhat - dxhat.mean(axis=-1, keepdims=True) - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True)) / sigma
    return dz, dgamma, dbeta


def gelu_tanh_bwd(u: np.ndarray, dg: np.ndarray) -> np.ndarray:
    """d/du of 0.5 u (1 + tanh(c (u + 0.044715 u^3))), c = sqrt(2/pi) (R5), times dg."""
    c = np.sqrt(2.0 / np.pi)
    t = np.tanh(c * (u + 0.044715 * u ** 3))
    return dg * (0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * c * (1.0 + 3.0 * 0.044715 * u * u))


def attention_core_bwd(q: np.ndarray, k: np.ndarray, v: np.ndarray, do: np.ndarray):
    """Gradient of block.attention_core (R6, R7) for q, k, v, do [NH, L, Dh]."""
    dh = q.shape[-1]
    a = (q @ np.swapaxes(k, -1, -2)) / np.sqrt(dh)
    a = a - a.max(axis=-1, keepdims=True)
    p = np.exp(a)
    p = p / p.sum(axis=-1, keepdims=True)
    dv = np.swapaxes(p, -1, -2) @ do
    dp = do @ np.swapaxes(v, -1, -2)
    da = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
    dq = (da @ k) / np.sqrt(dh)
    dk = (np.swapaxes(da, -1, -2) @ q) / np.sqrt(dh)
    return dq, dk, dv


def attention_lse(q: np.ndarray, k: np.ndarray) -> np.ndarray:
    """Row log-sum-exp of the scaled scores, natural log: log sum_j exp(q_i k_j / sqrt(Dh)),
    the softmax normaliser the backward needs (returned per head and row, [NH, L])."""
    a = (q @ np.swapaxes(k, -1, -2)) / np.sqrt(q.shape[-1])
    m = a.max(axis=-1, keepdims=True)
    return (m + np.log(np.exp(a - m).sum(axis=-1, keepdims=True)))[..., 0]


def mha_sequence_bwd(h: np.ndarray, w_qkv, w_o, num_heads: int, dout: np.ndarray):
    """Gradient of block.mha_sequence for ONE sequence h [L, C]: (dh, dw_qkv, dw_o)."""
    L, C = h.shape
    g = block.linear(h, w_qkv)
    q, k, v = block.split_heads(g, C, num_heads)
    o = block.attention_core(q, k, v)
    oc = o.transpose(1, 0, 2).reshape(L, C)
    doc, dw_o = linear_bwd(oc, w_o, dout)
    dh_ = C // num_heads
    do = doc.reshape(L, num_heads, dh_).transpose(1, 0, 2)
    dq, dk, dv = attention_core_bwd(q, k, v, do)
    merge = lambda t: t.transpose(1, 0, 2).reshape(L, C)
    dg = np.concatenate([merge(dq), merge(dk), merge(dv)], axis=1)     # [L, 3C], R8 layout
    dh, dw_qkv = linear_bwd(h, w_qkv, dg)
    return dh, dw_qkv, dw_o


def _zero_grads(W: dict, names) -> dict:
    return {n: np.zeros_like(W[n]) for n in names}


def spatial_stage_bwd(x: np.ndarray, W: dict, num_heads: int, dy1: np.ndarray):
    """Gradient of block.spatial_stage on [B, T', S, C] (whole frames): (dx, grads)."""
    gr = _zero_grads(W, ("w_qkv_s", "w_o_s"))
    h = block.layer_norm(x, W["ln1_w"], W["ln1_b"])
    dh = np.empty_like(h)
    for b in range(x.shape[0]):
        for t in range(x.shape[1]):
            dh[b, t], dq, do = mha_sequence_bwd(h[b, t], W["w_qkv_s"], W["w_o_s"], num_heads, dy1[b, t])
            gr["w_qkv_s"] += dq
            gr["w_o_s"] += do
    dz, gr["ln1_w"], gr["ln1_b"] = layer_norm_bwd(x, W["ln1_w"], dh)
    return dy1 + dz, gr


def temporal_stage_bwd(y1: np.ndarray, W: dict, num_heads: int, dy2: np.ndarray):
    """Gradient of block.temporal_stage on [B, T, S', C] (whole columns): (dy1, grads)."""
    gr = _zero_grads(W, ("w_qkv_t", "w_o_t"))
    h = block.layer_norm(y1, W["ln2_w"], W["ln2_b"])
    dh = np.empty_like(h)
    for b in range(y1.shape[0]):
        for s in range(y1.shape[2]):
            dh[b, :, s], dq, do = mha_sequence_bwd(h[b, :, s], W["w_qkv_t"], W["w_o_t"], num_heads, dy2[b, :, s])
            gr["w_qkv_t"] += dq
            gr["w_o_t"] += do
    dz, gr["ln2_w"], gr["ln2_b"] = layer_norm_bwd(y1, W["ln2_w"], dh)
    return dy2 + dz, gr


def mlp_stage_bwd(y2: np.ndarray, W: dict, dy: np.ndarray):
    """Gradient of block.mlp_stage (position-wise): (dy2, grads)."""
    gr = {}
    h = block.layer_norm(y2, W["ln3_w"], W["ln3_b"])
    u = block.linear(h, W["w_fc1"])
    g = block.gelu_tanh(u)
    dg, gr["w_fc2"] = linear_bwd(g, W["w_fc2"], dy)
    du = gelu_tanh_bwd(u, dg)
    dh, gr["w_fc1"] = linear_bwd(h, W["w_fc1"], du)
    dz, gr["ln3_w"], gr["ln3_b"] = layer_norm_bwd(y2, W["ln3_w"], dh)
    return dy + dz, gr


def st_block_bwd(x: np.ndarray, W: dict, num_heads: int, dy: np.ndarray):
    """Gradient of block.st_block (no cross stage) at x [B, T, S, C] for the upstream dy:
    (dx, {name: dW}) with the twelve weights of GRAD_NAMES."""
    y1 = block.spatial_stage(x, W, num_heads)
    y2 = block.temporal_stage(y1, W, num_heads)
    dy2, gm = mlp_stage_bwd(y2, W, dy)
    dy1, gt = temporal_stage_bwd(y1, W, num_heads, dy2)
    dx, gs = spatial_stage_bwd(x, W, num_heads, dy1)
    return dx, {**gs, **gt, **gm}


def simulate_sharded_bwd(x: np.ndarray, W: dict, num_heads: int, world: int, dy: np.ndarray):
    """The DSP schedule's backward over `world` simulated ranks (P:91-93 run in reverse).

    Forward (as sharded.simulate_sharded): T-shards -> spatial -> switch T->S -> temporal + MLP
    -> switch S->T.  Backward: dy split over T; the adjoint of the S->T switch is the T->S switch
    (a permutation's adjoint is its inverse); MLP and temporal backward local on S-shards; switch
    S->T (adjoint of T->S); spatial backward local on T-shards; every rank's weight gradients are
    summed over the ranks in rank order (the reduction ZeRO shards); dx gathered over T.
    Returns (dx, grads, per-rank T-sharded dx)."""
    xs = split(x, DIM_T, world)
    y1 = [block.spatial_stage(s, W, num_heads) for s in xs]
    y1s = switch(y1, DIM_T, DIM_S)
    y2 = [block.temporal_stage(s, W, num_heads) for s in y1s]
    dz = switch(split(dy, DIM_T, world), DIM_T, DIM_S)                  # adjoint of S->T
    grads = _zero_grads(W, GRAD_NAMES)
    dy1s = []
    for r in range(world):
        dy2_r, gm = mlp_stage_bwd(y2[r], W, dz[r])
        dy1_r, gt = temporal_stage_bwd(y1s[r], W, num_heads, dy2_r)
        dy1s.append(dy1_r)
        for n, v in {**gm, **gt}.items():
            grads[n] += v
    dy1 = switch(dy1s, DIM_S, DIM_T)                                    # adjoint of T->S
    dxs = []
    for r in range(world):
        dx_r, gs = spatial_stage_bwd(xs[r], W, num_heads, dy1[r])
        dxs.append(dx_r)
        for n, v in gs.items():
            grads[n] += v
    return gather(dxs, DIM_T), grads, dxs
