"""Multi-dimensional transformer block and its DSP schedule, float64 numpy (TEST INFRASTRUCTURE ONLY).

P:44-46: multi-dimensional transformers apply self-attention "along the spatial height and
width dimensions of each video frame, as well as the temporal dimension across frames"; P:93:
DSP "can generalize to all multi-dimensional transformers beyond the demonstrated
spatial-temporal transformer".  Block on x [d_0, ..., d_{n-2}, C] with attention stages along
the dims `order` (each once, pre-LN + residual, R1-R8 as for the ST block), then the MLP:

    for k in order:  x = x + MHA_k(LN_k(x))        one sequence along dim k per index of the others
    y = x + MLP(LN_mlp(x))

DSP schedule (same rule as the 4-D block, R10/R13): enter sharded on `shard_dim`; every stage
whose dim is not the sharded one is local; before the stage along the sharded dim, ONE switch
to the most recently attended dim (never attended again in the block); after the MLP, switch
back so every block enters and leaves on `shard_dim`.  Requires shard_dim != order[0].
"""
from __future__ import annotations

import numpy as np

from . import block
from .switch import Ledger, split_nd, switch_nd


def mha_along(h: np.ndarray, w_qkv, w_o, num_heads: int, axis: int) -> np.ndarray:
    """Self-attention along `axis` of h [..., C]: one sequence per index of all other non-channel
    dims, each through block.mha_sequence (the same per-sequence function as the ST block)."""
    hm = np.moveaxis(h, axis, -2)                    # [..., L, C]
    out = np.empty_like(hm)
    for idx in np.ndindex(*hm.shape[:-2]):
        out[idx] = block.mha_sequence(hm[idx], w_qkv, w_o, num_heads)
    return np.moveaxis(out, -2, axis)


def attn_stage(x, Wk: dict, num_heads: int, axis: int):
    """x + MHA_axis(LN(x)) with Wk = {ln_w, ln_b, w_qkv, w_o}."""
    return x + mha_along(block.layer_norm(x, Wk["ln_w"], Wk["ln_b"]), Wk["w_qkv"], Wk["w_o"], num_heads, axis)


def mlp_stage(x, Wm: dict):
    return x + block.mlp(block.layer_norm(x, Wm["ln_w"], Wm["ln_b"]), Wm["w_fc1"], Wm["w_fc2"])


def nd_block(x: np.ndarray, order, stages: list, Wm: dict, num_heads: int) -> np.ndarray:
    """The unsharded N-D block: stages[i] are the weights of the attention along order[i]."""
    for axis, Wk in zip(order, stages):
        x = attn_stage(x, Wk, num_heads, axis)
    return mlp_stage(x, Wm)


def simulate_sharded_nd(x: np.ndarray, order, stages: list, Wm: dict, num_heads: int, world: int, shard_dim: int,
                        ledger: Ledger | None = None, elem_bytes: int = 2):
    """split along shard_dim -> per-rank local stages -> message-passing N-D switches -> per-rank
    shards on shard_dim again.  Returns the list of per-rank output shards."""
    if shard_dim == order[0]:
        raise ValueError("DSP schedule: the first attended dim cannot be the sharded one")
    shards = split_nd(x, shard_dim, world)
    cur = shard_dim
    done = []
    for axis, Wk in zip(order, stages):
        if axis == cur:
            alt = done[-1]                               # most recently attended: never needed again
            shards = switch_nd(shards, cur, alt, ledger, f"switch_{cur}to{alt}", elem_bytes)
            cur = alt
        shards = [attn_stage(s, Wk, num_heads, axis) for s in shards]
        done.append(axis)
    shards = [mlp_stage(s, Wm) for s in shards]
    if cur != shard_dim:
        shards = switch_nd(shards, cur, shard_dim, ledger, f"switch_{cur}to{shard_dim}", elem_bytes)
    return shards
