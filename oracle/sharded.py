"""DSP schedule over N simulated ranks (TEST INFRASTRUCTURE ONLY).

P:91-93 (§3.1): "when calculating the spatial transformer block, the
computation is independent of the temporal sequence dimension, and the data can
be split across devices without affecting the results ... dynamically switch
the dimension of sequence parallelism according to the computation stage".
Schedule (R10, R13, R14): enter T-sharded; spatial stage local on T-shards;
switch T->S; temporal stage + MLP local on S-shards; switch S->T; exit T-sharded.
Each rank runs exactly the same per-sequence functions as `block.st_block`.
"""
from __future__ import annotations

import numpy as np

from . import block
from .switch import DIM_S, DIM_T, Ledger, gather, split, switch


def simulate_sharded(x: np.ndarray, W: dict, num_heads: int, world: int,
                     ledger: Ledger | None = None, elem_bytes: int = 2, tag: str = "block0",
                     mlp_before_switch: bool = True, ctx: np.ndarray | None = None):
    """split -> per-rank stages -> message-passing switches -> gather.

    Returns (gathered output, list of per-rank T-sharded outputs).
    `mlp_before_switch=False` runs the position-wise MLP after the S->T switch
    instead (R14: both placements must agree bit-for-bit).
    """
    shards = split(x, DIM_T, world)                                   # a0
    y1 = [block.spatial_stage(s, W, num_heads) for s in shards]      # a1-a4
    y1s = switch(y1, DIM_T, DIM_S, ledger, f"{tag}.switch_T2S", elem_bytes)   # a5
    y2 = [block.temporal_stage(s, W, num_heads) for s in y1s]        # a6-a9
    if ctx is not None:  # ST-DiT cross stage: position-independent, local on S-shards
        Wc = dict(ln_w=W["ln_c_w"], ln_b=W["ln_c_b"], w_q=W["w_q_c"], w_kv=W["w_kv_c"], w_o=W["w_o_c"])
        y2 = [block.cross_stage(s, ctx, Wc, num_heads) for s in y2]
    if mlp_before_switch:
        y = [block.mlp_stage(s, W) for s in y2]                      # a10
        out = switch(y, DIM_S, DIM_T, ledger, f"{tag}.switch_S2T", elem_bytes)  # a11
    else:
        y2t = switch(y2, DIM_S, DIM_T, ledger, f"{tag}.switch_S2T", elem_bytes)
        out = [block.mlp_stage(s, W) for s in y2t]
    return gather(out, DIM_T, ledger, "epilogue", elem_bytes), out   # a12
