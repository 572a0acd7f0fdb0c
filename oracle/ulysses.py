"""DeepSpeed-Ulysses schedule of the ST block over N simulated ranks (TEST INFRASTRUCTURE ONLY).

The comparison system of the paper: "DeepSpeed-Ulysses ... uses AlltoAll
for query, key, value, and output" around every attention layer, 8M/N per ST block (Table 1,
P:112-115).  Written from that description, as message passing between simulated ranks with a
byte ledger, like `switch.switch`:

* the activation stays sharded along T (the flattened T*S sequence in contiguous chunks, rank r
  holding frames [r*T/N, (r+1)*T/N)), exactly as the DSP block enters and leaves;
* per attention stage: LN and the q/k/v projection are local; q, k and v are each exchanged
  sequence-sharded -> head-sharded (rank g receives head group g = channels [g*C/N, (g+1)*C/N)
  of every token); attention over the full sequence with NH/N heads; o is exchanged back
  head-sharded -> sequence-sharded; the out-projection and residual are local;
* the MLP is local.

Each rank runs the same per-head arithmetic as `block.st_block` on the same values, so the
gathered output equals the unsharded block (up to BLAS blocking of the projections, R27).
"""
from __future__ import annotations

import numpy as np

from . import block
from .switch import DIM_T, Ledger, gather, split


def seq_to_head(parts: list, num_heads: int, ledger: Ledger | None, tag: str, elem_bytes: int = 2) -> list:
    """All-to-all of one tensor [B, T/N, S, C] per rank -> [B, T, S, C/N] per rank: rank r sends
    head group g of its tokens to rank g, which concatenates the pieces along T in rank order."""
    N = len(parts)
    C = parts[0].shape[-1]
    if C % N or num_heads % N:
        raise ValueError(f"Ulysses needs N | C and N | num_heads (N={N}, C={C}, heads={num_heads})")
    cn = C // N
    outbox = [[np.array(parts[r][..., g * cn:(g + 1) * cn], copy=True) for g in range(N)] for r in range(N)]
    out = [np.concatenate([outbox[r][g] for r in range(N)], axis=DIM_T) for g in range(N)]
    _record(ledger, outbox, tag, elem_bytes)
    return out


def head_to_seq(parts: list, ledger: Ledger | None, tag: str, elem_bytes: int = 2) -> list:
    """All-to-all of one tensor [B, T, S, C/N] per rank (head group g on rank g) -> [B, T/N, S, C]:
    rank g sends frames [r*T/N, (r+1)*T/N) of its head group to rank r, which concatenates the
    pieces along channels in head-group order."""
    N = len(parts)
    tn = parts[0].shape[DIM_T] // N
    outbox = [[np.array(parts[g][:, r * tn:(r + 1) * tn], copy=True) for r in range(N)] for g in range(N)]
    out = [np.concatenate([outbox[g][r] for g in range(N)], axis=-1) for r in range(N)]
    _record(ledger, outbox, tag, elem_bytes)
    return out


def _record(ledger, outbox, tag, elem_bytes):
    if ledger is None:
        return
    N = len(outbox)
    for r in range(N):
        sent = sum(outbox[r][q].size for q in range(N) if q != r)
        recv = sum(outbox[q][r].size for q in range(N) if q != r)
        ledger.record(r, "AllToAll", tag, sent, recv, sent * elem_bytes, recv * elem_bytes)


def _attention(x: np.ndarray, num_heads: int, axis: str) -> np.ndarray:
    """q, k, v [B, T, S, 3*Cg] of one head group (NHg heads) -> attention output [B, T, S, Cg], one
    sequence per (b, t) over S (spatial) or per (b, s) over T (temporal)."""
    B, T, S, C3 = x.shape
    cg = C3 // 3
    out = np.empty((B, T, S, cg))
    seqs = [(b, t) for b in range(B) for t in range(T)] if axis == "S" else [(b, s) for b in range(B) for s in range(S)]
    for b, i in seqs:
        g = x[b, i] if axis == "S" else x[b, :, i]
        q, k, v = block.split_heads(g, cg, num_heads)
        o = block.attention_core(q, k, v).transpose(1, 0, 2).reshape(g.shape[0], cg)
        if axis == "S":
            out[b, i] = o
        else:
            out[b, :, i] = o
    return out


def ulysses_attention_stage(xs: list, ln_w, ln_b, w_qkv, w_o, num_heads: int, axis: str,
                            ledger: Ledger | None, tag: str, elem_bytes: int = 2) -> list:
    """y_r = x_r + MHA_axis(LN x)_r with the four all-to-alls of DeepSpeed-Ulysses."""
    N = len(xs)
    C = xs[0].shape[-1]
    qkv = [block.linear(block.layer_norm(x, ln_w, ln_b), w_qkv) for x in xs]       # local projection
    heads = [seq_to_head([p[..., i * C:(i + 1) * C] for p in qkv], num_heads, ledger, f"{tag}.a2a_{n}", elem_bytes)
             for i, n in enumerate("qkv")]                                          # 3 all-to-alls
    o_h = [_attention(np.concatenate([heads[0][g], heads[1][g], heads[2][g]], axis=-1), num_heads // N, axis)
           for g in range(N)]                                                       # full sequence, NH/N heads
    o = head_to_seq(o_h, ledger, f"{tag}.a2a_o", elem_bytes)                        # 4th all-to-all
    return [x + block.linear(oo, w_o) for x, oo in zip(xs, o)]


def simulate_ulysses(x: np.ndarray, W: dict, num_heads: int, world: int, ledger: Ledger | None = None,
                     elem_bytes: int = 2, tag: str = "block0"):
    """split (T) -> per-rank Ulysses attention stages (spatial, temporal) -> local MLP -> gather.
    Returns (gathered output, list of per-rank T-sharded outputs)."""
    shards = split(x, DIM_T, world)
    y1 = ulysses_attention_stage(shards, W["ln1_w"], W["ln1_b"], W["w_qkv_s"], W["w_o_s"], num_heads, "S",
                                 ledger, f"{tag}.spatial", elem_bytes)
    y2 = ulysses_attention_stage(y1, W["ln2_w"], W["ln2_b"], W["w_qkv_t"], W["w_o_t"], num_heads, "T",
                                 ledger, f"{tag}.temporal", elem_bytes)
    out = [block.mlp_stage(s, W) for s in y2]
    return gather(out, DIM_T, ledger, "epilogue", elem_bytes), out
