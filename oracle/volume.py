"""Communication-volume analysis of §3.2 / Table 1 (TEST INFRASTRUCTURE ONLY).

P:99: Megatron-SP "employs 4 ... collective communication operations per
transformer block ... a total communication volume of 8M"; DeepSpeed-Ulysses
uses AlltoAll "for query, key, value, and output ... 8M/N".
P:101: DSP employs "only two AlltoAll operations in total ... communication
volume to 2M/N".  Table 1: Ring 4M, Megatron-SP 8M, Ulysses 8M/N,
DSP 2M/N.

Convention (R16): elements SENT per device per ST block (one spatial
+ one temporal attention stage), forward, self-chunk excluded.  Exact
values carry the (N-1)/N factor; Table 1 is the N -> infinity asymptote of
exact * N/(N-1) ... see `asymptote`.
"""
from __future__ import annotations

from fractions import Fraction


def per_switch_elements(M: int, N: int) -> int:
    """One all-to-all of an M-element activation: (N-1) * M / N^2 elements sent per rank."""
    v = Fraction((N - 1) * M, N * N)
    assert v.denominator == 1
    return int(v)


def predict_volume(kind: str, M: int, N: int, n_attn: int = 2, n_mlp: int = 1) -> int:
    """Exact elements sent per rank per block, forward (R16).

    dsp      : 2 switches                    -> 2 (N-1) M / N^2
    ulysses  : 4 a2a (q,k,v,o) per attention -> 4 n_attn (N-1) M / N^2
    megatron : AG + RS per attn/MLP layer    -> 2 (n_attn + n_mlp) (N-1) M / N
    ring     : K and V around the ring        -> 2 n_attn (N-1) M / N
    """
    if kind == "dsp":
        v = Fraction(2 * (N - 1) * M, N * N)
    elif kind == "ulysses":
        v = Fraction(4 * n_attn * (N - 1) * M, N * N)
    elif kind == "megatron":
        v = Fraction(2 * (n_attn + n_mlp) * (N - 1) * M, N)
    elif kind == "ring":
        v = Fraction(2 * n_attn * (N - 1) * M, N)
    else:
        raise ValueError(kind)
    assert v.denominator == 1, (kind, M, N)
    return int(v)


def op_count(kind: str, N: int, n_attn: int = 2, n_mlp: int = 1) -> int:
    """Collectives per block (forward): DSP 2; Ulysses 4 per attention;
    Megatron-SP AG+RS per layer (4 per transformer block); Ring 2(N-1) rounds
    per attention (K and V)."""
    return {"dsp": 2, "ulysses": 4 * n_attn, "megatron": 2 * (n_attn + n_mlp),
            "ring": 2 * (N - 1) * n_attn}[kind]


def ops_per_attention_stage(kind: str) -> int:
    """Reading R18: per attention stage, Megatron-SP 2 (AG+RS), Ulysses 4 (q,k,v,o), DSP 1."""
    return {"dsp": 1, "megatron": 2, "ulysses": 4}[kind]


def op_reduction(vs: str) -> Fraction:
    """Fractional reduction of DSP's per-stage op count vs another method (P:101 '50% to 75%')."""
    return 1 - Fraction(ops_per_attention_stage("dsp"), ops_per_attention_stage(vs))


def asymptote(kind: str, M: int, N: int) -> Fraction:
    """Table 1 entries: exact value with (N-1)/N -> 1 (Latte pair for Megatron: n_mlp = 2)."""
    n_mlp = 2 if kind == "megatron" else 1
    exact = Fraction(predict_volume(kind, M, N, 2, n_mlp))
    return exact * Fraction(N, N - 1)


TABLE1 = {  # P:112-115, as (coefficient, power of N): volume = coef * M * N^power
    "ring": (4, 0),
    "megatron": (8, 0),
    "ulysses": (8, -1),
    "dsp": (2, -1),
}
