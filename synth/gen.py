"""Counter-based SplitMix64 generator for the synthetic DSP workload.

No method arithmetic lives here (see synth/__init__.py). Everything is numpy,
vectorised over flat indices, and deterministic across platforms.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# Per-layer weight order; tensor id of weight k in layer l is 16*l + 1 + k, x is 0.
WEIGHT_NAMES = (
    "ln1_w", "ln1_b", "w_qkv_s", "w_o_s",
    "ln2_w", "ln2_b", "w_qkv_t", "w_o_t",
    "ln3_w", "ln3_b", "w_fc1", "w_fc2",
)
TENSOR_IDS = {"x": 0, **{n: 1 + k for k, n in enumerate(WEIGHT_NAMES)}}


def tensor_id(name: str, layer: int = 0) -> int:
    if name == "x":
        return 0
    return 16 * layer + TENSOR_IDS[name]


def splitmix64(key: np.ndarray) -> np.ndarray:
    """SplitMix64 output function applied to (key + golden gamma). uint64 in/out."""
    z = np.asarray(key, dtype=np.uint64) + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _keys(seed: int, tid: int, idx: np.ndarray) -> np.ndarray:
    assert 0 <= seed < (1 << 20) and 0 <= tid < (1 << 12)
    idx = np.asarray(idx, dtype=np.uint64)
    return (np.uint64(seed) << np.uint64(44)) ^ (np.uint64(tid) << np.uint64(32)) ^ idx


def uniform_pm1(seed: int, tid: int, idx: np.ndarray) -> np.ndarray:
    """v = 2*(z>>40)*2^-24 - 1 in [-1, 1) as float64 (each value exact in float32)."""
    z = splitmix64(_keys(seed, tid, idx))
    return (z >> np.uint64(40)).astype(np.float64) * (2.0 ** -23) - 1.0


def round_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float64/float32 -> bf16 bit patterns (uint16), round to nearest even."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = u + np.uint64(0x7FFF) + lsb
    return (u >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


@dataclasses.dataclass(frozen=True)
class BlockShape:
    """Global shape of one ST block activation [B, T, S, C] with NH heads."""
    B: int
    T: int
    S: int
    C: int
    NH: int
    dtype: str = "bf16"  # "bf16" or "f32"

    @property
    def M(self) -> int:
        return self.B * self.T * self.S * self.C

    @property
    def Dh(self) -> int:
        return self.C // self.NH

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4


CONFIGS = {
    # BASELINE.json configs[0..3]
    "tiny": BlockShape(1, 4, 16, 64, 4, "f32"),
    "blk": BlockShape(1, 16, 1024, 1152, 16, "bf16"),
    "long": BlockShape(1, 128, 4096, 1152, 16, "bf16"),
}


def _store(vals: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return round_to_bf16_bits(vals)
    if dtype == "f32":
        return vals.astype(np.float32)
    raise ValueError(dtype)


def to_f64(stored: np.ndarray, dtype: str) -> np.ndarray:
    """Widen stored values (bf16 bits or float32) to float64 exactly."""
    if dtype == "bf16":
        return bf16_bits_to_f64(stored)
    return np.asarray(stored, dtype=np.float64)


def make_x(shape: BlockShape, seed: int, t_range=None, s_range=None) -> np.ndarray:
    """x[B, T, S, C] (or the [t0:t1, s0:s1] slice of it) from global flat indices."""
    B, T, S, C = shape.B, shape.T, shape.S, shape.C
    t0, t1 = t_range or (0, T)
    s0, s1 = s_range or (0, S)
    b = np.arange(B, dtype=np.uint64)[:, None, None, None]
    t = np.arange(t0, t1, dtype=np.uint64)[None, :, None, None]
    s = np.arange(s0, s1, dtype=np.uint64)[None, None, :, None]
    c = np.arange(C, dtype=np.uint64)[None, None, None, :]
    idx = ((b * np.uint64(T) + t) * np.uint64(S) + s) * np.uint64(C) + c
    return _store(uniform_pm1(seed, 0, idx), shape.dtype)


def make_block_weights(shape: BlockShape, seed: int, layer: int = 0, kappa: float = 1.0) -> dict:
    """Weights of one block in nn.Linear [out, in] layout, stored dtype.

    Scales: LN gamma 1+0.1v, beta 0.1v; Wq, Wk rows
    v*sqrt(3*kappa/C) (score std ~ kappa after LN); Wv, Wo, W1 v*sqrt(3/C);
    W2 0.5*v*sqrt(3/(4C)).
    """
    C = shape.C
    out = {}

    def u(name, n):
        return uniform_pm1(seed, tensor_id(name, layer), np.arange(n, dtype=np.uint64))

    for i in (1, 2, 3):
        out[f"ln{i}_w"] = 1.0 + 0.1 * u(f"ln{i}_w", C)
        out[f"ln{i}_b"] = 0.1 * u(f"ln{i}_b", C)
    for st in ("s", "t"):
        w = u(f"w_qkv_{st}", 3 * C * C).reshape(3 * C, C)
        w[: 2 * C] *= math.sqrt(3.0 * kappa / C)
        w[2 * C:] *= math.sqrt(3.0 / C)
        out[f"w_qkv_{st}"] = w
        out[f"w_o_{st}"] = u(f"w_o_{st}", C * C).reshape(C, C) * math.sqrt(3.0 / C)
    out["w_fc1"] = u("w_fc1", 4 * C * C).reshape(4 * C, C) * math.sqrt(3.0 / C)
    out["w_fc2"] = u("w_fc2", 4 * C * C).reshape(C, 4 * C) * (0.5 * math.sqrt(3.0 / (4 * C)))
    return {k: _store(v, shape.dtype) for k, v in out.items()}


CROSS_NAMES = ("ln_c_w", "ln_c_b", "w_q_c", "w_kv_c", "w_o_c")


def make_cross_weights(shape: BlockShape, seed: int, layer: int = 0, kappa: float = 1.0) -> dict:
    """Cross-attention weights of one block (ST-DiT's text conditioning): LN_c gamma/beta,
    w_q_c [C, C], w_kv_c [2C, C] ([k | v] rows), w_o_c [C, C].  Tensor ids 3000 + 8*layer + k
    (disjoint from the 16*layer + k self-attention / MLP ids).  Scales as for self-attention."""
    C = shape.C

    def u(k, n):
        return uniform_pm1(seed, 3000 + 8 * layer + k, np.arange(n, dtype=np.uint64))

    out = {"ln_c_w": 1.0 + 0.1 * u(0, C), "ln_c_b": 0.1 * u(1, C),
           "w_q_c": u(2, C * C).reshape(C, C) * math.sqrt(3.0 * kappa / C)}
    kv = u(3, 2 * C * C).reshape(2 * C, C)
    kv[:C] *= math.sqrt(3.0 * kappa / C)
    kv[C:] *= math.sqrt(3.0 / C)
    out["w_kv_c"] = kv
    out["w_o_c"] = u(4, C * C).reshape(C, C) * math.sqrt(3.0 / C)
    return {k: _store(v, shape.dtype) for k, v in out.items()}


def make_context(shape: BlockShape, seed: int, ctx_len: int) -> np.ndarray:
    """Synthetic caption embeddings [B, ctx_len, C] (already projected to C; tensor id 4000),
    uniform in [-1, 1) like x -- the paper's text encoder and captions are out of scope."""
    n = shape.B * ctx_len * shape.C
    return _store(uniform_pm1(seed, 4000, np.arange(n, dtype=np.uint64)).reshape(shape.B, ctx_len, shape.C),
                  shape.dtype)


def zero_block_weights(shape: BlockShape) -> dict:
    C = shape.C
    dims = {"ln1_w": (C,), "ln1_b": (C,), "ln2_w": (C,), "ln2_b": (C,), "ln3_w": (C,), "ln3_b": (C,),
            "w_qkv_s": (3 * C, C), "w_o_s": (C, C), "w_qkv_t": (3 * C, C), "w_o_t": (C, C),
            "w_fc1": (4 * C, C), "w_fc2": (C, 4 * C)}
    return {k: _store(np.zeros(v), shape.dtype) for k, v in dims.items()}


def make_index_tagged(shape: BlockShape, seed: int, t_range=None, s_range=None) -> np.ndarray:
    """2-byte-element tensor whose token row (b,t,s) carries its global token index.

    c=0: low 16 bits of g=(b*T+t)*S+s, c=1: high 16 bits, c>=2: hash bits. Returned
    as uint16 so comparisons are bitwise (never float ==).
    """
    B, T, S, C = shape.B, shape.T, shape.S, shape.C
    assert C >= 2
    t0, t1 = t_range or (0, T)
    s0, s1 = s_range or (0, S)
    b = np.arange(B, dtype=np.uint64)[:, None, None, None]
    t = np.arange(t0, t1, dtype=np.uint64)[None, :, None, None]
    s = np.arange(s0, s1, dtype=np.uint64)[None, None, :, None]
    c = np.arange(C, dtype=np.uint64)[None, None, None, :]
    g = (b * np.uint64(T) + t) * np.uint64(S) + s
    idx = g * np.uint64(C) + c
    h = (splitmix64(_keys(seed, 0xFFF, idx)) & np.uint64(0xFFFF))
    v = np.where(c == 0, g & np.uint64(0xFFFF), np.where(c == 1, (g >> np.uint64(16)) & np.uint64(0xFFFF), h))
    return v.astype(np.uint16)


LATTE_NAMES = ("ln_m_w", "ln_m_b", "w_fc1_s", "w_fc2_s")


def make_latte_weights(shape: BlockShape, seed: int, layer: int = 0) -> dict:
    """The Latte pair's spatial MLP (R38): LN_m gamma / beta, w_fc1_s [4C, C], w_fc2_s
    [C, 4C]; tensor ids 1000 + 8*layer + k; scales as the block's MLP."""
    C = shape.C

    def u(k, n):
        return uniform_pm1(seed, 1000 + 8 * layer + k, np.arange(n, dtype=np.uint64))

    out = {"ln_m_w": 1.0 + 0.1 * u(0, C), "ln_m_b": 0.1 * u(1, C),
           "w_fc1_s": u(2, 4 * C * C).reshape(4 * C, C) * math.sqrt(3.0 / C),
           "w_fc2_s": u(3, 4 * C * C).reshape(C, 4 * C) * (0.5 * math.sqrt(3.0 / (4 * C)))}
    return {k: _store(v, shape.dtype) for k, v in out.items()}


def make_modulation(shape: BlockShape, seed: int, layer: int = 0, sublayers=("s", "t", "m")) -> dict:
    """adaLN-Zero modulation (R36) of sample b: {sublayer: (shift, scale, gate)}, each
    [B, C] float32 (the per-step conditioning, already through SiLU + Linear): shift = 0.1 v,
    scale = 0.1 v, gate = 1 + 0.25 v (a trained, non-zero gate).  Tensor ids 1500 + 16*layer + 4*i + j."""
    B, C = shape.B, shape.C
    out = {}
    for i, k in enumerate(sublayers):
        def u(j):
            return uniform_pm1(seed, 1500 + 16 * layer + 4 * i + j, np.arange(B * C, dtype=np.uint64)).reshape(B, C)
        out[k] = ((0.1 * u(0)).astype(np.float32), (0.1 * u(1)).astype(np.float32),
                  (1.0 + 0.25 * u(2)).astype(np.float32))
    return out


def make_temporal_pe(shape: BlockShape) -> np.ndarray:
    """Sinusoidal temporal positional embedding [T, C] (R37, Latte / "Attention is all
    you need" table): pe[t, 2i] = sin(t / 10000^(2i/C)), pe[t, 2i+1] = cos(...), stored dtype."""
    T, C = shape.T, shape.C
    t = np.arange(T, dtype=np.float64)[:, None]
    i = np.arange(C // 2, dtype=np.float64)[None, :]
    ang = t / np.power(10000.0, 2.0 * i / C)
    pe = np.empty((T, C))
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang)
    return _store(pe, shape.dtype)
