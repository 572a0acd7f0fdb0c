"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no LayerNorm, attention, MLP or
switch logic). It only turns (seed, tensor id, global flat index) into values,
so that the CPU oracle (`oracle/`) and the GPU path see bit-identical inputs and
any rank can generate its own shard from global indices.

Recipe:
  key = (seed << 44) ^ (tid << 32) ^ i          i < 2**32 global flat index
  z   = SplitMix64 finaliser of (key + 0x9E3779B97F4A7C15)
  v   = 2 * (z >> 40) * 2**-24 - 1              in [-1, 1), exactly a float32
Scales are applied in float64, then values are rounded to the storage dtype
(bf16 round-to-nearest-even, or float32), and the oracle consumes those rounded
values widened to float64.
"""
from .gen import (  # noqa: F401
    splitmix64, uniform_pm1, round_to_bf16_bits, bf16_bits_to_f64, to_f64,
    TENSOR_IDS, WEIGHT_NAMES, CONFIGS, BlockShape, make_x, make_block_weights,
    zero_block_weights, make_index_tagged, tensor_id, CROSS_NAMES, make_cross_weights, make_context,
    LATTE_NAMES, make_latte_weights, make_modulation, make_temporal_pe,
)
