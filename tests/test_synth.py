"""Pins for the shared seeded input generator (synth/)."""
import numpy as np
import pytest
import torch

import synth


def test_splitmix64_reference_sequence(golden):
    want = [int(v, 16) for v in golden("splitmix64_seed0.txt")]
    keys = np.arange(len(want), dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    got = [int(v) for v in synth.splitmix64(keys)]
    assert got == want


def test_uniform_determinism_range_seed():
    idx = np.arange(100000, dtype=np.uint64)
    a = synth.uniform_pm1(7, 3, idx)
    b = synth.uniform_pm1(7, 3, idx)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1 / np.sqrt(3)) < 0.01
    assert not np.array_equal(a, synth.uniform_pm1(8, 3, idx))
    assert not np.array_equal(a, synth.uniform_pm1(7, 4, idx))
    # every value is exactly a float32
    assert np.array_equal(a.astype(np.float32).astype(np.float64), a)


def test_bf16_rounding_matches_torch():
    v = synth.uniform_pm1(1, 1, np.arange(50000, dtype=np.uint64)) * 3.7
    ours = synth.round_to_bf16_bits(v)
    ref = torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    back = synth.bf16_bits_to_f64(ours)
    assert np.array_equal(back, torch.from_numpy(v.astype(np.float32)).to(torch.bfloat16).double().numpy())


def test_shard_generation_equals_global_slice():
    sh = synth.BlockShape(2, 8, 12, 16, 2, "bf16")
    x = synth.make_x(sh, 7)
    assert np.array_equal(x[:, 2:4], synth.make_x(sh, 7, t_range=(2, 4)))
    assert np.array_equal(x[:, :, 3:9], synth.make_x(sh, 7, s_range=(3, 9)))


def test_index_tagged_decodes_token_index():
    sh = synth.BlockShape(2, 4, 6, 8, 2, "bf16")
    x = synth.make_index_tagged(sh, 3).astype(np.int64)
    g = x[..., 0] | (x[..., 1] << 16)
    assert np.array_equal(g.reshape(-1), np.arange(2 * 4 * 6))


def test_weights_scales():
    sh = synth.BlockShape(1, 2, 2, 64, 4, "f32")
    W = synth.make_block_weights(sh, 7, kappa=1.0)
    C = sh.C
    assert W["w_qkv_s"].shape == (3 * C, C) and W["w_fc2"].shape == (C, 4 * C)
    assert np.abs(W["w_qkv_s"][:C]).max() <= np.sqrt(3 / C) + 1e-7
    assert np.abs(W["ln1_w"] - 1).max() <= 0.1 + 1e-7
    assert not np.array_equal(W["w_qkv_s"], W["w_qkv_t"])   # distinct tensor ids
