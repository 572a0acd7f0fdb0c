"""Pins for oracle/volume.py and the measured ledger against §3.2 / Table 1."""
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import sharded, volume
from oracle.switch import Ledger


def test_spec_volume_numbers(golden):
    for ln in golden("spec_volumes.txt"):
        kind, M, N, na, nm, want = ln.split()
        assert volume.predict_volume(kind, int(M), int(N), int(na), int(nm)) == int(want)


def test_measured_dsp_ledger_matches_spec_S294():
    """Run the simulated DSP block at B=1,T=4,S=4,D=8 (M=128), N=2: ledger = 64 elements."""
    sh = synth.BlockShape(1, 4, 4, 8, 2, "f32")
    x = synth.to_f64(synth.make_x(sh, 7), "f32")
    W = {k: synth.to_f64(v, "f32") for k, v in synth.make_block_weights(sh, 7).items()}
    led = Ledger()
    sharded.simulate_sharded(x, W, sh.NH, 2, led, elem_bytes=4)
    assert led.sent(0) == 64 and led.sent(1) == 64
    assert led.ops(0, "AllToAll") == 2
    assert led.sent(0, exclude_tags=()) == 64 + 64          # epilogue gather tagged separately


@pytest.mark.parametrize("N", [2, 4, 8, 16, 64])
def test_ratios_and_table1(N, golden):
    M = 1 * 16 * 1024 * 1152
    dsp = volume.predict_volume("dsp", M, N)
    uly = volume.predict_volume("ulysses", M, N)
    assert Fraction(dsp, uly) == Fraction(1, 4)             # S:305, E3 ">= 75% less"
    meg = volume.predict_volume("megatron", M, N, 2, 2)
    assert Fraction(uly, meg) == Fraction(1, N)             # Ulysses:Megatron = 1:N
    for ln in golden("table1.txt"):
        kind, coef, pw = ln.split()
        want = Fraction(int(coef)) * M * Fraction(N) ** int(pw)
        assert volume.asymptote(kind, M, N) == want, kind
    # exact -> asymptote within 2% at N = 64
    if N == 64:
        assert abs(dsp / float(volume.asymptote("dsp", M, N)) - 1) < 0.02


def test_op_counts(golden):
    g = dict(ln.split() for ln in golden("paper_ops.txt"))
    assert volume.op_count("dsp", 8) == int(g["dsp_alltoall_per_block"])
    assert volume.ops_per_attention_stage("ulysses") == int(g["ulysses_alltoall_per_attention"])
    assert volume.op_count("megatron", 8, n_attn=1, n_mlp=1) == int(g["megatron_collectives_per_transformer_block"])
    reds = sorted([volume.op_reduction("megatron"), volume.op_reduction("ulysses")])
    assert reds == [Fraction(int(g["reduction_min_percent"]), 100), Fraction(int(g["reduction_max_percent"]), 100)]


def test_n1_zero_communication():
    for k in ("dsp", "ulysses", "megatron", "ring"):
        assert volume.predict_volume(k, 4096, 1) == 0
