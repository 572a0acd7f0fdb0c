"""GPU tests of the DeepSpeed-Ulysses schedule on the same kernels.

N virtual ranks on one device (see test_gpu_block.VirtualGroup): the P2P transport stores into
the peers' buffers directly; the NCCL transport runs the library's pack / unpack kernels with the
all-to-all emulated over the peer mappings (dsp_ctx_set_collective_emulation).  Per-head attention
is the same arithmetic on the same values as the DSP block, so the Ulysses block over N ranks
equals the N = 1 block BITWISE; it is also checked against the oracle's Ulysses simulation.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import switch as osw
from oracle import ulysses as ou
from tests.gpu_util import assert_block_close, bits16, to_dev, to_f64, weights_dev, weights_f64
from tests.test_gpu_block import VirtualGroup, _run_block_n1, _setup

pytestmark = pytest.mark.gpu


def dsp():
    import paper_2403_10266_b200 as m
    return m


def _run_ulysses(sh, xs, Ws, N, impl, prepared):
    m = dsp()
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    ws = (m.ulysses_workspace_bytes(shape, N) + 1023) // 1024 * 1024
    act = sh.M * 2 // N
    g = VirtualGroup(N, ws + act)
    if impl == "nccl":
        for c in g.ctx:
            c.set_collective_emulation(True)
    W = weights_dev(Ws, "bf16")
    if prepared:
        W["prepared"] = g.ctx[0].prepare_block(shape, W)
        torch.cuda.synchronize()
    xsh = osw.split(xs, osw.DIM_T, N)
    X = [to_dev(xsh[r], "bf16").reshape(-1) for r in range(N)]
    Y = [g.view(r, ws, act, torch.bfloat16) for r in range(N)]
    for r in range(N):
        g.ctx[r].set_workspace(g.region[r][:ws])
    g.run(lambda r: g.ctx[r].st_block_forward_ulysses(shape, W, X[r], Y[r], impl=impl))
    for c in g.ctx:
        c.check_errors()
    return np.concatenate([bits16(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1), Y, g


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("impl", ["p2p", "nccl"])
@pytest.mark.parametrize("prepared", [False, True])
def test_ulysses_block_equals_dsp_n1_bitwise(N, impl, prepared):
    """configs[1] shape (T=16, S=1024, C=1152, 16 heads): Ulysses over N virtual ranks == the N = 1
    block bitwise (raw and prepared weights, both transports)."""
    sh = synth.CONFIGS["blk"]
    xs, Ws = _setup(sh)
    ref = bits16(_run_block_n1(sh, xs, Ws, prepared=prepared))
    got, _, _ = _run_ulysses(sh, xs, Ws, N, impl, prepared)
    assert np.array_equal(got.reshape(-1), ref.reshape(-1))


@pytest.mark.parametrize("N", [2, 4])
def test_ulysses_block_vs_oracle_ulysses(N):
    """B = 2 (non-trivial strides in every exchange), reduced shape, against the oracle's
    message-passing Ulysses simulation (itself pinned to the unsharded block and S:303)."""
    sh = synth.BlockShape(2, 8, 128, 256, 4, "bf16")
    xs, Ws = _setup(sh)
    got, Y, _ = _run_ulysses(sh, xs, Ws, N, "p2p", False)
    ref, _ = ou.simulate_ulysses(synth.to_f64(xs, "bf16"), weights_f64(Ws, "bf16"), sh.NH, N)
    gotf = np.concatenate([to_f64(Y[r]).reshape(sh.B, sh.T // N, sh.S, sh.C) for r in range(N)], axis=1)
    print(assert_block_close(gotf, ref))


def test_ulysses_rejects_heads_not_divisible():
    m = dsp()
    sh = synth.BlockShape(1, 8, 128, 384, 6, "bf16")  # 6 heads, N = 4
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, "bf16")
    c = m.Context(rank=0, world=4)
    c.ensure_workspace(m.ulysses_workspace_bytes(shape, 4))
    W = weights_dev(synth.make_block_weights(sh, 7), "bf16")
    X = torch.zeros(sh.M // 4, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(m.DSPError) as e:
        c.st_block_forward_ulysses(shape, W, X, torch.empty_like(X), impl="p2p")
    assert e.value.name == "DSP_ERR_UNSUPPORTED"
