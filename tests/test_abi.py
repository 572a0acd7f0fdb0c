"""CPU tests of the C ABI: the library loads, exports every symbol include/*.h declares,
and its host-only functions (volume, plan, workspace, validation) are right.  No GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import synth
from oracle import switch as osw
from oracle import volume

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dsp():
    import paper_2403_10266_b200 as m
    return m


def declared_symbols():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(dsp_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    L = dsp().lib()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", dsp().LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", nm, re.M), n


def test_abi_version_and_status_strings():
    L = dsp().lib()
    assert L.dsp_abi_version() == 6
    for code, name in dsp().STATUS.items():
        assert L.dsp_status_str(code).decode() == name


@pytest.mark.parametrize("cfg", ["tiny", "blk", "long"])
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_switch_volume_matches_paper_analysis(cfg, N):
    m = dsp()
    sh = synth.CONFIGS[cfg]
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    if sh.T % N or sh.S % N:
        with pytest.raises(m.DSPError) as e:
            m.switch_volume(shape, N)
        assert e.value.name == "DSP_ERR_DIVISIBILITY"
        return
    sent, recv = m.switch_volume(shape, N)
    assert sent == recv == volume.per_switch_elements(sh.M, N) * sh.elem_bytes
    # two switches per block = DSP's 2(N-1)M/N^2 (Table 1)
    assert 2 * sent == volume.predict_volume("dsp", sh.M, N) * sh.elem_bytes


def test_switch_plan_validation_errors():
    m = dsp()
    shape = m.make_shape(1, 16, 1024, 1152, 16, "bf16")
    for args, name in [((2, 0, "T", "T"), "DSP_ERR_SAME_DIM"), ((3, 0, "T", "S"), "DSP_ERR_DIVISIBILITY"),
                       ((2, 5, "T", "S"), "DSP_ERR_SHAPE")]:
        with pytest.raises(m.DSPError) as e:
            m.switch_plan(shape, *args)
        assert e.value.name == name
    bad = m.make_shape(1, 16, 1024, 4, 1, "bf16")   # C*2 = 8 bytes: not a multiple of 16
    with pytest.raises(m.DSPError) as e:
        m.switch_plan(bad, 2, 0, "T", "S")
    assert e.value.name == "DSP_ERR_ALIGNMENT"
    p = m.lib()
    code = p.dsp_switch_plan(ctypes.byref(shape), 2, 0, 3, 1, ctypes.byref(m.SwitchPlan()))
    assert code == 5  # DSP_ERR_BAD_DIM


def test_workspace_bytes():
    m = dsp()
    sh = synth.CONFIGS["blk"]
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, sh.NH, sh.dtype)
    for N in (1, 2, 8):
        tok = sh.B * sh.T * sh.S // N
        assert m.workspace_bytes(shape, N) >= tok * 6 * sh.C * 2


def execute_plan(plan, x_local: np.ndarray, N: int, rank: int, y_local: np.ndarray, peers_out):
    """Host re-execution of a dsp_switch_plan_t as byte moves (used by the gloo test)."""
    xb = x_local.view(np.uint8).reshape(-1)
    for i0 in range(plan.n[0]):
        for i1 in range(plan.n[1]):
            for i2 in range(plan.n[2]):
                s = i0 * plan.src_stride[0] + i1 * plan.src_stride[1] + i2 * plan.src_stride[2]
                d = plan.dst_peer_off + i1 * plan.dst_stride[1] + i2 * plan.dst_stride[2]
                peers_out[i0].append((d, xb[s:s + plan.run_bytes].copy()))


@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("B", [1, 2])
def test_switch_plan_reproduces_oracle_switch(N, B):
    """Every rank's plan, executed as byte moves, yields the oracle switch bit-exactly."""
    m = dsp()
    sh = synth.BlockShape(B, 8, 16, 8, 1, "bf16")
    shape = m.make_shape(sh.B, sh.T, sh.S, sh.C, 1, "bf16")
    x = synth.make_index_tagged(sh, 4)
    for frm, to, src in ((osw.DIM_T, osw.DIM_S, osw.split(x, osw.DIM_T, N)),
                         (osw.DIM_S, osw.DIM_T, osw.split(x, osw.DIM_S, N))):
        want = osw.switch(src, frm, to)
        inbox = [[] for _ in range(N)]
        for r in range(N):
            plan = m.switch_plan(shape, N, r, frm, to)
            execute_plan(plan, src[r], N, r, None, inbox)
        for q in range(N):
            y = np.zeros(want[q].size * 2, dtype=np.uint8)
            for d, run in inbox[q]:
                y[d:d + run.size] = run
            assert np.array_equal(y.view(np.uint16).reshape(want[q].shape), want[q])
