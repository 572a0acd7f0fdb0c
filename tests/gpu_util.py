"""Helpers for the -m gpu tests: synth arrays <-> torch tensors, tolerance checks."""
import numpy as np
import torch

import synth


def to_dev(stored: np.ndarray, dtype: str, device="cuda") -> torch.Tensor:
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(stored).view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(stored, dtype=np.float32)).to(device)


def to_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().double().cpu().numpy()


def weights_dev(W: dict, dtype: str) -> dict:
    return {k: to_dev(v, dtype) for k, v in W.items()}


def weights_f64(W: dict, dtype: str) -> dict:
    return {k: synth.to_f64(v, dtype) for k, v in W.items()}


BF16_U = 2.0 ** -8  # unit roundoff of bf16 (8-bit significand)


def assert_block_close(got: np.ndarray, ref: np.ndarray, atol=2e-2, rtol=1e-2, rel_l2=1e-2, stored=None):
    """DESIGN.md tolerance R22 (north_star 'max-abs 2e-2 / rel 1e-2', read as allclose) + rel-L2.
    stored (R34): list of the residual-stream values (oracle, same shape) the block stores in bf16 on
    the way to `ref` (y1, y2, ..., y); an element is also within tolerance if its error is within
    atol + the storage bound sum_k u*|z_k|, u = 2^-8 -- what bf16 storage alone may cost at large
    magnitudes (|z| ~ 17 in deep layers: 1.5 % for four stores, more than rtol's 1 %)."""
    err = np.abs(got - ref)
    allowed = atol + rtol * np.abs(ref)
    if stored is not None:
        allowed = np.maximum(allowed, atol + BF16_U * sum(np.abs(z) for z in stored))
    bad = err > allowed
    l2 = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    msg = (f"max-abs {err.max():.3e}, max-rel {(err / np.maximum(np.abs(ref), 1e-6)).max():.3e}, "
           f"rel-L2 {l2:.3e}, violations {int(bad.sum())}/{bad.size}")
    assert not bad.any() and l2 <= rel_l2, msg
    return msg


def bits16(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy()
