"""Library context for the roofline: cuBLAS (torch.matmul) at the block's GEMM shapes and
torch SDPA backends at the spatial / temporal attention shapes (blk, N=1).  Not a bench."""
import torch
import torch.nn.functional as F

def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3

tok, C = 16384, 1152
for name, (M, N, K) in {"qkv": (tok, 3 * C, C), "proj": (tok, C, C), "fc1": (tok, 4 * C, C), "fc2": (tok, C, 4 * C),
                        "8192^3": (8192, 8192, 8192)}.items():
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    us = t(lambda: A @ W.t())
    print(f"cuBLAS {name:7s} {us:8.1f} us  {2*M*N*K/us/1e6:7.1f} TFLOP/s")
from torch.nn.attention import sdpa_kernel, SDPBackend
for label, (B, H, L, D) in {"spatial": (16, 16, 1024, 72), "temporal": (1024, 16, 16, 72)}.items():
    q, k, v = (torch.randn(B, H, L, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    fl = 4 * B * H * L * L * D
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel([be]):
                us = t(lambda: F.scaled_dot_product_attention(q, k, v))
            print(f"SDPA {label:8s} {be.name:20s} {us:8.1f} us  {fl/us/1e6:7.1f} TFLOP/s")
        except Exception as e:
            print(f"SDPA {label:8s} {be.name:20s} unavailable: {str(e)[:80]}")
try:
    import flashinfer
    q = torch.randn(16 * 1024, 16, 72, device="cuda", dtype=torch.bfloat16)
    print("flashinfer", flashinfer.__version__)
except Exception as e:
    print("flashinfer unavailable", str(e)[:80])
