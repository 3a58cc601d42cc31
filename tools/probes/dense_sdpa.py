"""Probe: dense SDPA time at the HunyuanVideo 720p shape (the >=5x comparator)."""
import time
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

torch.manual_seed(0)
H, N, D = 24, 118800, 128
q = torch.randn(1, H, N, D, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q)
v = torch.randn_like(q)
flops = 4.0 * N * N * D * H
for name, be in [("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)]:
    try:
        with sdpa_kernel([be]):
            for _ in range(2):
                F.scaled_dot_product_attention(q, k, v)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            n = 3
            for _ in range(n):
                F.scaled_dot_product_attention(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            print(f"{name}: {ms:.2f} ms  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
    except Exception as ex:  # noqa: BLE001
        print(f"{name}: unavailable ({type(ex).__name__}: {str(ex)[:120]})", flush=True)
