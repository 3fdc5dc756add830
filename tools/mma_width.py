"""Tensor throughput of the GEMM kernel vs output tile width (deep K, no
epilogue stores): isolates per-UMMA cost at small N."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

e0, e1 = dv.Event(), dv.Event()
for N, BN in [(64, 64), (96, 96), (128, 128), (192, 192), (256, 256), (512, 256)]:
    M, K = 65536, 4096
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    p = dv.plan_dense(A, W, None, D, BN=BN, split_k=1, pair=False)

    for _ in range(3):
        p.run()
    e0.record()
    for _ in range(10):
        p.run()
    e1.record()
    us = e0.elapsed_us(e1) / 10
    tiles = (M // 128) * (N // BN)
    print(f"N={N:4d} BN={BN:3d}: {us:8.1f} us {p.flops / us / 1e6:7.1f} TF/s  per-UMMA "
          f"{us * 1e-6 * 1.9e9 * 148 / (tiles * K / 16):6.1f} clk  stages {p.info()['stages']}")
