"""Reference point only (not on the product path): cuBLAS bf16 via
torch.matmul on the same narrow GEMM shapes as the encoder convs."""
import torch

e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for M, K, N in [(225792, 864, 96), (225792, 576, 96), (903168, 576, 192), (225792, 256, 256), (8192, 4096, 4096),
                (65536, 4096, 64), (65536, 4096, 256)]:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        C = A @ B
    e0.record()
    for _ in range(10):
        C = A @ B
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / 10
    print(f"cuBLAS M={M} K={K} N={N}: {us:8.1f} us {2 * M * N * K / us / 1e6:7.1f} TF/s")
