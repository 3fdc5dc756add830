"""The ViT/BERT dense GEMM shapes of a served VQA pass (M = tokens of ~96
requests): our tcgen05 plan (BN 256, single CTA / CTA pair, with and without
the GELU epilogue) vs cuBLAS (torch.matmul), warm, CUDA-event timed.

    python tools/vqa_gemm.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_us(e1) / reps


for M, N, K, act in ((18912, 3072, 768, 2), (18912, 768, 3072, 0), (18912, 2304, 768, 0), (18912, 768, 768, 0)):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, device="cuda")
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    tc = t(lambda: torch.matmul(A, W.t()))
    line = f"M={M} N={N} K={K} act={act}: cuBLAS {fl / tc / 1e6:6.0f} TF/s"
    for BN in (128, 256):
        for pair in (False, True):
            for a_ in sorted({0, act}):
                try:
                    p = dv.plan_dense(A, W, b, D, BN=BN, act=a_, pair=pair)
                    us = t(p.run)
                    inf = p.info()
                    line += f" | BN{BN}{' pair' if pair else ''} act{a_} {fl / us / 1e6:6.0f} (g{inf['grid_x']} st{inf['stages']})"
                except Exception as ex:  # noqa: BLE001
                    line += f" | BN{BN} pair={pair} n/a {str(ex)[:40]}"
    print(line, flush=True)
