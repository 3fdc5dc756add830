"""Microbenchmark of single GEMM plans (warm, CUDA-event timed): TF/s with
and without the epilogue stores, for representative encoder shapes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pick_conv_tile  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def t_plan(p, reps=10):
    for _ in range(3):
        p.run()
    e0.record()
    for _ in range(reps):
        p.run()
    e1.record()
    return e0.elapsed_us(e1) / reps


def conv(n, H, Cin, Cout, k, s, BN, tile=None):
    X = torch.randn(n, H, H, Cin, device="cuda").to(torch.bfloat16)
    cc = -(-Cin // 64) * 64
    W = (torch.randn(Cout, k * k * cc, device="cuda") * 0.02).to(torch.bfloat16)
    OH = (H + 2 * (k // 2) - k) // s + 1
    D = torch.empty(n * OH * OH, Cout, device="cuda", dtype=torch.bfloat16)
    tile = tile or pick_conv_tile(n, OH, OH)
    p = dv.plan_conv(X, n, H, H, Cin, Cin, k, k, s, k // 2, W, Cout, None, D, ldd=Cout, BN=BN, tile=tile)
    return p, f"conv {k}x{k}/{s} {Cin}->{Cout} n={n} {H}^2 BN={BN} tile={tile}"


def dense(M, K, N, BN):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    return dv.plan_dense(A, W, None, D, BN=BN, split_k=1), f"dense M={M} K={K} N={N} BN={BN}"


cases = [conv(288, 56, 64, 192, 3, 1, 192), conv(288, 56, 64, 192, 3, 1, 96),
         conv(288, 28, 96, 96, 3, 1, 96), conv(288, 28, 64, 96, 3, 1, 96),
         conv(288, 14, 160, 224, 3, 1, 224), conv(288, 7, 192, 320, 3, 1, 160),
         dense(903168, 64, 64, 64), dense(225792, 256, 256, 256), dense(73728, 576, 512, 256),
         dense(8192, 4096, 4096, 256)]
rows = []
for p, label in cases:
    us = t_plan(p)
    try:
        p.set_pair()
        us_pair = t_plan(p)
    except Exception as exc:  # plans the pair kernel does not support
        us_pair = float("nan")
        print("  pair n/a:", exc)
    print(f"{us:8.1f} us {p.flops / us / 1e6:7.1f} TF/s | pair {us_pair:8.1f} us {p.flops / us_pair / 1e6:7.1f} TF/s  {label}")
    continue
    dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 1), "debug")
    us_ns = t_plan(p)
    dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 0), "debug")
    inf = p.info()
    print(f"{us:8.1f} us {p.flops / us / 1e6:7.1f} TF/s | no-store {us_ns:8.1f} us {p.flops / us_ns / 1e6:7.1f} TF/s"
          f" | stages {inf['stages']} grid {inf['grid_x']}  {label}")
