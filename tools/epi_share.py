"""How much of a served-shape GEMM is its epilogue: each plan as the encoder
builds it (183 rgb frames), timed with and without the convert + store half of
the epilogue (ms_gemm_plan_debug flag 1: TMEM is still drained and released).

    python tools/epi_share.py [--n 183]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=183)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_conv_weight, pack_conv_weight_k32, pick_bn, pick_conv_tile  # noqa: E402

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


n = a.n
torch.manual_seed(0)
plans = []
for H, cin, cout in ((28, 64, 96), (28, 96, 96), (28, 64, 64), (14, 64, 96), (14, 96, 128), (14, 128, 160),
                     (14, 160, 160), (14, 192, 256), (7, 160, 224), (7, 192, 320)):
    X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
    w = torch.randn(cout, cin, 3, 3) * (2.0 / (9 * cin)) ** 0.5
    b = torch.randn(cout, device="cuda") * 0.1
    k32 = cin % 64 != 0 and cin % 32 == 0
    Wk = (pack_conv_weight_k32(w) if k32 else pack_conv_weight(w)).to("cuda")
    D = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
    p = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wk, cout, b, D, ldd=cout, BN=pick_bn(cout),
                     tile=pick_conv_tile(n, H, H), k32=k32)
    plans.append((p, f"conv 3x3 {H}^2 {cin}->{cout}{' k32' if k32 else ''}", [X, Wk, b, D]))
for M, K, N in ((n * 784, 192, 224), (n * 784, 256, 256), (n * 196, 576, 512), (n * 49, 1024, 832)):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda") * 0.1
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(N)
    p = dv.plan_dense(A, W, b, D, BN=BN, relu=True)
    plans.append((p, f"dense M={M} K={K} N={N}", [A, W, b, D]))
for p, label, _ in plans:
    us = t(p.run)
    dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 1), "debug")
    us_ns = t(p.run)
    dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 0), "debug")
    inf = p.info()
    print(f"{label:34s} {us:7.1f} us {p.flops / us / 1e6:6.0f} TF/s | no convert/store {us_ns:7.1f} us "
          f"{p.flops / us_ns / 1e6:6.0f} TF/s x{us / us_ns:4.2f} | grid {inf['grid_x']} st {inf['stages']}", flush=True)
