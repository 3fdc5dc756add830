"""3x3/1/1 conv variants on the served-mix shapes (183 rgb frames): the
encoder's current choice (tap-box / K32) vs halo (single CTA) vs halo on
CTA pairs (cta_group::2, half of the weights per SM, resident when they fit),
graph-timed, plus bitwise agreement of every variant with the current one.

    python tools/conv_variants.py [--n 183]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=183)
ap.add_argument("--inner", type=int, default=10)
ap.add_argument("--only", default="")
ap.add_argument("--tap-pair", action="store_true", help="tap-box / K32 plan vs the same plan on CTA pairs")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import (pack_conv_weight, pack_conv_weight_k32, pick_bn,  # noqa: E402
                                            pick_conv_tile)

e0, e1 = dv.Event(), dv.Event()


def timed(fn, inner=a.inner):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(inner):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    ts = []
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / inner)
    return float(np.median(ts))


SHAPES = [(56, 64, 192), (28, 64, 64), (28, 64, 96), (28, 96, 96), (14, 64, 96), (14, 96, 128), (14, 128, 128),
          (14, 128, 160), (14, 160, 160), (14, 128, 192), (14, 160, 192), (14, 192, 192), (14, 192, 256)]
n = a.n
torch.manual_seed(0)
for H, cin, cout in SHAPES:
    if a.only and f"{H}:{cin}:{cout}" not in a.only.split(","):
        continue
    X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
    w = torch.randn(cout, cin, 3, 3) * (2.0 / (9 * cin)) ** 0.5
    b = torch.randn(cout, device="cuda") * 0.1
    k32 = cin % 64 != 0 and cin % 32 == 0
    Wk = (pack_conv_weight_k32(w) if k32 else pack_conv_weight(w)).to("cuda")
    W64 = pack_conv_weight(w).to("cuda")
    D0 = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(cout)
    tile = pick_conv_tile(n, H, H)
    p0 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wk, cout, b, D0, ldd=cout, BN=BN, tile=tile, k32=k32)
    t0 = timed(p0.run)
    p0.run()
    torch.cuda.synchronize()
    ref = D0.clone()
    fl = p0.flops
    line = f"{H:2d}x{H} {cin:3d}->{cout:3d} {'k32' if k32 else 'tap'} {t0:6.1f} us {fl / t0 / 1e6:5.0f} TF/s"
    if a.tap_pair:  # the same tap-box / K32 plan on CTA pairs (M = 256 tiles, half of each weight box per SM)
        D1 = torch.empty_like(D0)
        try:
            p1 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wk, cout, b, D1, ldd=cout, BN=BN, tile=tile, k32=k32)
            p1.set_pair(True)
            t1 = timed(p1.run)
            p1.run()
            torch.cuda.synchronize()
            err = (D1.float() - ref.float()).abs().max().item()
            inf = p1.info()
            line += (f" | tap-pair {t1:6.1f} us {fl / t1 / 1e6:5.0f} TF/s x{t0 / t1:4.2f} st{inf['stages']} "
                     f"g{inf['grid_x']} maxdiff {err:.3g}")
        except Exception as ex:  # noqa: BLE001
            line += f" | tap-pair n/a ({str(ex)[:60]})"
        print(line, flush=True)
        continue
    cc = -(-cin // 64)
    bns = -(-cout // 32) * 32
    while bns > 32 and 9 * cc * (bns // 2) * 128 > 150 * 1024:  # half of the weights resident per CTA
        bns -= 32
    for name, pair, bn_ in (("halo", False, BN), ("halo-pair", True, BN), (f"halo-pair BN{bns}", True, bns)):
        if name.startswith("halo-pair BN") and bns == BN:
            continue
        D1 = torch.empty_like(D0)
        try:
            p1 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, W64, cout, b, D1, ldd=cout, BN=bn_, halo=True)
            if pair:
                p1.set_pair(True)
        except Exception as ex:  # noqa: BLE001
            line += f" | {name} n/a ({str(ex)[:50]})"
            continue
        t1 = timed(p1.run)
        p1.run()
        torch.cuda.synchronize()
        err = (D1.float() - ref.float()).abs().max().item()
        inf = p1.info()
        line += (f" | {name} {t1:6.1f} us {fl / t1 / 1e6:5.0f} TF/s x{t0 / t1:4.2f} st{inf['stages']} "
                 f"g{inf['grid_x']} maxdiff {err:.3g}")
    print(line, flush=True)
