"""3x3 conv with 96/160/224 input channels: per-tap 64-channel chunks (padded)
vs K32 halves (K = 9*C exactly), graph-timed."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_conv_weight, pack_conv_weight_k32, pick_bn, pick_conv_tile  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def timed(fn, inner=10):
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


for n, H, cin, cout, st in [(192, 28, 96, 96, 1), (192, 28, 96, 96, 2), (192, 14, 96, 128, 1), (192, 14, 160, 192, 1),
                            (192, 14, 160, 160, 1), (192, 7, 224, 224, 1), (96, 28, 96, 96, 1), (48, 14, 160, 192, 1)]:
    X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(cout, cin, 3, 3) * 0.02).to(torch.bfloat16)
    W0, W1 = pack_conv_weight(w).cuda(), pack_conv_weight_k32(w).cuda()
    b = torch.zeros(cout, device="cuda")
    OH = (H + 2 - 3) // st + 1
    D = torch.empty(n * OH * OH, cout, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(cout)
    tile = pick_conv_tile(n, OH, OH)
    p0 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, st, 1, W0, cout, b, D, ldd=cout, BN=BN, tile=tile)
    p1 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, st, 1, W1, cout, b, D, ldd=cout, BN=BN, tile=tile, k32=True)
    t0, t1 = timed(p0.run), timed(p1.run)
    print(f"n={n:3d} {H}x{H}/{st} {cin:3d}->{cout:3d}: chunks64{' pair' if getattr(p0, 'pair', False) else '     '} "
          f"{t0:7.1f} us {p0.flops / t0 / 1e6:6.0f} TF/s | k32 {t1:7.1f} us {p1.flops / t1 / 1e6:6.0f} TF/s  x{t0 / t1:.2f}",
          flush=True)
