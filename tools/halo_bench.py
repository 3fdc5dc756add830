"""3x3/1/1 conv: tap-box implicit GEMM (with auto 2-SM pairs) vs halo reuse,
graph-timed, at serving-like frame counts."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pick_bn, pick_conv_tile  # noqa: E402

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


for n, H, cin, cout in [(192, 28, 96, 96), (192, 28, 64, 96), (192, 28, 64, 64), (192, 14, 160, 224),
                        (192, 14, 192, 192), (192, 56, 64, 192), (96, 28, 96, 96), (48, 28, 96, 96),
                        (48, 14, 160, 224), (288, 56, 64, 192)]:
    X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
    cc = -(-cin // 64) * 64
    W = (torch.randn(cout, 9 * cc, device="cuda") * 0.02).to(torch.bfloat16)
    b = torch.zeros(cout, device="cuda")
    D = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(cout)
    p0 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, W, cout, b, D, ldd=cout, BN=BN,
                      tile=pick_conv_tile(n, H, H))
    # halo: the widest N tile whose 9 x cchunks weight blocks fit in smem (resident)
    BNh = BN
    while BNh > 32 and 9 * (cc // 64) * BNh * 128 > 150 * 1024:
        BNh -= 32
    p1 = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, W, cout, b, D, ldd=cout, BN=BNh, halo=True)
    t0, t1 = timed(p0.run), timed(p1.run)
    dv.check(dv.lib().ms_gemm_plan_debug(p0.addr, 1), "dbg")
    dv.check(dv.lib().ms_gemm_plan_debug(p1.addr, 1), "dbg")
    t0n, t1n = timed(p0.run), timed(p1.run)
    fl = p0.flops
    print(f"n={n:3d} {H}x{H} {cin:3d}->{cout:3d}: tap-box{' pair' if getattr(p0, 'pair', False) else '     '} "
          f"{t0:7.1f} us {fl / t0 / 1e6:6.0f} TF/s | halo BN={BNh} {t1:7.1f} us {fl / t1 / 1e6:6.0f} TF/s  x{t0 / t1:.2f}"
          f" | no-epilogue: tap-box {t0n:6.1f} us halo {t1n:6.1f} us",
          flush=True)
