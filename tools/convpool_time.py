"""conv2 + pool2: fused ms_gemm_plan_conv_pool vs the unfused halo conv +
max pool pair, graph-timed at served frame counts (rgb 183, flow 108).

    python tools/convpool_time.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_conv_weight  # noqa: E402

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


cin, cout = 64, 192
for H, n in ((56, 183), (56, 108), (56, 48), (64, 72)):
    X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
    w = torch.randn(cout, cin, 3, 3) * (2.0 / (9 * cin)) ** 0.5
    Wt = pack_conv_weight(w).to("cuda")
    b = torch.randn(cout, device="cuda") * 0.1
    D = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
    PH = (H - 3 + 1) // 2 + 1
    Y = torch.empty(n * PH * PH, cout, device="cuda", dtype=torch.bfloat16)
    Y2 = torch.empty_like(Y)
    if H == 64:  # audio's conv2: tap boxes (halo rows of 72 do not tile 128)
        from paper_2310_18481_b200.encoders import pick_conv_tile
        conv = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=cout,
                            tile=pick_conv_tile(n, H, H))
    else:
        conv = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=cout, halo=True)
    P = dv.Program()
    P.gemm(conv)
    P.pool(D, n, H, H, cout, cout, 3, 2, 0, True, True, Y2, cout, 0)
    P.seal()
    fused = dv.plan_conv_pool(X, n, H, H, cin, cin, Wt, cout, b, Y, ldy=cout)
    t_conv = timed(conv.run)
    t_pair = timed(P.run)
    t_fused = timed(fused.run)
    torch.cuda.synchronize()
    same = torch.equal(Y, Y2)
    fl = conv.flops
    print(f"{H}x{H} n={n:3d}: conv {t_conv:6.1f} us + pool = {t_pair:6.1f} us | fused {t_fused:6.1f} us "
          f"({fl / t_fused / 1e6:.0f} TF/s)  x{t_pair / t_fused:.2f}  grid {fused.info()['grid_x']} "
          f"stages {fused.info()['stages']}  {'bitwise equal' if same else 'MISMATCH'}", flush=True)
