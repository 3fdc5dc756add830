"""Conv tile-shape sweep: TMA box geometry (bn, bh, bw) vs throughput."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def run(n, H, Cin, Cout, s, BN, tile, pair=False):
    X = torch.randn(n, H, H, Cin, device="cuda").to(torch.bfloat16)
    cc = -(-Cin // 64) * 64
    W = (torch.randn(Cout, 9 * cc, device="cuda") * 0.02).to(torch.bfloat16)
    OH = (H + 2 - 3) // s + 1
    D = torch.empty(n * OH * OH, Cout, device="cuda", dtype=torch.bfloat16)
    p = dv.plan_conv(X, n, H, H, Cin, Cin, 3, 3, s, 1, W, Cout, None, D, ldd=Cout, BN=BN, tile=tile)
    if pair:
        p.set_pair()
    for _ in range(3):
        p.run()
    e0.record()
    for _ in range(10):
        p.run()
    e1.record()
    us = e0.elapsed_us(e1) / 10
    return us, p.flops / us / 1e6


for (Cin, Cout, H, s) in [(96, 96, 28, 1), (64, 96, 28, 1), (64, 192, 56, 1), (160, 224, 14, 1), (96, 96, 28, 2)]:
    OH = (H + 2 - 3) // s + 1
    for tile in [(8, 4, 4), (1, 4, 28), (1, 8, 14), (2, 2, 28), (4, 2, 14), (1, 8, 16), (2, 8, 8), (32, 2, 2),
                 (2, 7, 7), (1, 9, 14), (1, 7, 14), (4, 4, 7)]:
        bn, bh, bw = tile
        if bn * bh * bw > 128 or bh > OH or bw > OH:
            continue
        us, tf = run(288, H, Cin, Cout, s, Cout if Cout <= 256 else 160, tile)
        print(f"conv {Cin}->{Cout} {H}^2/s{s} tile {tile}: {us:7.1f} us {tf:7.1f} TF/s")
