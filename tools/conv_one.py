"""One 3x3/1/1 conv launch (for ncu): --variant tap|halo|halo-pair|tap-pair.
Launches the plan twice (ncu: --launch-skip 1 --launch-count 1).

    ncu --set full -k regex:gemm_tc --launch-skip 1 --launch-count 1 \
        python tools/conv_one.py --h 14 --cin 128 --cout 128 --variant halo
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=183)
ap.add_argument("--h", type=int, default=14)
ap.add_argument("--cin", type=int, default=128)
ap.add_argument("--cout", type=int, default=128)
ap.add_argument("--variant", default="tap")
ap.add_argument("--bn", type=int, default=0)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_conv_weight, pack_conv_weight_k32, pick_bn, pick_conv_tile  # noqa

n, H, cin, cout = a.n, a.h, a.cin, a.cout
X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
w = torch.randn(cout, cin, 3, 3) * (2.0 / (9 * cin)) ** 0.5
b = torch.zeros(cout, device="cuda")
k32 = cin % 64 != 0 and cin % 32 == 0 and a.variant.startswith("tap")
Wt = (pack_conv_weight_k32(w) if k32 else pack_conv_weight(w)).to("cuda")
D = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
BN = a.bn or pick_bn(cout)
if a.variant.startswith("halo"):
    p = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=BN, halo=True)
else:
    p = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=BN,
                     tile=pick_conv_tile(n, H, H), k32=k32, pair=a.variant.endswith("pair") or None)
if a.variant == "halo-pair":
    p.set_pair(True)
print(p.label, p.info(), flush=True)
for _ in range(2):
    p.run()
torch.cuda.synchronize()
