"""Per-CTA %globaltimer timeline of one 3x3/1/1 conv plan variant (tap / halo /
halo-pair), launched right after itself in a CUDA graph (PDL chain).

    python tools/conv_trace.py --h 14 --cin 128 --cout 128
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=183)
ap.add_argument("--h", type=int, default=14)
ap.add_argument("--cin", type=int, default=128)
ap.add_argument("--cout", type=int, default=128)
ap.add_argument("--variants", default="tap,halo,halo-pair")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_conv_weight, pack_conv_weight_k32, pick_bn, pick_conv_tile  # noqa

NAMES = ["entry", "prolog", "pdlwait", "load0", "data0", "lastmma", "acc0", "epi_end", "ldtm0", "cvt0", "store0",
         "tile0end"]
n, H, cin, cout = a.n, a.h, a.cin, a.cout
X = torch.randn(n, H, H, cin, device="cuda").to(torch.bfloat16)
w = torch.randn(cout, cin, 3, 3) * (2.0 / (9 * cin)) ** 0.5
b = torch.zeros(cout, device="cuda")
for v in a.variants.split(","):
    k32 = cin % 64 != 0 and cin % 32 == 0 and v == "tap"
    Wt = (pack_conv_weight_k32(w) if k32 else pack_conv_weight(w)).to("cuda")
    D = torch.empty(n * H * H, cout, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(cout)
    if v.startswith("halo"):
        p = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=BN, halo=True)
        if v == "halo-pair":
            p.set_pair(True)
    else:
        p = dv.plan_conv(X, n, H, H, cin, cin, 3, 3, 1, 1, Wt, cout, b, D, ldd=cout, BN=BN,
                         tile=pick_conv_tile(n, H, H), k32=k32)
    info = p.info()
    NS = len(NAMES)
    buf = torch.zeros(info["grid_x"] * NS, dtype=torch.int64, device="cuda")
    dv.check(dv.lib().ms_gemm_plan_set_trace(p.addr, buf.data_ptr()), "set_trace")
    for _ in range(3):
        p.run()
    torch.cuda.synchronize()
    t = buf.view(-1, NS).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    print(f"{v}: {p.label} grid {info['grid_x']} stages {info['stages']} smem {info['smem_bytes']} "
          f"span {np.nanmax(rel[:, 7]):.1f} us")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        if np.all(np.isnan(col)):
            continue
        print(f"   {nm:8s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f}")
