"""%globaltimer stamps inside the fused head kernel (per CTA, relative to the
earliest start): 0 start, 1 first K block ready, 2 FC1 done, 3 cluster
barrier, 4 FC1 reduce-scatter done, 5 FC2 done, 6 FC2 reduce-scatter done,
6 (unused), 7 logits stored.

    python tools/head_trace.py [--n 1] [--k 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--k", type=int, default=3)
a = ap.parse_args()
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead  # noqa: E402

K, n = a.k, a.n
head = FusionHead(K, 1024, 499, FEAT_DIM)
feats = [torch.randn(1024, FEAT_DIM, device="cuda").to(torch.bfloat16) for _ in range(K)]
iv = torch.arange(n, dtype=torch.int32).repeat(K, 1).cuda()
p = dv.plan_fused_head(feats, iv, head.w1, head.b1, head.w2, head.b2, head.logits, M=n, feat_dim=FEAT_DIM)
ctas = 8 * -(-n // 128)
buf = torch.zeros(ctas * 12, dtype=torch.int64, device="cuda")
dv.check(dv.lib().ms_gemm_plan_set_trace(p.addr, buf.data_ptr()), "trace")
for it in range(3):
    p.run()
    torch.cuda.synchronize()
t = buf.view(ctas, 12)[:, :8].cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
print("cta  " + " ".join(f"{s:>7d}" for s in range(8)))
for c in range(ctas):
    print(f"{c:3d}  " + " ".join(f"{(v - t0) / 1e3:7.2f}" for v in t[c]))
