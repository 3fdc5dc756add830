"""One head_gemv_kernel launch (K = 4 modalities, n requests) for an ncu
capture:  ncu --set full -k regex:head_gemv -c 1 python tools/head_one.py 1"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = 4
head = FusionHead(K, 1024, 499, FEAT_DIM)
feats = [torch.randn(1024, FEAT_DIM, device="cuda").to(torch.bfloat16) for _ in range(K)]
masks = np.arange(n) % ((1 << K) - 1) + 1
iv = torch.full((K, n), -1, dtype=torch.int32)
for k in range(K):
    sel = np.flatnonzero((masks >> k) & 1)
    iv[k, sel] = torch.arange(len(sel), dtype=torch.int32)
prog = head.program(n, feats, iv.cuda(), gemv=True)
for _ in range(3):
    prog.run()
torch.cuda.synchronize()
print("ok", head.logits[:n].float().abs().sum().item())
