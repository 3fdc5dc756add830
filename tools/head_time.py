"""Late-fusion head: the one-launch cluster kernel vs the three-launch path
(gather GEMM, FC2 split-K GEMM, finalize) vs the two-launch GEMV head,
graph-timed per request count.

    python tools/head_time.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import FEAT_DIM, FusionHead  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def timed(fn, inner=20):
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
    for _ in range(7):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / inner)
    return float(np.median(ts))


for K in (3, 4):
    head = FusionHead(K, 1024, 499, FEAT_DIM)
    feats = [torch.randn(1024, FEAT_DIM, device="cuda").to(torch.bfloat16) for _ in range(K)]
    for n in (1, 4, 8, 16, 24, 32, 48, 64, 1024):
        masks = np.arange(n) % ((1 << K) - 1) + 1
        iv = torch.full((K, n), -1, dtype=torch.int32)
        for k in range(K):
            sel = np.flatnonzero((masks >> k) & 1)
            iv[k, sel] = torch.arange(len(sel), dtype=torch.int32)
        iv = iv.cuda()
        pu = head.program(n, feats, iv, fused=False, gemv=False)
        pf = head.program(n, feats, iv, fused=True, gemv=False)
        pg = head.program(n, feats, iv, gemv=True)
        tu, tf, tg = timed(pu.run), timed(pf.run), timed(pg.run)
        wb = head.w1.numel() * 2 + head.w2.numel() * 2
        print(f"K={K} n={n:5d}  unfused {tu:6.2f} us ({pu.n_launches} launches)  fused {tf:6.2f} us  "
              f"gemv {tg:6.2f} us ({wb / tg / 1e3:5.0f} GB/s of weights)  best {min((tu, 'unfused'), (tf, 'fused'), (tg, 'gemv'))[1]}",
              flush=True)
