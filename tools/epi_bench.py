"""Epilogue cost microbenchmark: one 128-row tile per CTA (M = 148*128),
K = 64 (one K block), N = 32..256; the per-launch time growth with N is the
epilogue's per-chunk cost.  Each plan runs 20x inside one CUDA graph."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def graph_time(run, reps=20):
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                run()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    ts = []
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / reps)
    return float(np.median(ts))


for K in (64, 576):
    for N in (32, 64, 128, 192, 256):
        M = 148 * 128
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
        b = torch.zeros(N, device="cuda")
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res = []
        for relu in (False, True):
            p = dv.plan_dense(A, W, b, D, BN=N, relu=relu, split_k=1, pair=False)
            res.append(graph_time(p.run))
        D2 = torch.empty(M, N, device="cuda", dtype=torch.float32)
        p2 = dv.plan_dense(A, W, b, D2, BN=N, out_fp32=True, split_k=1, pair=False)
        f32 = graph_time(p2.run)
        print(f"K={K:4d} N={N:3d}: bf16 TMA-store {res[0]:6.2f} us, +relu {res[1]:6.2f} us, fp32 direct {f32:6.2f} us",
              flush=True)
