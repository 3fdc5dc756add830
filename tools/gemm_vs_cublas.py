"""Our dense tcgen05 GEMM vs cuBLAS (torch.matmul) on L2-friendly shapes:
per-UMMA cycle cost and TF/s, with and without the epilogue."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

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


for M, N, K in [(16384, 256, 2048), (16384, 96, 2048), (32768, 192, 1024), (8192, 512, 4096), (8192, 8192, 8192)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    tc = timed(lambda: torch.matmul(A, W.t(), out=D))
    res = [f"M={M} N={N} K={K}: cuBLAS {fl / tc / 1e6:6.0f} TF/s"]
    for pair in (False, True):
        for BN in sorted({min(256, N), 128} if N >= 128 else {N}):
            try:
                p = dv.plan_dense(A, W, None, D, BN=BN, split_k=1, pair=pair)
            except Exception as exc:  # noqa: BLE001
                continue
            t = timed(p.run)
            dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 1), "dbg")
            tn = timed(p.run)
            res.append(f"ours{' pair' if pair else ''} BN={BN} {fl / t / 1e6:6.0f} TF/s (no-epi {fl / tn / 1e6:6.0f})")
    print(" | ".join(res), flush=True)
