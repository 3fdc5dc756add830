"""tcgen05 attention alone: ViT-B/16 (L=197) and BERT (L=40) shapes, 12
heads, n sequences; CUDA-graph timed, FLOP = 4*n*H*L*L*64.

    python tools/attn_time.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

e0, e1 = dv.Event(), dv.Event()
H = 12
for L, n in ((197, 32), (197, 96), (40, 32), (40, 256)):
    qkv = torch.randn(n * L, 3 * H * 64, device="cuda").to(torch.bfloat16)
    out = torch.empty(n * L, H * 64, device="cuda", dtype=torch.bfloat16)
    P = dv.Program()
    for _ in range(10):
        P.attention(qkv, 3 * H * 64, L, H, n, out, H * 64, 0.125)
    P.seal()
    P.run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            P.run(s)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    ts = []
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / 10)
    t = float(np.median(ts))
    fl = 4 * n * H * L * L * 64
    byts = n * L * 3 * H * 64 * 2 + n * L * H * 64 * 2
    print(f"L={L:3d} n={n:3d}: {t:7.1f} us  {fl / t / 1e6:6.0f} TFLOP/s  {byts / t / 1e3:6.0f} GB/s")
