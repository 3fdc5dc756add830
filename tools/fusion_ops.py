"""Per-op device time of the fusion head program (gather-concat FC1 [+ split-K
finalize] + head FC2), graph-timed, at several batch sizes (C5, K=4)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import FusionHead  # noqa: E402

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
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / inner)
    return float(np.median(ts))


K = 4
head = FusionHead(K, 1024, 499, 1024)
feats = [torch.randn(1024, 1024, device="cuda").to(torch.bfloat16) for _ in range(K)]
rng = np.random.default_rng(0)
for n in (1, 64, 256, 1024):
    masks = rng.integers(1, 16, size=n)
    inv = torch.full((K, n), -1, dtype=torch.int32)
    for k in range(K):
        sel = np.flatnonzero((masks >> k) & 1)
        inv[k, sel] = torch.arange(len(sel), dtype=torch.int32)
    inv = inv.cuda()
    prog = head.program(n, feats, inv)
    total = timed(prog.run)
    parts = []
    for kind, op in prog.ops:
        P = dv.Program()
        P.ops = [(kind, op)]
        P.keep = prog.keep
        P.seal()
        parts.append((op.label, getattr(op, "split_k", 1), op.info(), timed(P.run)))
    print(f"N={n:5d}: program {total:6.1f} us | " + " | ".join(
        f"{lb} split{sk} grid{inf['grid_x']} {us:.1f} us" for lb, sk, inf, us in parts), flush=True)
