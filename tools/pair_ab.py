"""Single-SM vs CTA-pair (cta_group::2, half of B per SM) for the tap-box /
dense GEMMs of one served-mix encoder program: each op timed alone, R
launches back to back in a CUDA graph.

    python tools/pair_ab.py [--mod 0] [--n 61]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--mod", type=int, default=0)
ap.add_argument("--n", type=int, default=61)
ap.add_argument("--rep", type=int, default=10)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=96)
m.use_graphs = False
m.forward(np.arange(a.n), np.full(a.n, 7, dtype=np.int16))
torch.cuda.synchronize()
prog = m.encoders[a.mod].program(a.n)
e0, e1 = dv.Event(), dv.Event()


def timed(op):
    P = dv.Program()
    P.ops = [("gemm", op)] * a.rep
    P.keep = prog.keep
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
        ts.append(e0.elapsed_us(e1) / a.rep)
    return float(np.median(ts))


for i, (kind, op) in enumerate(prog.ops):
    if kind != "gemm" or getattr(op, "pair", False):
        continue
    lab = op.label
    if "stem" in lab or getattr(op, "split_k", 1) > 1:
        continue
    outs = [t for t in op.keep[3:4] if t is not None] + [sg[2] for sg in (op.keep[4] or [])]
    t1 = timed(op)
    ref = [o.clone() for o in outs]
    try:
        op.set_pair(True)
    except Exception as e:  # noqa: BLE001
        print(f"op {i:2d} {lab:44s} single {t1:6.1f} us  pair n/a ({e})")
        continue
    for o in outs:
        o.zero_()
    t2 = timed(op)
    same = all(torch.equal(o, r) for o, r in zip(outs, ref))
    print(f"op {i:2d} {lab:44s} single {t1:6.1f} us  pair {t2:6.1f} us  {t1 / t2:4.2f}x  "
          f"({op.flops / t1 / 1e6:4.0f} -> {op.flops / t2 / 1e6:4.0f} TF/s)  grid {op.info()['grid_x']} "
          f"stages {op.info()['stages']} {'bitwise equal' if same else 'MISMATCH'}")
