"""Warm per-op device times of one masked TBN pass: every op of every
encoder program (and the head) run alone between CUDA events, in program
order, after a full warm-up pass.  Each op is timed as REP back-to-back
launches inside one CUDA graph (no host launch latency; PDL overlap between
consecutive launches as in a pass graph).  Prints ops sorted by time with achieved
TFLOP/s for GEMMs.

    python tools/op_times.py --n 96 [--mixed]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=96)
ap.add_argument("--mixed", action="store_true")
ap.add_argument("--mask", type=int, default=7)
ap.add_argument("--top", type=int, default=45)
ap.add_argument("--rep", type=int, default=10)
ap.add_argument("--counts", type=int, nargs=3, default=None, help="per-modality request counts (served mix)")
a = ap.parse_args()
REP = a.rep

import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=a.n, n_slots=max(8, a.n))
rng = np.random.default_rng(0)
masks = rng.integers(1, 8, size=a.n).astype(np.int16) if a.mixed else np.full(a.n, a.mask, dtype=np.int16)
if a.counts:
    masks = np.zeros(a.n, dtype=np.int16)
    for k, c in enumerate(a.counts):
        masks[rng.permutation(a.n)[:c]] |= 1 << k
    masks[masks == 0] = 1
slots = np.arange(a.n) % m.n_slots
m.use_graphs = False
for _ in range(2):
    m.forward(slots, masks)
torch.cuda.synchronize()
counts = m.counts_for(masks)
e0, e1 = dv.Event(), dv.Event()
rows = []
for k, (enc, c) in enumerate(zip(m.encoders, counts)):
    if not c:
        continue
    prog = enc.program(c)
    for i, (kind, op) in enumerate(prog.ops):
        # the op repeated REP times inside one CUDA graph: device time per
        # launch without host launch latency (as inside a pass graph)
        single = dv.Program()
        single.ops = [(kind, op)] * REP
        single.keep = prog.keep
        single.seal()
        single.run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                single.run()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        ts = []
        for _ in range(5):
            e0.record()
            g.replay()
            e1.record()
            ts.append(e0.elapsed_us(e1) / REP)
        us = float(np.median(ts))
        fl = op.flops if kind == "gemm" else 0
        if kind == "gemm":
            lab = op.label
        elif kind == "pool":
            lab = f"{'max' if op[10] else 'avg'} {op[6]}x{op[6]}/{op[7]} C={op[4]} {op[1]}x{op[2]}x{op[3]}"
        else:
            lab = ""
        if kind == "gemm":
            info = op.info()
            lab += f" [grid {info['grid_x']}x{info['grid_y']} st{info['stages']} smem{info['smem_bytes'] // 1024}K" \
                   f"{' pair' if getattr(op, 'pair', False) else ''}{' sk' + str(op.split_k) if op.split_k > 1 else ''}]"
        rows.append((us, k, i, kind, lab, fl))
tot = sum(r[0] for r in rows)
gem = [r for r in rows if r[3] == "gemm"]
gt = sum(r[0] for r in gem)
print(f"encoders: {tot:.0f} us ({len(rows)} ops); GEMM {gt:.0f} us = {sum(r[5] for r in gem) / gt / 1e6:.0f} TFLOP/s; "
      f"other {tot - gt:.0f} us")
by_kind = {}
for r in rows:
    by_kind[r[3]] = by_kind.get(r[3], 0.0) + r[0]
print("by kind:", {k: round(v) for k, v in sorted(by_kind.items(), key=lambda x: -x[1])})
for r in sorted(rows, key=lambda r: -r[0])[: a.top]:
    tf = f"{r[5] / r[0] / 1e6:7.1f} TF/s" if r[5] else " " * 12
    print(f"{r[0]:8.1f} us {tf} mod{r[1]} #{r[2]:<3d} {r[3]:8s} {r[4]}")
