"""Per-template efficiency of one served-mix TBN pass (the bench's operating
point: ~61 requests, all rgb, ~36 flow, ~24 audio; or --counts).  Every op
of every present encoder program is timed alone (REP back-to-back launches in
one CUDA graph, CUDA events), FLOP from the plan; ops are grouped by kernel
template (conv mode / dense / stem / pools) and reported as share of encoder
time, TFLOP/s and fraction of the measured bf16 peaks.

    python tools/pass_templates.py [--counts 61 36 24] > profiles/r02_pass_templates.md
"""
import argparse
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
ap = argparse.ArgumentParser()
ap.add_argument("--counts", type=int, nargs=3, default=(61, 36, 24))
ap.add_argument("--rep", type=int, default=10)
ap.add_argument("--ops", action="store_true", help="also print one row per op")
a = ap.parse_args()

import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
burst, sust = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
n = max(a.counts)
m = build_tbn_model(max_req=96, n_slots=192)
rng = np.random.default_rng(0)
masks = np.zeros(n, dtype=np.int16)
for k, c in enumerate(a.counts):
    masks[rng.permutation(n)[:c]] |= 1 << k
masks[masks == 0] = 1
counts = m.counts_for(masks)
m.use_graphs = False
for _ in range(2):
    m.forward(np.arange(n) % m.n_slots, masks)
torch.cuda.synchronize()
e0, e1 = dv.Event(), dv.Event()


def template(kind, op):
    if kind == "gemm":
        lab = op.label
        if lab.startswith("stem"):
            return "stem (conv1+pool1 fused)"
        if lab.startswith("dense"):
            return "dense 1x1 / FC"
        if lab.startswith("gather"):
            return "fusion gather GEMM"
        if "halo" in lab:
            return "3x3 halo"
        if "k32" in lab:
            return "3x3 K32"
        mm = re.match(r"conv (\d)x\d/(\d)", lab)
        pair = " (2-SM pair)" if getattr(op, "pair", False) else ""
        return f"conv {mm.group(1)}x{mm.group(1)}/{mm.group(2)} tap-box{pair}" if mm else lab
    if kind == "pool":
        return "max pool" if op[10] else "avg pool"
    return kind


rows = []
oprows = []
for k, (enc, c) in enumerate(zip(m.encoders, counts)):
    if not c:
        continue
    prog = enc.program(c)
    for i, (kind, op) in enumerate(prog.ops):
        single = dv.Program()
        single.ops = [(kind, op)] * a.rep
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
            ts.append(e0.elapsed_us(e1) / a.rep)
        rows.append((template(kind, op), float(np.median(ts)), op.flops if kind == "gemm" else 0))
        if a.ops:
            lab = op.label if kind == "gemm" else f"{kind} {op[1:6]}"
            inf = op.info() if kind == "gemm" else {}
            oprows.append((k, i, lab, rows[-1][1], rows[-1][2], inf))
tot = sum(r[1] for r in rows)
fl = sum(r[2] for r in rows)
agg = {}
for t, us, f in rows:
    x = agg.setdefault(t, [0, 0.0, 0])
    x[0] += 1
    x[1] += us
    x[2] += f
print(f"# Per-template efficiency, served-mix TBN pass (counts rgb/flow/audio = {tuple(counts)})\n")
print(f"Ops timed alone (median of 5 x {a.rep} back-to-back launches in a CUDA graph); FLOP from the plans "
      f"(real channels). Encoder time {tot:.0f} us for {fl / 1e9:.1f} GFLOP = {fl / tot / 1e6:.0f} TFLOP/s = "
      f"{fl / tot / 1e6 / burst:.3f} of burst {burst} / {fl / tot / 1e6 / sust:.3f} of sustained {sust} TF/s.\n")
print("| template | ops | time us | share | TFLOP/s | frac burst | frac sustained |")
print("|---|---|---|---|---|---|---|")
for t, (nop, us, f) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    tf = f / us / 1e6 if f else 0.0
    print(f"| {t} | {nop} | {us:.0f} | {us / tot:.3f} | {tf:.0f} | {tf / burst:.3f} | {tf / sust:.3f} |")
if a.ops:
    print("\n| enc | op | label | grid | stages | us | TFLOP/s |")
    print("|---|---|---|---|---|---|---|")
    for k, i, lab, us, f, inf in oprows:
        print(f"| {k} | {i} | {lab} | {inf.get('grid_x', '')} | {inf.get('stages', '')} | {us:.1f} | {f / us / 1e6:.0f} |")
