"""Run a few TBN masked passes for ncu (launch list / full capture).

    python tools/profile_pass.py --n 48 --mask 7 --reps 2 [--mixed]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--mask", type=int, default=7)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--graphs", type=int, default=0)
ap.add_argument("--mixed", action="store_true", help="masks uniform over the 7 combos")
a = ap.parse_args()

import torch  # noqa: E402
from paper_2310_18481_b200 import build  # noqa: E402
build.build()
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=a.n, n_slots=max(8, a.n))
m.use_graphs = bool(a.graphs)
rng = np.random.default_rng(0)
masks = rng.integers(1, 8, size=a.n).astype(np.int16) if a.mixed else np.full(a.n, a.mask, dtype=np.int16)
slots = np.arange(a.n) % m.n_slots
for _ in range(a.reps):
    m.forward(slots, masks)
torch.cuda.synchronize()
print("launches per pass", m.launches_per_pass(m.counts_for(masks)), "flops", m.flops(masks))

if a.graphs == 0:
    import json
    order = []
    counts = m.counts_for(masks)
    order.append(("compact_index", "", 0))
    for k, c in enumerate(counts):
        if c:
            order.append(("gather", f"mod{k}", 0))
    for k, (e, c) in enumerate(zip(m.encoders, counts)):
        if not c:
            continue
        for kind, op in e.program(c).ops:
            if kind == "gemm":
                order.append(("gemm", f"mod{k} " + op.label, op.flops))
            else:
                order.append((kind, f"mod{k}", 0))
    for kind, op in m.head.program(a.n, [e.out for e in m.encoders], m.inv[: m.K * a.n].view(m.K, a.n)).ops:
        order.append(("gemm", "head " + op.label, op.flops))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/pass_ops.json").write_text(json.dumps(order))
