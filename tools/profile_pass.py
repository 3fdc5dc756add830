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
