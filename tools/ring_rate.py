"""Steady-state device time per pass on the SERVED path: back-to-back
device-formed passes through MaskedModel.run_ring (pipelined: pass P+1's
compaction and stems overlap pass P), served-mix masks (61 requests,
rgb/flow/audio = 61/36/24), no host IO.  The mean over P passes between two
events on the serving stream; repeated R times (median reported).

    python tools/ring_rate.py [--passes 60] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--passes", type=int, default=60)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--counts", type=int, nargs=3, default=(61, 36, 24))
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=192)
counts = tuple(a.counts)
n = max(counts)
rng = np.random.default_rng(0)
masks = np.zeros(n, dtype=np.int16)
for k, c in enumerate(counts):
    masks[rng.permutation(n)[:c]] |= 1 << k
assert (masks != 0).all(), "every request needs a modality: max(counts) rows, rgb first"
for s in range(len(m.ring_ev)):
    m.mask_ring[s, :n].copy_(torch.as_tensor(masks))
import time  # noqa: E402

t_w = time.perf_counter()
m.ensure_warm()
torch.cuda.synchronize()
t_w = time.perf_counter() - t_w
rings = [0] * m.K
i = 0


def one():
    global i
    slot = i % len(m.ring_ev)
    i += 1
    bases = list(rings)
    for k in range(m.K):
        rings[k] = (bases[k] + counts[k]) % m.n_slots
    m.run_ring(n, counts, slot, bases)


e0, e1 = dv.Event(), dv.Event()
for _ in range(10):
    one()
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0.record()
    for _ in range(a.passes):
        one()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_us(e1) / a.passes)
print(f"served-path pass {counts}: {np.median(ts):8.1f} us/pass (reps {', '.join(f'{t:.1f}' for t in ts)}; warm {t_w:.1f} s)",
      flush=True)
