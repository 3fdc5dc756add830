"""Device time of whole TBN passes at several sizes (served modality mix
61/36/24 scaled, and all-modality), CUDA graphs, modality streams concurrent.

    python tools/pass_sizes.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=192)
e0, e1 = dv.Event(), dv.Event()
rng = np.random.default_rng(0)
for n in (1, 4, 12, 24, 40, 61, 96):
    masks = np.zeros(n, dtype=np.int16)
    for k, frac in enumerate((1.0, 36 / 61, 24 / 61)):
        c = max(1, int(round(frac * n))) if k == 0 else int(round(frac * n))
        masks[rng.permutation(n)[:c]] |= 1 << k
    masks[masks == 0] = 1
    slots = np.arange(n)
    for _ in range(3):
        m.forward(slots, masks)
    ts = []
    for _ in range(15):
        e0.record()
        m.forward(slots, masks)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_us(e1))
    print(f"n={n:3d} counts={m.counts_for(masks)} {np.median(ts):8.1f} us", flush=True)
