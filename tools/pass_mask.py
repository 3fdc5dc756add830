"""Whole-pass device time (graphs, lanes, modality streams) for fixed-mask
batches, vs the serial sum of the encoder's op times."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=96)
e0, e1 = dv.Event(), dv.Event()
for mask in (1, 7):
    for n in (16, 32, 64, 96):
        masks = np.full(n, mask, dtype=np.int16)
        slots = np.arange(n)
        for lanes in (True, False):
            for e in m.encoders:
                e.program(1)
                e._lanes.concurrent = lanes
            m._graphs.clear()
            for _ in range(3):
                m.forward(slots, masks)
            ts = []
            for _ in range(7):
                e0.record()
                m.forward(slots, masks)
                e1.record()
                ts.append(e0.elapsed_us(e1))
            print(f"mask {mask} n={n:3d} lanes={'on ' if lanes else 'off'} pass {np.median(ts):8.1f} us "
                  f"({n / np.median(ts) * 1e6:8.0f} req/s)", flush=True)
