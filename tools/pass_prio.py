"""Served-pass composition (61 rgb, 36 flow, 24 audio requests): pass device
time with modality side streams at equal vs descending priority."""
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
n = 61
masks = np.ones(n, dtype=np.int16)
masks[:36] |= 2
masks[20:44] |= 4
print("counts", m.counts_for(masks))
e0, e1 = dv.Event(), dv.Event()
slots = np.arange(n)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
for name, prios in (("equal", (0, 0, 0)), ("rgb>flow>audio", (-2, -1, 0)), ("rgb high", (-2, 0, 0))):
    m._side = [torch.cuda.Stream(priority=p) for p in prios]
    for _ in range(3):
        m.forward(slots, masks)
    ts = []
    for _ in range(9):
        e0.record()
        m.forward(slots, masks)
        e1.record()
        ts.append(e0.elapsed_us(e1))
    print(f"{name:16s} pass {np.median(ts):8.1f} us", flush=True)
