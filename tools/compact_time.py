"""Device time of one pass's compaction (ms_compact: index + per-modality
gathers) for the TBN model at mixed masks, and its HBM roofline fraction."""
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
rng = np.random.default_rng(5)
for n in (24, 64, 96):
    masks = rng.integers(1, 8, size=n).astype(np.int16)
    slots = rng.integers(0, m.n_slots, size=n)
    m.stage_inputs(slots, masks)
    for _ in range(3):
        m._compact(n)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        m._compact(n)
    e1.record()
    us = e0.elapsed_us(e1) / 10
    b = m.compaction_bytes(masks)
    print(f"n={n:3d}: {us:7.1f} us  {b / 1e6:7.1f} MB  {b / us / 1e3:7.1f} GB/s")
