"""Device time of whole masked TBN passes (CUDA graphs), modality streams
concurrent vs serial, for a few batch sizes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import TBN_MODALITIES, request_flops  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=96)
e0, e1 = dv.Event(), dv.Event()
fl_req = sum(request_flops(x) for x in TBN_MODALITIES)
for n in (1, 8, 24, 48, 96):
    masks = np.full(n, 7, dtype=np.int16)
    slots = np.arange(n)
    res = {}
    for par in (True, False):
        m.parallel_modalities = par
        for _ in range(3):
            m.forward(slots, masks)
        ts = []
        for _ in range(5):
            e0.record()
            m.forward(slots, masks)
            e1.record()
            ts.append(e0.elapsed_us(e1))
        res[par] = float(np.median(ts))
    print(f"n={n:3d} concurrent {res[True]:8.1f} us  serial {res[False]:8.1f} us  "
          f"-> {n * fl_req / min(res.values()) / 1e6:6.1f} TFLOP/s, {n / min(res.values()) * 1e6:7.1f} req/s")
