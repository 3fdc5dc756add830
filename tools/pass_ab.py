"""A/B of whole masked TBN pass device time (CUDA graphs, modality streams
concurrent): programmatic dependent launch on/off x Inception branch lanes
concurrent/serial, all-modality and mixed masks.

    python tools/pass_ab.py [--ns 1,8,24,48,96]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="1,4,8,16,24,32,48,96")
ap.add_argument("--configs", default="base,pdl,lanes,pdl+lanes")
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import TBN_MODALITIES, request_flops  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

Ns = [int(x) for x in a.ns.split(",")]
fl = [request_flops(x) for x in TBN_MODALITIES]
e0, e1 = dv.Event(), dv.Event()
rng = np.random.default_rng(0)
mixed = {n: rng.integers(1, 8, size=n).astype(np.int16) for n in Ns}
res = {}
for cfg in a.configs.split(","):
    dv.set_pdl("pdl" in cfg)
    m = build_tbn_model(max_req=max(Ns), n_slots=max(Ns))
    for e in m.encoders:
        e.program(1)  # creates the lane context
        e._lanes.concurrent = "lanes" in cfg
    for n in Ns:
        for kind, masks in (("all", np.full(n, 7, dtype=np.int16)), ("mixed", mixed[n])):
            slots = np.arange(n)
            for _ in range(3):
                m.forward(slots, masks)
            ts = []
            for _ in range(7):
                e0.record()
                m.forward(slots, masks)
                e1.record()
                ts.append(e0.elapsed_us(e1))
            us = float(np.median(ts))
            flops = sum(fl[k] * int(((masks >> k) & 1).sum()) for k in range(3))
            res[(cfg, kind, n)] = us
            print(f"{cfg:10s} {kind:5s} n={n:3d} {us:8.1f} us {flops / us / 1e6:7.1f} TF/s "
                  f"{n / us * 1e6:8.1f} req/s", flush=True)
    del m
    torch.cuda.empty_cache()
dv.set_pdl(True)
