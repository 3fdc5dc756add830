"""Device time of whole TBN passes at the bench's served mix (rgb/flow/audio
counts 61/36/24 of 61 requests) and all-modality 96-request passes, through
model.forward (CUDA graphs, modality streams concurrent).  Env A/B switches
(MS_*) apply as set by the caller.

    python tools/pass_mix.py
"""
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

import os  # noqa: E402

if os.environ.get("MS_PDL") == "0":
    dv.set_pdl(False)
m = build_tbn_model(max_req=96, n_slots=192)
if os.environ.get("MS_SERIAL") == "1":
    m.parallel_modalities = False
e0, e1 = dv.Event(), dv.Event()
fl = [request_flops(x) for x in TBN_MODALITIES]
rng = np.random.default_rng(0)


def mix(n, counts):
    masks = np.zeros(n, dtype=np.int16)
    for k, c in enumerate(counts):
        masks[rng.permutation(n)[:c]] |= 1 << k
    masks[masks == 0] = 1
    return masks


for name, masks in (("served mix 61/36/24", mix(61, (61, 36, 24))), ("served mix 96 (96/57/38)", mix(96, (96, 57, 38))),
                    ("all-modality 96", np.full(96, 7, dtype=np.int16)), ("all-modality 24", np.full(24, 7, dtype=np.int16))):
    n = len(masks)
    slots = np.arange(n)
    for _ in range(3):
        m.forward(slots, masks)
    ts = []
    for _ in range(10):
        e0.record()
        m.forward(slots, masks)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_us(e1))
    flops = sum(fl[k] * int(((masks >> k) & 1).sum()) for k in range(3))
    t = float(np.median(ts))
    print(f"{name:28s} {t:8.1f} us  {flops / t / 1e6:6.0f} TFLOP/s  ({n / t * 1e6:7.0f} req/s if back to back)")
