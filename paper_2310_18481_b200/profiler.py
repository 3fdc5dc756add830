"""Device-side profiler: refreshes the (combo x batch) latency table from
CUDA-event timings of the real masked forward.

The reference's profiles are hand-written or synthetic tables
(profile.py:96-212, :402-443); MOSEL profiled with PyTorch + CUDA
(PAPER.md:434).  Here every cell is the median CUDA-event time of one
device pass of ``batch`` requests all using combo ``mask``, made
non-decreasing in batch size (``load_profile`` rejects decreasing rows,
profile.py:136-140) and emitted as a ``ModelProfile`` that ``save_profile``
writes in the reference YAML format.  Accuracies cannot be measured on a
random-init model, so they come from a fixed table.
"""

from __future__ import annotations

import numpy as np

from . import device as dv
from .registry import ModelProfile

# Fixed synthetic EPIC-style combo accuracies for the TBN rgb/flow/audio
# model, indexed by mask-1 (bit0 rgb, bit1 flow, bit2 audio); supersets are
# more accurate, audio alone least.
TBN_ACCURACY = (0.55, 0.50, 0.62, 0.38, 0.60, 0.56, 0.66)


def time_pass(model, slots, masks, reps: int = 5, warmup: int = 1):
    """Median CUDA-event microseconds of ``model.forward(slots, masks)``."""
    e0, e1 = dv.Event(), dv.Event()
    for _ in range(warmup):
        model.forward(slots, masks)
    times = []
    for _ in range(reps):
        e0.record()
        model.forward(slots, masks)
        e1.record()
        times.append(e0.elapsed_us(e1))
    return float(np.median(times))


def profile_model(model, modalities, accuracy, max_batch: int, name: str = "tbn-b200",
                  reps: int = 5, seed: int = 0) -> ModelProfile:
    """Sweep every combo x batch 1..max_batch on the device."""
    k = len(modalities)
    rng = np.random.default_rng(seed)
    rows = []
    for mask in range(1, 1 << k):
        row = []
        for b in range(1, max_batch + 1):
            slots = rng.integers(0, model.n_slots, size=b)
            us = time_pass(model, slots, np.full(b, mask, dtype=np.int16), reps=reps)
            row.append(max(1, int(round(us))))
        rows.append(tuple(int(v) for v in np.maximum.accumulate(row)))
    return ModelProfile(name, tuple(modalities), max_batch, tuple(rows), tuple(accuracy))


def refresh_profile(profile: ModelProfile, model, masks_batches, reps: int = 3) -> ModelProfile:
    """Re-measure only the given (mask, batch) cells and return an updated,
    still monotone profile (the online refresh path)."""
    table = [list(r) for r in profile.latency_us]
    rng = np.random.default_rng(1)
    for mask, b in masks_batches:
        slots = rng.integers(0, model.n_slots, size=b)
        table[mask - 1][b - 1] = max(1, int(round(time_pass(model, slots, np.full(b, mask), reps))))
    table = [tuple(int(v) for v in np.maximum.accumulate(r)) for r in table]
    return ModelProfile(profile.name, profile.modalities, profile.max_batch, tuple(table),
                        profile.accuracy)
