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


class PassCostModel:
    """Device cost of ONE masked pass for cross-job batching.

    The reference's cost model is additive per part (strategy.py:99-102),
    which overestimates a merged pass.  Here each modality encoder's graph
    and the fusion head are timed alone with CUDA events for every batch
    size, and a pass over compacted counts (N_1..N_K) is estimated as
    ``compact + sum_k enc_k(N_k) + head(N)`` scaled by an EWMA of
    observed/estimated pass time (the modality encoders overlap on side
    streams, which the EWMA learns).
    """

    def __init__(self, enc_us, head_us, compact_us: float, weight: float = 0.2):
        self.enc_us = [list(map(float, r)) for r in enc_us]  # [K][n-1]
        self.head_us = list(map(float, head_us))
        self.compact_us = float(compact_us)
        self.factor = 1.0
        self.weight = weight

    @property
    def max_n(self) -> int:
        return len(self.head_us)

    def raw_us(self, counts, n: int) -> float:
        t = self.compact_us + self.head_us[n - 1]
        for k, c in enumerate(counts):
            if c:
                t += self.enc_us[k][c - 1]
        return t

    def estimate_us(self, counts, n: int) -> float:
        return self.raw_us(counts, n) * self.factor

    def observe(self, counts, n: int, observed_us: float) -> None:
        r = observed_us / max(1.0, self.raw_us(counts, n))
        self.factor = (1.0 - self.weight) * self.factor + self.weight * r

    def to_json(self):
        return {"enc_us": self.enc_us, "head_us": self.head_us, "compact_us": self.compact_us}


def profile_pass_costs(model, max_n: int | None = None, reps: int = 5) -> PassCostModel:
    """Time every encoder graph (per modality, per count) and the head."""
    import torch
    top = min(max_n or model.max_req, model.max_req)
    e0, e1 = dv.Event(), dv.Event()

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            e0.record()
            fn()
            e1.record()
            ts.append(e0.elapsed_us(e1))
        return float(np.median(ts))

    enc = []
    for k, e in enumerate(model.encoders):
        row = []
        for n in range(1, top + 1):
            g = model._graph(("enc", k, n), e.program(n).run)
            row.append(timed(g.replay))
        enc.append(list(np.maximum.accumulate(row)))
    # head + compaction on a staged all-modality batch
    head = []
    masks = np.full(top, (1 << model.K) - 1, dtype=np.int16)
    model.stage_inputs(np.arange(top) % model.n_slots, masks)
    model._compact(top)
    model.stage_inputs(np.arange(top) % model.n_slots, masks)
    torch.cuda.synchronize()
    for n in range(1, top + 1):
        g = model._graph(("head", n), model._head(n).run)
        head.append(timed(g.replay))
    comp = timed(lambda: model._compact(top))
    return PassCostModel(enc, list(np.maximum.accumulate(head)), comp)
