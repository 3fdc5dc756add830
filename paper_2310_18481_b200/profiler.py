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

    def __init__(self, enc_us, head_us, compact_us: float, weight: float = 0.2, pass_all_us=None):
        self.enc_us = [list(map(float, r)) for r in enc_us]  # [K][n-1]
        self.head_us = list(map(float, head_us))
        self.compact_us = float(compact_us)
        self.factor = 1.0
        self.weight = weight
        # measured whole all-modality passes [(n, us)]: with modality streams
        # overlapping at small n and not at large n, the sum of per-encoder
        # times is wrong at both ends; a pass is priced as the all-modality
        # pass of the same work (counts weighted by each encoder's marginal
        # cost), interpolated in n
        self.pass_all = sorted((int(n), float(t)) for n, t in (pass_all_us or []))
        top = len(self.head_us)
        ref = min(24, top)
        slope = [max(1e-3, (r[ref - 1] - r[0]) / max(1, ref - 1)) for r in self.enc_us]
        self.work_w = [x / sum(slope) for x in slope]  # all-modality request = 1 unit

    @property
    def max_n(self) -> int:
        return len(self.head_us)

    def pass_all_us(self, w: float) -> float:
        """Interpolated all-modality pass time at (fractional) work ``w``."""
        pts = self.pass_all
        if w <= pts[0][0]:
            return pts[0][1] * max(w, 0.0) / pts[0][0] if w < 1.0 else pts[0][1]
        for (n0, t0), (n1, t1) in zip(pts, pts[1:]):
            if w <= n1:
                return t0 + (t1 - t0) * (w - n0) / (n1 - n0)
        (n0, t0), (n1, t1) = pts[-2], pts[-1]
        return t1 + (t1 - t0) / (n1 - n0) * (w - n1)

    def work(self, counts) -> float:
        return sum(wk * c for wk, c in zip(self.work_w, counts))

    def raw_us(self, counts, n: int) -> float:
        if len(self.pass_all) >= 2:
            return self.pass_all_us(max(1.0, self.work(counts)))
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

    def device_table(self):
        """The integer pass-time model ``ms_pass_select`` evaluates
        (``dv.PassCost``): per-request work of modality k in 1/1024 of an
        all-modality request (``work_w``), and the measured all-modality
        passes as knots (work, ns), non-decreasing; below the first knot the
        first time (this model's ``max(1, work)`` clamp), past the last the
        last segment extrapolated."""
        if len(self.pass_all) < 1:
            raise ValueError("device_table needs measured whole passes (profile_pass_costs)")
        w = [int(round(x * 1024)) for x in self.work_w]
        u = [int(n) * 1024 for n, _ in self.pass_all]
        t = np.maximum.accumulate([int(round(v * 1000.0)) for _, v in self.pass_all]).tolist()
        return dv.PassCost.make(w, u, t)

    def to_json(self):
        return {"enc_us": self.enc_us, "head_us": self.head_us, "compact_us": self.compact_us,
                "pass_all_us": self.pass_all, "work_w": self.work_w}


def marginal_profile(cost: PassCostModel, modalities, accuracy, max_batch: int, ref_n: int = 24,
                     part_fixed_us: float | None = None, name: str = "tbn-b200-batched") -> ModelProfile:
    """The latency table a BATCHING executor should hand the reference's
    scheduler.  The reference cost model is additive per part
    (strategy.py:99-102) with each part priced as if it ran alone
    (profile.py:164-168); under cross-job batching a part really costs its
    marginal share of a merged pass.  Here ``latency(mask, b) = F + b *
    sum_{k in mask} m_k`` where ``m_k`` is encoder k's measured marginal
    per-request time (slope of the CUDA-event pass costs between batch 1 and
    ``ref_n``) and ``F`` a per-part share of the fixed pass cost (default:
    the fixed cost of an all-modality pass divided by the jobs a pass of
    ``ref_n`` requests typically merges, ~6).  Strategies, frontiers and the
    ``optimized`` policy then trade accuracy for the time modalities really
    cost in a batched pass, so under load the policy drops modalities
    (MOSEL's selection) instead of seeing no violation until requests are
    already late.  The latency-feedback EWMA (scheduler.py:86-91) corrects
    the residual scale.  Monotone by construction; ints >= 1 (profile.py)."""
    ref_n = max(2, min(ref_n, cost.max_n))
    if len(cost.pass_all) >= 2:  # slope of whole measured passes, split by encoder work share
        slope = (cost.pass_all_us(ref_n) - cost.pass_all_us(1)) / (ref_n - 1)
        marg = [slope * w for w in cost.work_w]
        fixed = cost.pass_all_us(1) - slope
    else:
        marg = [(r[ref_n - 1] - r[0]) / (ref_n - 1) for r in cost.enc_us]
        fixed = cost.compact_us + cost.head_us[0] + max(r[0] - m for r, m in zip(cost.enc_us, marg))
    if part_fixed_us is None:
        part_fixed_us = fixed / 6.0
    k = len(modalities)
    rows = []
    for mask in range(1, 1 << k):
        per = sum(marg[j] for j in range(k) if (mask >> j) & 1)
        rows.append(tuple(max(1, int(round(part_fixed_us + b * per))) for b in range(1, max_batch + 1)))
    return ModelProfile(name, tuple(modalities), max_batch, tuple(rows), tuple(accuracy))


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
    # whole all-modality passes exactly as serving runs them (graphs, modality streams)
    full = (1 << model.K) - 1
    grid = sorted({n for n in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, top) if n <= top})
    rng = np.random.default_rng(3)
    pass_all = [(n, time_pass(model, rng.integers(0, model.n_slots, size=n), np.full(n, full, dtype=np.int16),
                              reps=reps)) for n in grid]
    t = np.maximum.accumulate([v for _, v in pass_all])
    return PassCostModel(enc, list(np.maximum.accumulate(head)), comp,
                         pass_all_us=[(n, float(v)) for (n, _), v in zip(pass_all, t)])
