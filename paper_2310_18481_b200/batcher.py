"""Pass formation on the device: the batched executor's policy step.

The reference scheduler decides one job at a time (``apply_policy`` then
``next_dispatch``, scheduler.py:382-449) and never batches across jobs
(SPEC.md:398).  The B200 executor runs one masked pass over many jobs, so its
policy step chooses every member's modality subset against the cost of THAT
pass: ``ms_pass_select`` (csrc/select.cu; contract in
``include/mosel_b200.h``), one warp per formation, P5's per-request argmax
 with the latency budget coupled through the shared pass.  It is
restated bit-for-bit by ``oracle/selection.py:pass_select``.

Host side (this module): each admitted job carries its frontier packed once
(per-candidate per-modality request counts and per-request masks, cached per
(size, SLO bucket) since frontiers depend only on those); a formation packs
the head and the EDF queue into pinned staging buffers that the kernel reads
in place (mapped host memory, no memcpy), the kernel writes the pass's
per-request masks straight into the device mask ring the compaction reads,
and the host reads back only (members, requests, per-modality counts,
estimate, choices) -- what it needs to pick the encoder graphs.
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass

import numpy as np

from . import device as dv
from .executor import request_masks
from .planner import StrategyMatrix, candidates_for_job
from .registry import scaled_accuracy


class FrontierPack:
    """A job's frontier in the kernel's layout."""

    __slots__ = ("size", "n_cand", "counts", "masks")

    def __init__(self, cands, size: int, K: int):
        self.size = size
        self.n_cand = len(cands)
        m = np.stack([request_masks(c.strategy.parts, size) for c in cands]).astype(np.uint16)  # [C, size]
        bits = (m[:, :, None].astype(np.int32) >> np.arange(K)) & 1
        self.counts = np.ascontiguousarray(bits.sum(axis=1), dtype=np.int16)  # [C, K]
        self.masks = np.ascontiguousarray(m.reshape(-1))


class FrontierCache:
    """candidates_with_rounding (scheduler.py:138-167) + FrontierPack, cached.

    For a profiled size the frontier (strategy.py:540-567) depends on the SLO
    only through which matrix alphas reach it (scaled_accuracy(alpha) >=
    scaled_accuracy(slo)), so (size, that count) keys the cache; rounded-up
    sizes are computed per call."""

    def __init__(self, matrix: StrategyMatrix, K: int, top_only: bool = False):
        """``top_only``: every job keeps only its most accurate candidate (the
        reference's ``none`` policy: no modality is ever dropped) -- the
        modality-agnostic baseline MOSEL is measured against."""
        from .policy import candidates_with_rounding
        self._cwr = candidates_with_rounding
        self.matrix = matrix
        self.K = K
        self.top_only = top_only
        self._alpha_scaled = sorted(scaled_accuracy(a) for a in matrix.alphas)
        self._sizes = set(matrix.sizes)
        self._cache = {}

    def warm_iter(self):
        """Fill every (profiled size, alpha count) entry, one per step (a
        frontier depends on the SLO only through that count): afterwards
        lookups during serving never miss."""
        for size in sorted(self._sizes):
            for c in range(len(self._alpha_scaled) + 1):
                if (size, c) in self._cache:
                    continue
                # an SLO whose scaled value bisects to c
                s_scaled = self._alpha_scaled[c] if c < len(self._alpha_scaled) else self._alpha_scaled[-1] + 1
                slo = s_scaled / 1e4
                if bisect.bisect_left(self._alpha_scaled, scaled_accuracy(slo)) != c:
                    continue  # float round trip landed elsewhere: leave it to lookup()
                self.lookup(size, slo)
                yield size, c

    def warm(self) -> None:
        for _ in self.warm_iter():
            pass

    def lookup(self, size: int, slo: float):
        """(candidates, FrontierPack or None when empty)."""
        if size in self._sizes:
            key = (size, bisect.bisect_left(self._alpha_scaled, scaled_accuracy(slo)))
            hit = self._cache.get(key)
            if hit is None:
                cands = candidates_for_job(self.matrix, size, slo)
                if self.top_only:
                    cands = cands[-1:]
                hit = (cands, FrontierPack(cands, size, self.K) if cands else None)
                self._cache[key] = hit
            return hit
        cands = self._cwr(self.matrix, size, slo)
        if self.top_only:
            cands = cands[-1:]
        return cands, (FrontierPack(cands, size, self.K) if cands else None)


@dataclass
class PassChoice:
    members: int
    requests: int
    counts: tuple
    est_ns: int
    choices: np.ndarray  # [members]


class DevicePassSelector:
    """Runs ``ms_pass_select`` for the serving loop on a high-priority stream.

    ``mask_ring``: device int16 [R, ld] -- formation i writes its pass's
    per-request masks into row ``slot``; ``slot_free[slot]`` (a CUDA event
    recorded by the caller after the compaction that last read that row) is
    waited on by the selection stream before it overwrites the row."""

    def __init__(self, K: int, cost: dv.PassCost, cap: int, max_pass_ns: int, mask_ring, record: bool = False):
        import torch
        self.torch = torch
        self.K = K
        self.cost = cost
        self.cap = int(cap)
        self.max_pass_ns = int(max_pass_ns)
        self.mask_ring = mask_ring
        self.stream = torch.cuda.Stream(priority=-1)
        self.ev0 = torch.cuda.Event(enable_timing=True)
        self.ev1 = torch.cuda.Event(enable_timing=True)
        self.launches = 0
        self.device_us = 0.0
        self.wait_us = 0.0
        self.record = record
        self.records = []
        self._cap_jobs = 0
        self._cap_rows = 0
        self._cap_masks = 0
        self._prob = torch.zeros(4, dtype=torch.int64).pin_memory()  # job_off, n_jobs (i32 x2), now, factor
        self._summary = torch.zeros(dv.PASS_SUMMARY, dtype=torch.int32).pin_memory()
        self._est = torch.zeros(1, dtype=torch.int64).pin_memory()
        self._clock = torch.zeros(2, dtype=torch.int64).pin_memory()  # kernel start/end (device global timer)
        self.kernel_us = 0.0
        self._grow(256, 4096, 16384)

    def _grow(self, jobs: int, rows: int, masks: int):
        torch = self.torch
        if jobs > self._cap_jobs:
            self._cap_jobs = jobs
            self._size = torch.zeros(jobs, dtype=torch.int32).pin_memory()
            self._dl = torch.zeros(jobs, dtype=torch.int64).pin_memory()
            self._ncand = torch.zeros(jobs, dtype=torch.int32).pin_memory()
            self._coff = torch.zeros(jobs, dtype=torch.int32).pin_memory()
            self._moff = torch.zeros(jobs, dtype=torch.int32).pin_memory()
            self._choice = torch.zeros(jobs, dtype=torch.int32).pin_memory()
        if rows > self._cap_rows:
            self._cap_rows = rows
            self._cc = torch.zeros(rows * self.K, dtype=torch.int16).pin_memory()
        if masks > self._cap_masks:
            self._cap_masks = masks
            self._rm = torch.zeros(masks, dtype=torch.int16).pin_memory()

    def select(self, jobs, now_us: int, factor: float, slot: int, slot_free=None) -> PassChoice:
        """One formation over ``jobs`` = [head] + the EDF queue (each with a
        ``pack`` FrontierPack)."""
        q = len(jobs)
        packs = [j.pack for j in jobs]
        ncand = np.fromiter((p.n_cand for p in packs), np.int32, q)
        size = np.fromiter((p.size for p in packs), np.int32, q)
        rows = int(ncand.sum())
        nmask = int((ncand * size).sum())
        if q > self._cap_jobs or rows > self._cap_rows or nmask > self._cap_masks:
            self._grow(max(q, 2 * self._cap_jobs) if q > self._cap_jobs else 0,
                       max(rows, 2 * self._cap_rows) if rows > self._cap_rows else 0,
                       max(nmask, 2 * self._cap_masks) if nmask > self._cap_masks else 0)
        sz = self._size.numpy()
        sz[:q] = size
        self._ncand.numpy()[:q] = ncand
        self._dl.numpy()[:q] = np.fromiter((j.deadline_us for j in jobs), np.int64, q)
        coff = self._coff.numpy()
        coff[0] = 0
        np.cumsum(ncand[:-1], out=coff[1:q])
        moff = self._moff.numpy()
        moff[0] = 0
        np.cumsum((ncand * size)[:-1], out=moff[1:q])
        np.concatenate([p.counts for p in packs], out=self._cc.numpy()[: rows * self.K].reshape(rows, self.K))
        np.concatenate([p.masks for p in packs], out=self._rm.numpy().view(np.uint16)[:nmask])
        pr = self._prob.numpy()
        pr.view(np.int32)[:2] = (0, q)
        pr[1] = now_us
        pr.view(np.float64)[2] = factor
        base = self._prob.data_ptr()
        # every launch names the selection stream explicitly (no stream context:
        # a framework stream switch costs tens of microseconds of host time per pass)
        if slot_free is not None:
            self.stream.wait_event(slot_free)
        self.ev0.record(self.stream)
        dv.pass_select(1, base, base + 4, base + 8, base + 16, self._size.data_ptr(), self._dl.data_ptr(),
                       self._ncand.data_ptr(), self._coff.data_ptr(), self._moff.data_ptr(), self._cc.data_ptr(),
                       self._rm.data_ptr(), self.cost, self.cap, self.max_pass_ns, self._choice.data_ptr(),
                       self._summary.data_ptr(), self._est.data_ptr(), self.mask_ring[slot].data_ptr(),
                       self.mask_ring.shape[1], stream=self.stream, out_clock=self._clock.data_ptr())
        self.ev1.record(self.stream)
        self.ev1.synchronize()
        self.launches += 1
        self.device_us += self.ev0.elapsed_time(self.ev1) * 1000.0
        clk = self._clock.numpy()
        self.kernel_us += (int(clk[1]) - int(clk[0])) / 1000.0
        summ = self._summary.numpy()
        m, n = int(summ[0]), int(summ[1])
        res = PassChoice(m, n, tuple(int(x) for x in summ[2:2 + self.K]), int(self._est.numpy()[0]),
                         self._choice.numpy()[:m].copy())
        if self.record:
            self.records.append(self.snapshot(q, rows, nmask, now_us, factor, res))
        return res

    def snapshot(self, q, rows, nmask, now_us, factor, res):
        """The formation's packed inputs and the kernel's outputs (parity replay)."""
        return {"size": self._size.numpy()[:q].copy(), "deadline_us": self._dl.numpy()[:q].copy(),
                "n_cand": self._ncand.numpy()[:q].copy(),
                "cand_counts": self._cc.numpy()[: rows * self.K].reshape(rows, self.K).copy(),
                "req_masks": self._rm.numpy().view(np.uint16)[:nmask].copy(), "now_us": int(now_us),
                "factor": float(factor), "members": res.members, "requests": res.requests,
                "counts": res.counts, "est_ns": res.est_ns, "choices": res.choices.copy()}


def unpack_jobs(rec, K: int):
    """A recorded formation as the oracle's job list."""
    jobs = []
    c0 = m0 = 0
    for s, d, nc in zip(rec["size"], rec["deadline_us"], rec["n_cand"]):
        s, nc = int(s), int(nc)
        cc = rec["cand_counts"][c0:c0 + nc]
        mk = rec["req_masks"][m0:m0 + nc * s].reshape(nc, s)
        jobs.append((s, int(d), cc, mk))
        c0 += nc
        m0 += nc * s
    return jobs
