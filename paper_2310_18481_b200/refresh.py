"""Profiler -> matrix refresh loop during serving.

The paper's draft exploration stage keeps re-running the offline algorithm
and "constantly update[s] the policy"; the reference can
only rebuild a matrix offline against a profile fingerprint
(strategy.py:505-520, load_matrix's stale-matrix check).  Here a serving
replica re-profiles itself from the CUDA-event durations of the passes it is
already running -- no serving pause:

  1. every completed pass contributes (work, device us);
  2. every ``period_s`` the knots of the pass cost model are re-fitted: each
     knot is scaled by the median observed / modelled ratio of the passes
     whose work lies nearest to it (>= ``min_obs`` of them), then made
     non-decreasing;
  3. a background thread derives the serving profile from the new model
     (``profiler.marginal_profile``, the reference YAML table), rebuilds the
     strategy matrix with the device DP (``ms_strategy_dp`` on its own
     low-priority stream; byte-identical to the host DP) and checks its
     fingerprint against the new profile;
  4. the serving loop swaps (cost model, device cost table, frontier cache,
     profile, matrix) atomically between two pass formations.  Jobs already
     queued keep their frontiers; new arrivals use the new matrix.
"""

from __future__ import annotations

import sys
import threading
import time
from dataclasses import dataclass

import numpy as np

from .planner import MatrixError, StrategyMatrix, build_matrix_device
from .profiler import PassCostModel, marginal_profile
from .registry import ModelProfile


@dataclass
class Refresh:
    at_s: float
    cost: PassCostModel
    profile: ModelProfile
    matrix: StrategyMatrix
    build_s: float
    knots_before: list
    knots_after: list


class ProfileRefresher:
    def __init__(self, cost: PassCostModel, modalities, accuracy, max_batch: int, sizes, alphas,
                 period_s: float = 1.0, min_obs: int = 16, name: str = "tbn-b200-batched"):
        self.cost = cost
        self.modalities = tuple(modalities)
        self.accuracy = tuple(accuracy)
        self.max_batch = max_batch
        self.sizes = tuple(sizes)
        self.alphas = tuple(alphas)
        self.period_s = period_s
        self.min_obs = min_obs
        self.name = name
        self._obs = []  # (work, us)
        self._last = None
        self._thread = None
        self._result = None
        self._error = None
        self.history: list[Refresh] = []

    def observe(self, counts, n: int, dur_us: float) -> None:
        self._obs.append((max(1.0, self.cost.work(counts)), float(dur_us)))

    def due(self, now_s: float) -> bool:
        if self._thread is not None:
            return False
        if self._last is None:
            self._last = now_s
            return False
        return now_s - self._last >= self.period_s and len(self._obs) >= self.min_obs

    def refit(self, obs):
        """New knots: each scaled by the median observed/modelled raw time of
        the observations nearest to it (in work), then non-decreasing."""
        pts = self.cost.pass_all
        ns = np.array([n for n, _ in pts], dtype=float)
        w = np.array([o[0] for o in obs])
        r = np.array([o[1] / max(1.0, self.cost.pass_all_us(o[0])) for o in obs])
        near = np.abs(w[:, None] - ns[None, :]).argmin(axis=1)
        new = []
        for i, (n, t) in enumerate(pts):
            sel = r[near == i]
            new.append((n, t * float(np.median(sel)) if len(sel) >= self.min_obs else t))
        ts = np.maximum.accumulate([t for _, t in new])
        return [(n, float(t)) for (n, _), t in zip(new, ts)]

    def start(self, now_s: float) -> None:
        obs, self._obs = self._obs, []
        self._last = now_s
        knots = self.refit(obs)
        c = self.cost
        new_cost = PassCostModel(c.enc_us, c.head_us, c.compact_us, c.weight, pass_all_us=knots)
        new_cost.work_w = list(c.work_w)  # the encoders' work shares are not re-fitted
        before = list(c.pass_all)

        def work():
            import torch
            t0 = time.perf_counter()
            old = sys.getswitchinterval()
            sys.setswitchinterval(2e-4)  # short GIL slices: the serving loop keeps its latency
            try:
                prof = marginal_profile(new_cost, self.modalities, self.accuracy, self.max_batch, name=self.name)
                st = torch.cuda.Stream(priority=0)
                with torch.cuda.stream(st):
                    m = build_matrix_device(prof, self.sizes, self.alphas)
                st.synchronize()
                if m.profile_fingerprint != prof.fingerprint():  # strategy.py:505-520 stale-matrix rule
                    raise MatrixError("refreshed matrix fingerprint does not match its profile")
                self._result = Refresh(now_s, new_cost, prof, m, time.perf_counter() - t0, before, knots)
            except Exception as e:  # surfaced by poll()
                self._error = e
            finally:
                sys.setswitchinterval(old)

        self._thread = threading.Thread(target=work, daemon=True)
        self._thread.start()

    def poll(self):
        """The finished refresh (once), or None; re-raises a failed one."""
        if self._thread is None or self._thread.is_alive():
            return None
        self._thread = None
        if self._error is not None:
            e, self._error = self._error, None
            raise e
        res, self._result = self._result, None
        if res is not None:
            res.cost.factor = 1.0  # the knots absorbed the observed bias
            self.cost = res.cost
            self.history.append(res)
        return res

    def close(self):
        if self._thread is not None:
            self._thread.join()
            self._thread = None
