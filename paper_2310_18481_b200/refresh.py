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
     whose work lies nearest to it (>= ``min_obs`` of them; otherwise by the
     median ratio of all passes), then made non-decreasing;
  3. a helper PROCESS derives the serving profile from the new model
     (``profiler.marginal_profile``, the reference YAML table) and rebuilds
     the strategy matrix (the host DP, byte-identical to the device DP
     ``ms_strategy_dp`` used for offline builds), checking its fingerprint
     against the new profile;
  4. the serving loop fills the new frontier cache a few entries at a time
     while the GPU queue is full (``advance``), then swaps (cost model,
     device cost table, frontier cache, profile, matrix) atomically between
     two pass formations.  Jobs already queued keep their frontiers; new
     arrivals use the new matrix.  The new model's EWMA factor continues the
     old one (old factor / the ratio the knots absorbed), so a swap changes
     no prediction abruptly.

Why a process and not a thread: a Python build thread in the serving process
holds the GIL for ~0.1 s, and every ctypes call of the serving loop (event
queries, launches, ms_pass_select) releases and re-acquires the GIL -- each
re-acquire waited out the builder's switch interval, and passes went late in
a burst after every swap (tools/refresh_diag.py: 2-11 % of requests late with
a build thread, 0 % without the refresher).
"""

from __future__ import annotations

import os
import pickle
import struct
import subprocess
import sys
import threading
import time
from dataclasses import dataclass

import numpy as np

from .batcher import FrontierCache
from .planner import MatrixError, StrategyMatrix, build_matrix
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
    fcache: object
    absorbed: float


def _rebuild(cost: PassCostModel, modalities, accuracy, max_batch, name, sizes, alphas):
    """Helper-process side of a refresh: serving profile + strategy matrix."""
    t0 = time.perf_counter()
    prof = marginal_profile(cost, modalities, accuracy, max_batch, name=name)
    m = build_matrix(prof, sizes, alphas)
    return prof, m, time.perf_counter() - t0


def _read_exact(fd: int, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        chunk = os.read(fd, n - len(buf))
        if not chunk:
            raise EOFError("refresh helper closed its pipe")
        buf += chunk
    return bytes(buf)


def _send(fd: int, obj) -> None:
    data = pickle.dumps(obj, protocol=pickle.HIGHEST_PROTOCOL)
    os.write(fd, struct.pack("<Q", len(data)))
    view = memoryview(data)
    while len(view):
        view = view[os.write(fd, view):]


def _worker_main() -> None:
    """``python -m paper_2310_18481_b200.refresh``: serve rebuild requests
    (pickled argument tuples on stdin) until EOF; reply (ok, result) on stdout."""
    fin, fout = sys.stdin.fileno(), sys.stdout.fileno()
    while True:
        try:
            n = struct.unpack("<Q", _read_exact(fin, 8))[0]
        except EOFError:
            return
        args = pickle.loads(_read_exact(fin, n))
        try:
            _send(fout, (True, _rebuild(*args)))
        except Exception as e:  # noqa: BLE001 -- surfaced in the serving process
            _send(fout, (False, e))


class _Helper:
    """One persistent helper interpreter (a fresh ``python -m``, no CUDA, no
    torch) and a reader thread that collects each reply's bytes off the
    serving thread (os.read releases the GIL); the serving thread unpickles."""

    def __init__(self):
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        self.proc = subprocess.Popen([sys.executable, "-m", "paper_2310_18481_b200.refresh"], stdin=subprocess.PIPE,
                                     stdout=subprocess.PIPE, env=env, cwd=root)
        self._reply = None
        self._thread = None

    def submit(self, args) -> None:
        _send(self.proc.stdin.fileno(), args)
        self._reply = None

        def read():
            fd = self.proc.stdout.fileno()
            try:
                n = struct.unpack("<Q", _read_exact(fd, 8))[0]
                self._reply = _read_exact(fd, n)
            except EOFError as e:
                self._reply = pickle.dumps((False, e))

        self._thread = threading.Thread(target=read, daemon=True)
        self._thread.start()

    def done(self) -> bool:
        return self._thread is not None and not self._thread.is_alive()

    def result(self):
        self._thread = None
        ok, val = pickle.loads(self._reply)
        if not ok:
            raise val
        return val

    def close(self) -> None:
        try:
            self.proc.stdin.close()
        except OSError:
            pass
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()


class ProfileRefresher:
    def __init__(self, cost: PassCostModel, modalities, accuracy, max_batch: int, sizes, alphas,
                 period_s: float = 1.0, min_obs: int = 16, name: str = "tbn-b200-batched", top_only: bool = False):
        self.cost = cost
        self.modalities = tuple(modalities)
        self.accuracy = tuple(accuracy)
        self.max_batch = max_batch
        self.sizes = tuple(sizes)
        self.alphas = tuple(alphas)
        self.period_s = period_s
        self.min_obs = min_obs
        self.name = name
        self.top_only = top_only
        self._obs = []  # (work, us)
        self._last = None
        self._busy = False
        self._pending = None  # (Refresh, warm iterator) being filled by advance()
        self.history: list[Refresh] = []
        self._helper = _Helper()  # starts now: its imports overlap serving warm-up

    def observe(self, counts, n: int, dur_us: float) -> None:
        self._obs.append((max(1.0, self.cost.work(counts)), float(dur_us)))

    def due(self, now_s: float) -> bool:
        if self._busy or self._pending is not None:
            return False
        if self._last is None:
            self._last = now_s
            return False
        return now_s - self._last >= self.period_s and len(self._obs) >= self.min_obs

    def refit(self, obs):
        """(new knots, global ratio): each knot scaled by the median
        observed/modelled raw time of the observations nearest to it (in
        work), or by the median over all observations when fewer than
        ``min_obs`` are near it; then non-decreasing."""
        pts = self.cost.pass_all
        ns = np.array([n for n, _ in pts], dtype=float)
        w = np.array([o[0] for o in obs])
        r = np.array([o[1] / max(1.0, self.cost.pass_all_us(o[0])) for o in obs])
        g = float(np.median(r))
        near = np.abs(w[:, None] - ns[None, :]).argmin(axis=1)
        new = []
        for i, (n, t) in enumerate(pts):
            sel = r[near == i]
            new.append((n, t * (float(np.median(sel)) if len(sel) >= self.min_obs else g)))
        ts = np.maximum.accumulate([t for _, t in new])
        return [(n, float(t)) for (n, _), t in zip(new, ts)], g

    def start(self, now_s: float) -> None:
        obs, self._obs = self._obs, []
        self._last = now_s
        knots, g = self.refit(obs)
        c = self.cost
        new_cost = PassCostModel(c.enc_us, c.head_us, c.compact_us, c.weight, pass_all_us=knots)
        new_cost.work_w = list(c.work_w)  # the encoders' work shares are not re-fitted
        self._meta = (now_s, new_cost, list(c.pass_all), knots, g)
        self._helper.submit((new_cost, self.modalities, self.accuracy, self.max_batch, self.name, self.sizes,
                             self.alphas))
        self._busy = True

    def advance(self, entries: int = 16) -> None:
        """Serving-loop slice: collect a finished rebuild, then fill its
        frontier cache ``entries`` lookups at a time."""
        if self._busy and self._helper.done():
            self._busy = False
            prof, m, build_s = self._helper.result()  # re-raises a failed rebuild
            if m.profile_fingerprint != prof.fingerprint():  # strategy.py:505-520 stale-matrix rule
                raise MatrixError("refreshed matrix fingerprint does not match its profile")
            at_s, new_cost, before, knots, g = self._meta
            fc = FrontierCache(m, len(self.modalities), top_only=self.top_only)
            self._pending = (Refresh(at_s, new_cost, prof, m, build_s, before, knots, fc, g), fc.warm_iter())
        if self._pending is not None:
            it = self._pending[1]
            for _ in range(entries):
                if next(it, None) is None:
                    self._pending = (self._pending[0], None)
                    break

    def poll(self):
        """The finished, warmed refresh (once), or None."""
        if self._pending is None or self._pending[1] is not None:
            return None
        res, self._pending = self._pending[0], None
        # continue the serving model's EWMA: the knots absorbed ratio g
        res.cost.factor = self.cost.factor / max(1e-6, res.absorbed)
        self.cost = res.cost
        self.history.append(res)
        return res

    def close(self):
        self._helper.close()


if __name__ == "__main__":
    _worker_main()
