"""ORACLE — CPU restatement of the selection half of the hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker.  The product package never imports it.

Every function restates one piece of the reference (``/root/reference/pkg/
src/modserve``) in plain Python/numpy integer arithmetic and cites the
lines it follows.  It is pinned against golden vectors produced by the real
reference (``tests/golden/make_golden.py``) in ``tests/test_oracle.py``.
"""

from __future__ import annotations

import math

import numpy as np

ACC_SCALE = 10_000  # profile.py:25
DROP = -1


# --------------------------------------------------------------------------
# scalar semantics


def scaled_accuracy(acc: float) -> int:
    """profile.py:41-47 — floor(acc * 1e4 + 1e-9)."""
    return math.floor(acc * ACC_SCALE + 1e-9)


def credit_threshold(alpha: float, size: int) -> int:
    """strategy.py:119-125 / scheduler.py:166 — ceil(alpha*size*1e4 - 1e-6)."""
    return max(0, math.ceil(alpha * size * ACC_SCALE - 1e-6))


def estimate_us(latency_us: int, factor: float) -> int:
    """scheduler.py:82-83 — Python round() of a float64 product (half-even)."""
    return round(latency_us * factor)


def feedback_update(factor: float, predicted_us: int, observed_us: int,
                    weight: float = 0.2) -> float:
    """scheduler.py:86-91 — EWMA, evaluated in exactly this order in fp64."""
    return (1.0 - weight) * factor + weight * (observed_us / predicted_us)


# --------------------------------------------------------------------------
# P5: the per-job policy step


def policy_select_one(lat_us, deadline_us: int, dispatch_us: int,
                      factor: float) -> int:
    """Closed form of ``apply_policy(OPTIMIZED)`` on a one-job queue.

    Follows scheduler.py:382-425 (apply_policy) through detect_violation
    (:202-209), compute_budget (:212-233), reassign_optimized's 1 ms grid
    (:251-294) and try_upgrade (:366-379):

      est_i = round(lat_i * f)
      B     = deadline - dispatch
      1. est_top <= B                      -> top
      2. B <= 0                            -> DROP
      3. ceil(est_0/1000) > floor(B/1000)  -> DROP (ms-grid quirk)
      4. otherwise max{i : est_i <= B}
    """
    n = len(lat_us)
    if n == 0:
        return DROP
    est = [estimate_us(int(v), factor) for v in lat_us]
    budget = deadline_us - dispatch_us
    if est[-1] <= budget:
        return n - 1
    if budget <= 0:
        return DROP
    if -(-est[0] // 1000) > budget // 1000:
        return DROP
    best = 0
    for i in range(n):
        if est[i] <= budget:
            best = i
    return best


def policy_select(lat_us: np.ndarray, n_cand: np.ndarray, deadline_us: np.ndarray,
                  dispatch_us: int, factor: float) -> np.ndarray:
    """Batched P5 over an SoA candidate table ``lat_us[N, C]``."""
    out = np.empty(len(n_cand), dtype=np.int32)
    for j in range(len(n_cand)):
        out[j] = policy_select_one(lat_us[j, : n_cand[j]], int(deadline_us[j]),
                                   dispatch_us, factor)
    return out


def dispatch_drop(lat_fastest_us: int, deadline_us: int, now_us: int,
                  factor: float) -> bool:
    """scheduler.py:439-444 — head dropped if now + est(fastest) > deadline."""
    return now_us + estimate_us(lat_fastest_us, factor) > deadline_us


# --------------------------------------------------------------------------
# frontier (S5/S6)


def frontier(cells, slo_scaled: int):
    """strategy.py:540-567 restated.

    ``cells`` is a list of (alpha_scaled, key, latency_us, credit) for one
    job size, ``key`` identifying the strategy.  Returns the Pareto list of
    (key, latency_us, credit) sorted by latency with strictly increasing
    credit.
    """
    pool = {}
    for alpha_scaled, key, lat, credit in cells:
        if alpha_scaled < slo_scaled:
            continue
        pool[key] = (lat, credit)
    ranked = sorted(pool.items(), key=lambda kv: (kv[1][0], -kv[1][1]))
    out = []
    for key, (lat, credit) in ranked:
        if out and credit <= out[-1][2]:
            continue
        out.append((key, lat, credit))
    return out


# --------------------------------------------------------------------------
# grouping (G2) and compaction (G1)


def parts_for_requests(parts, size: int):
    """G2(i): requests 0..size-1, in index order, fill the job's canonical
    parts (strategy.py:54-60) in order; for a rounded-up strategy
    (scheduler.py:138-167: more part rows than requests) the parts are taken
    in order of decreasing modality count, so the rows truncated are the
    least-informed subsets; an empty part is skipped.  Returns (mask per
    request, [(mask, lo, hi)])."""
    masks = np.zeros(size, dtype=np.uint16)
    spans = []
    lo = 0
    if sum(b for _, b in parts) > size:  # rounded up: the most-modality parts first (stable)
        parts = sorted(parts, key=lambda pb: -bin(int(pb[0])).count("1"))
    for mask, batch in parts:
        hi = min(size, lo + batch)
        if hi > lo:
            masks[lo:hi] = mask
            spans.append((mask, lo, hi))
        lo = hi
    return masks, spans


def group_free_masks(masks: np.ndarray, max_batch: int):
    """G2(ii): stable counting sort of requests by mask ascending; each mask
    group chunked like all_modalities_strategy (strategy.py:109-116) and
    sorted by (mask, batch) so the remainder chunk comes first.

    Returns (perm, combo_offsets[2^K+1] over masks 0..2^K-1, chunks) where
    chunks is a list of (mask, start, count) into perm.
    """
    masks = np.asarray(masks, dtype=np.int64)
    n_masks = int(masks.max()) + 1 if masks.size else 1
    n_masks = 1 << max(1, int(n_masks - 1).bit_length())
    perm = np.argsort(masks, kind="stable").astype(np.int32)
    counts = np.bincount(masks, minlength=n_masks)
    offsets = np.zeros(n_masks + 1, dtype=np.int32)
    offsets[1:] = np.cumsum(counts)
    chunks = []
    for m in range(1, n_masks):
        c = int(counts[m])
        if c == 0:
            continue
        sizes = [max_batch] * (c // max_batch)
        if c % max_batch:
            sizes.append(c % max_batch)
        sizes.sort()
        start = int(offsets[m])
        for s in sizes:
            chunks.append((m, start, s))
            start += s
    return perm, offsets, chunks


def compact(masks: np.ndarray, n_modalities: int):
    """G1: per modality k the stable list idx_k = [i : mask_i>>k & 1], the
    counts, and the inverse map inv_k[i] (position in idx_k or -1)."""
    masks = np.asarray(masks, dtype=np.int64)
    idx, inv, counts = [], [], []
    for k in range(n_modalities):
        sel = np.flatnonzero((masks >> k) & 1).astype(np.int32)
        iv = np.full(len(masks), -1, dtype=np.int32)
        iv[sel] = np.arange(len(sel), dtype=np.int32)
        idx.append(sel)
        inv.append(iv)
        counts.append(len(sel))
    return idx, inv, np.asarray(counts, dtype=np.int32)


def dropped_modalities(mask: int, n_modalities: int) -> int:
    """profile.py:157-159 — dropped set = all_mask & ~mask."""
    return ((1 << n_modalities) - 1) & ~mask


# --------------------------------------------------------------------------
# Pass-level selection (the served policy step of the batched executor)
#
# The reference never batches across jobs; SURVEY §8f #4 asks
# for a cost model of its own.  This is the restatement that pins the device
# kernel ``ms_pass_select`` (csrc/select.cu) bit-for-bit.  Its per-member step
# is P5 (above) with the budget coupled through the shared pass: the largest
# frontier index whose PASS estimate meets every member's deadline, the jobs
# left queued, and the pass-length cap.  Integer arithmetic throughout except
# the fp64 EWMA factor, applied exactly like scheduler.py:82-83 (one fp64
# multiply, round half-even).


SLOPE_SHIFT = 20


def pass_raw_ns(u: int, pts_u, pts_t) -> int:
    """Piecewise-linear pass time (ns) at work ``u`` (1/1024-request units):
    clamped to the first knot below it, the first segment whose right knot is
    >= u, the last segment extrapolated past it; each segment's slope is held
    in 2^-20 ns per work unit, floor((dt << 20) / du), and applied with an
    arithmetic shift (all terms non-negative)."""
    n = len(pts_u)
    if n == 1 or u <= pts_u[0]:
        return int(pts_t[0])
    i = 0
    while i + 2 < n and u > pts_u[i + 1]:
        i += 1
    slope = ((int(pts_t[i + 1]) - int(pts_t[i])) << SLOPE_SHIFT) // (int(pts_u[i + 1]) - int(pts_u[i]))
    return int(pts_t[i]) + (((u - int(pts_u[i])) * slope) >> SLOPE_SHIFT)


def pass_estimate_ns(counts, w, pts_u, pts_t, factor: float) -> int:
    """round(raw(sum_k w_k * counts_k) * factor), half-even like Python round."""
    u = 0
    for wk, c in zip(w, counts):
        u += int(wk) * int(c)
    return round(pass_raw_ns(u, pts_u, pts_t) * factor)


def pass_select(jobs, now_us: int, w, pts_u, pts_t, factor: float, cap: int,
                max_pass_ns: int):
    """One pass formation.

    ``jobs``: the head (already popped by next_dispatch, scheduler.py:428-449)
    followed by the queued jobs in EDF order, each ``(size, deadline_us,
    cand_counts[C][K], cand_masks[C][size])``; candidates are the job's
    frontier (latency up, credit strictly up, strategy.py:540-567).

      1. membership: queued jobs join in EDF order at their fastest candidate
         while n <= cap, now + est <= every member's deadline and
         est <= max_pass (max_pass_ns < 0: no cap); the first misfit ends it;
      2. rest = the jobs left queued: rest_fast = est(their fastest counts),
         rest_dl = the earliest rest deadline >= now + est + rest_fast
         (the jobs one following all-fastest pass can still serve);
      3. upgrades: each member in EDF order takes the LARGEST candidate index
         >= its current one whose pass estimate keeps now + est <= tight
         (the members' earliest deadline), now + est + rest_fast <= rest_dl
         and est <= max_pass; repeated until no member moves.

    Returns (members M, choices[M], est_ns, counts[K], masks[n_req]).
    """
    K = len(w)
    now_ns = now_us * 1000

    def est(c):
        return pass_estimate_ns(c, w, pts_u, pts_t, factor)

    size0, dl0, cc0, _ = jobs[0]
    counts = [int(x) for x in cc0[0]]
    n = int(size0)
    tight = int(dl0)
    m = 1
    for size, dl, cc, _ in jobs[1:]:
        if n + size > cap:
            break
        c2 = [a + int(b) for a, b in zip(counts, cc[0])]
        e2 = est(c2)
        if now_ns + e2 > min(tight, int(dl)) * 1000 or (max_pass_ns >= 0 and e2 > max_pass_ns):
            break
        counts, n, tight, m = c2, n + int(size), min(tight, int(dl)), m + 1
    e_mem = est(counts)
    rest = jobs[m:]
    rest_counts = [0] * K
    for _, _, cc, _ in rest:
        rest_counts = [a + int(b) for a, b in zip(rest_counts, cc[0])]
    rest_fast = est(rest_counts) if rest else 0
    rest_dl = None
    for _, dl, _, _ in rest:
        if int(dl) * 1000 >= now_ns + e_mem + rest_fast:
            rest_dl = int(dl) if rest_dl is None else min(rest_dl, int(dl))

    def feasible(e):
        if now_ns + e > tight * 1000:
            return False
        if rest_dl is not None and now_ns + e + rest_fast > rest_dl * 1000:
            return False
        return max_pass_ns < 0 or e <= max_pass_ns

    choice = [0] * m
    moved = True
    while moved:
        moved = False
        for j in range(m):
            cc = jobs[j][2]
            cur = choice[j]
            base = [a - int(b) for a, b in zip(counts, cc[cur])]
            best = -1
            for c in range(cur + 1, len(cc)):
                if feasible(est([a + int(b) for a, b in zip(base, cc[c])])):
                    best = c
            if best > cur:
                choice[j] = best
                counts = [a + int(b) for a, b in zip(base, cc[best])]
                moved = True
    masks = []
    for j in range(m):
        masks.extend(int(x) for x in jobs[j][3][choice[j]])
    return m, choice, est(counts), counts, masks
