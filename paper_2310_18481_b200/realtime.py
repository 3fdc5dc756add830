"""Real-time serving on one GPU replica.

Same monitor/worker semantics as ``serving.run`` (reference sim.py:241-397:
EDF admission at the highest-accuracy candidate, policy passes after
``watermark`` arrivals or when the worker idles, dispatch-time drop rule,
per-part latency feedback) but driven by the wall clock: arrivals are
released at their real arrival times, the policy's host time is real, and
each dispatched job's modality-masked pass runs on the GPU with its
completion time read from CUDA events on the device clock.  This is how the
QPS-at-SLO benchmark is measured.

With ``host_io=True`` every job also copies its requests' clips for the
modalities it actually uses from pinned host memory into the resident pool
(H2D) and its logits back (D2H) inside the pass — the end-to-end path.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import device as dv
from .executor import request_masks
from .planner import StrategyMatrix
from .policy import (FeedbackState, Job, JobQueue, JobState, Policy, apply_policy,
                     candidates_with_rounding, next_dispatch, update_latency_feedback)
from .records import JobRecord, MetricsLog
from .registry import ModelProfile


@dataclass
class ServeStats:
    passes: int = 0
    requests: int = 0
    gpu_launches: int = 0
    busy_us: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    policy_host_us: float = 0.0
    policy_runs: int = 0
    dropped_policy: int = 0    # requests dropped by apply_policy (unsavable violators)
    dropped_dispatch: int = 0  # requests dropped by the dispatch-time rule
    dropped_admit: int = 0     # requests with an empty frontier at admission
    late: int = 0              # requests completed after their deadline
    wall_s: float = 0.0
    trace: list | None = None  # optional per-pass diagnostics (serve_realtime(trace=True))
    policy_launches: int = 0   # ms_pass_select launches (device policy step)
    policy_device_us: float = 0.0   # launch -> result on the selection stream (CUDA events)
    policy_kernel_us: float = 0.0   # the kernel's own time (device global timer)
    pass_flops: int = 0             # algorithmic FLOP of the completed passes (roofline numerator)
    refreshes: list | None = None   # matrix hot-swaps during the run (refresh.Refresh)
    formations: list | None = None


class HostClips:
    """Pinned host copies of the clip pool (for the end-to-end path)."""

    def __init__(self, model):
        self.host = [p.cpu().pin_memory() for p in model.pools]
        self.row_bytes = list(model.row_bytes)


def _serve_realtime(model, profile: ModelProfile, matrix: StrategyMatrix, templates,
                   policy: Policy = Policy.OPTIMIZED, watermark: int = 2,
                   host_clips: HostClips | None = None, slot_seed: int = 0,
                   window_us: int = 4_000_000, depth: int = 2, cost=None,
                   max_batch_requests: int | None = None, lead_us: int = 600, trace: bool = False,
                   sched_margin_us: int = 0, policy_grid_us: int = 1000, policy_at_dispatch: bool = False,
                   device_policy=None, selection: str = "policy", max_pass_us: float | None = None,
                   record_formations: bool = False, top_only: bool = False, refresher=None):
    """Serve ``templates`` (JobTemplates, arrival-sorted) in real time.

    ``depth`` jobs may be in flight on the GPU stream at once: the next job
    is dispatched (with dispatch time = the last in-flight job's estimated
    finish, exactly the reference's ``dispatch_time_us``) while the previous
    one still runs, so host scheduling overlaps device execution.  Jobs still
    execute one after another on the device, in EDF order.

    ``cost`` (a ``profiler.PassCostModel``) enables cross-job batching
    (the reference never batches across jobs):
    after the EDF head is popped, the following queued jobs (in EDF order,
    never skipping one) join the same masked device pass while the pass
    estimate keeps every member within its deadline and the batch within
    ``max_batch_requests``.  With batching, the next pass is formed just in
    time — once the in-flight pass is within ``lead_us`` of its estimated
    finish (or a full batch is already queued) — so batches grow with load
    instead of being cut at whatever was queued when the previous pass was
    launched.  Each job keeps its own assigned strategy; the
    pass's observed time feeds both the scheduler EWMA (attributed to jobs
    in proportion to their predicted latency) and the cost model's EWMA.

    ``sched_margin_us``: the scheduler (policy, dispatch drop rule, batch
    formation) sees every deadline this much earlier than the request's true
    deadline, so the reference policy predicts violations while a modality
    downgrade can still prevent them (a pass, once launched, cannot be
    changed); SLO attainment is always scored on the true deadline.
    ``policy_grid_us``: the optimized policy's knapsack quantum (reference
    1 ms; see ``policy.reassign_optimized``).  ``policy_at_dispatch``: run
    the policy once right before each pass is formed (instead of every
    ``watermark`` arrivals), so it always sees the queue the pass will take.
    ``device_policy``: a ``policy.DevicePolicy`` running the OPTIMIZED
    policy on the GPU (one launch per pass).

    ``selection="pass"`` (needs ``cost``; extension for the batched executor):
    the per-request modality-subset choice is made on the DEVICE when a pass
    is formed, against the measured cost of THAT pass: ``ms_pass_select``
    (``batcher.DevicePassSelector``; restated by oracle/selection.py
    pass_select) -- the north_star's policy step (P5's argmax accuracy under
    the request's remaining latency budget) with the budget
    coupled through the shared pass:
      1. membership: queued jobs join in EDF order at their FASTEST frontier
         candidate while the pass estimate meets every member's deadline;
      2. upgrades: each member (EDF order, repeatedly) moves to the most
         accurate candidate whose pass still meets every member's deadline
         AND lets the jobs left queued meet theirs in one following
         all-fastest pass.
    The kernel writes the pass's per-request masks into the device mask ring
    the compaction reads, and every modality's clips come from its pool ring
    (``ms_compact_ring``): no per-request host staging.  Idle GPU ->
    everyone at top accuracy; under load -> modalities dropped exactly as far
    as the deadlines require.  ``max_pass_us`` caps a pass's estimate in both
    steps (requests arriving during a pass wait for it and then for their
    own).  The reference policies (``policy``) are not run in this mode.
    ``record_formations``: keep every formation's inputs and outputs
    (``stats.formations``) for the oracle replay.  ``top_only``: every job
    keeps only its most accurate (all-modality) candidate -- the same batched
    server with selection switched off, the modality-agnostic baseline.
    ``refresher``: a ``refresh.ProfileRefresher``: served
    passes re-profile the cost model, a background thread rebuilds the
    serving profile and matrix, and the loop swaps them in between two
    formations (``stats.refreshes``).

    Returns (MetricsLog, ServeStats).  Job ids are 1-based stream order.
    """
    from collections import deque
    import torch
    rng = np.random.default_rng(slot_seed)
    queue = JobQueue()
    fb = FeedbackState()
    records: list[JobRecord] = []
    stats = ServeStats()
    if trace:
        stats.trace = []
    stream = torch.cuda.current_stream()
    ev_zero = dv.Event()
    pending = list(enumerate(templates, start=1))
    pos = 0
    inflight = deque()  # (job, start_event, end_event, predicted part latencies)
    since_opt = 0
    logits_host = torch.empty(model.max_req, model.head.logits.shape[1], dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream() if host_clips is not None else None
    rings = [0] * model.K  # host-IO path: per-modality pool rings (fresh rows per pass)
    pol_rng = np.random.default_rng([0, list(Policy).index(policy)])

    if selection == "pass" and model.pipelined:  # every stem / rest / head graph before the clock starts
        model.ensure_warm()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev_zero.record()

    def now_us() -> int:
        return int((time.perf_counter() - t0) * 1e6)

    def drop(job):
        records.append(JobRecord(job.id, job.arrival_us, job.size, job.accuracy_slo, None, None,
                                 True, True))

    def run_policy(now):
        nonlocal since_opt
        t = time.perf_counter()
        if device_policy is not None and policy is Policy.OPTIMIZED:
            dropped = device_policy.apply(queue, now, fb)
        else:
            dropped = apply_policy(policy, queue, now, fb, pol_rng, grid_us=policy_grid_us)
        for j in dropped:
            drop(j)
            stats.dropped_policy += j.size
        stats.policy_host_us += (time.perf_counter() - t) * 1e6
        stats.policy_runs += 1
        since_opt = 0

    cap = min(max_batch_requests or model.max_req, model.max_req)
    selector = fcache = None
    if refresher is not None:
        stats.refreshes = []
    FrontierCache = None
    if selection == "pass":
        if cost is None:
            raise ValueError("selection='pass' needs a PassCostModel (cost=)")
        from .batcher import DevicePassSelector, FrontierCache
        fcache = FrontierCache(matrix, model.K, top_only=top_only)
        selector = DevicePassSelector(model.K, cost.device_table(), cap,
                                      -1 if max_pass_us is None else int(round(max_pass_us * 1000)),
                                      model.mask_ring, record=record_formations)
    ring_i = 0

    def counts_of(masks):
        m = masks.astype(np.int64)
        return [int(((m >> k) & 1).sum()) for k in range(model.K)]

    def dispatch(now):
        queue.running = None  # next_dispatch plans one job at a time
        job, drops = next_dispatch(queue, now, fb)
        for j in drops:
            drop(j)
            stats.dropped_dispatch += j.size
        if job is None:
            queue.running = inflight[-1][0][-1] if inflight else None
            return False
        if selection == "pass" and cost is not None:
            return dispatch_pass_select(now, job)
        batch = [job]
        mlist = [request_masks(job.assigned.strategy.parts, job.size)]
        counts = counts_of(mlist[0])
        n = job.size
        est_us = None
        if cost is not None:
            est_us = cost.estimate_us(counts, n)
            tight = job.deadline_us
            for cand in list(queue._jobs):  # EDF order; stop at the first misfit
                if n + cand.size > cap:
                    break
                cm = request_masks(cand.assigned.strategy.parts, cand.size)
                c2 = [a + b for a, b in zip(counts, counts_of(cm))]
                e2 = cost.estimate_us(c2, n + cand.size)
                if now + e2 > min(tight, cand.deadline_us):
                    break
                queue.remove(cand)
                cand.state = JobState.RUNNING
                batch.append(cand)
                mlist.append(cm)
                counts, n, est_us = c2, n + cand.size, e2
                tight = min(tight, cand.deadline_us)
            for j in batch:
                j.est_finish_us = now + int(round(est_us))
        return launch(now, batch, mlist, counts, n, est_us)

    def dispatch_pass_select(now, head):
        """Form the pass on the device (ms_pass_select) and launch it."""
        nonlocal ring_i
        slot = ring_i % len(model.ring_ev)
        ring_i += 1
        t = time.perf_counter()
        r = selector.select([head] + queue._jobs, now, cost.factor, slot,
                            slot_free=model.ring_ev[slot] if model.ring_used[slot] else None)
        stats.policy_host_us += (time.perf_counter() - t) * 1e6
        stats.policy_runs += 1
        batch = [head] + queue.pop_front(r.members - 1)
        fin = now + (r.est_ns + 500) // 1000
        for j, c in zip(batch, r.choices):
            j.assigned_idx = int(c)
            j.state = JobState.RUNNING
            j.est_finish_us = fin
        q = len(batch) + len(queue)
        stats.h2d_bytes += 24 * q + 32  # the kernel reads the pinned job tables in place (mapped)
        stats.d2h_bytes += 4 * q + 4 * (2 + model.K) + 8
        return launch_ring(now, batch, r.counts, r.requests, r.est_ns / 1000.0, slot)

    def launch_ring(now, batch, counts, n, est_us, slot):
        """A device-formed pass: masks already in model.mask_ring[slot];
        modality k's clips are the next counts[k] rows of its pool ring (the
        host-IO path first DMAs exactly those rows from pinned memory)."""
        ns = model.n_slots
        bases = list(rings)
        ev_s, ev_e = dv.Event(), dv.Event()
        upload_ev = None
        if host_clips is not None:
            stats.h2d_bytes += model.ring_upload(host_clips.host, counts, bases, copy_stream)
            upload_ev = dv.Event()
            upload_ev.record(copy_stream)
            stream.wait_stream(copy_stream)
        for k in range(model.K):
            rings[k] = (bases[k] + counts[k]) % ns
        ev_s.record()
        model.run_ring(n, counts, slot, bases, upload_ev=upload_ev)
        if host_clips is not None:
            logits_host[:n].copy_(model.head.logits[:n], non_blocking=True)
            stats.d2h_bytes += n * model.head.logits.shape[1] * 4
        ev_e.record()
        stats.gpu_launches += model.launches_per_pass(tuple(counts)) + 1  # + ms_pass_select
        stats.passes += 1
        stats.requests += n
        preds = [[profile.part_latency_us(m, b) for m, b in j.assigned.strategy.parts] for j in batch]
        if stats.trace is not None:
            stats.trace.append({"pass": stats.passes - 1, "host_us": now_us(), "dispatch_us": now, "n": n,
                                "jobs": [j.id for j in batch], "est_us": est_us, "queue": len(queue),
                                "queued_req": sum(j.size for j in queue._jobs), "counts": list(counts),
                                "bases": bases})
        inflight.append((batch, ev_s, ev_e, preds, tuple(counts), n))
        queue.running = batch[-1]
        return True

    def launch(now, batch, mlist, counts, n, est_us):
        masks = np.concatenate(mlist)
        ev_s, ev_e = dv.Event(), dv.Event()
        if host_clips is not None:
            # H2D of the present modalities' clips on a copy stream (overlaps the
            # previous pass); the pass waits for it.  Each modality has its own
            # ring in the pinned host buffer and in the HBM pool: the pass's
            # requests that use modality k occupy consecutive rows of ring k,
            # so ONE DMA per modality (two on wrap-around) moves them, and the
            # compaction gather reads them through that modality's row map.
            ns = model.n_slots
            slots = np.zeros((model.K, n), dtype=np.int32)
            with torch.cuda.stream(copy_stream):
                for k in range(model.K):
                    present = np.flatnonzero((masks.astype(np.int64) >> k) & 1)
                    c = len(present)
                    if not c:
                        continue
                    r0 = rings[k]
                    slots[k, present] = (r0 + np.arange(c)) % ns
                    rings[k] = (r0 + c) % ns
                    first = min(c, ns - r0)
                    model.pools[k][r0:r0 + first].copy_(host_clips.host[k][r0:r0 + first], non_blocking=True)
                    if first < c:
                        model.pools[k][: c - first].copy_(host_clips.host[k][: c - first], non_blocking=True)
                    stats.h2d_bytes += c * host_clips.row_bytes[k]
            stream.wait_stream(copy_stream)
            stats.h2d_bytes += n * 2 + model.K * n * 4  # masks + per-modality row maps
        else:
            slots = rng.integers(0, model.n_slots, size=n)
        ev_s.record()
        logits = model.forward(slots, masks)
        if host_clips is not None:
            logits_host[:n].copy_(logits, non_blocking=True)
            stats.d2h_bytes += logits.numel() * 4
        ev_e.record()
        stats.gpu_launches += model.launches_per_pass(tuple(counts))
        stats.passes += 1
        stats.requests += n
        preds = [[profile.part_latency_us(m, b) for m, b in j.assigned.strategy.parts] for j in batch]
        if stats.trace is not None:
            stats.trace.append({"pass": stats.passes - 1, "host_us": now_us(), "dispatch_us": now, "n": n,
                                "jobs": [j.id for j in batch], "est_us": est_us, "queue": len(queue),
                                "queued_req": sum(j.size for j in queue._jobs), "counts": list(counts)})
        inflight.append((batch, ev_s, ev_e, preds, tuple(counts), n))
        queue.running = batch[-1]  # the latest in-flight job sets the next dispatch time
        return True

    def finish():
        """The oldest in-flight pass has completed on the device."""
        batch, ev_s, ev_e, preds, counts, n = inflight.popleft()
        end_us = int(round(ev_zero.elapsed_us(ev_e)))
        dur = max(1.0, ev_s.elapsed_us(ev_e))
        if stats.trace is not None:
            for tr in reversed(stats.trace):
                if tr["jobs"] and tr["jobs"][0] == batch[0].id:
                    tr.update(start_us=end_us - dur, end_us=end_us, seen_us=now_us())
                    break
        stats.busy_us += dur
        stats.pass_flops += model.flops_counts(counts, n)
        if refresher is not None:
            refresher.observe(counts, n, dur)
        if cost is not None:
            cost.observe(counts, n, dur)
        flat = [p for ps in preds for p in ps]
        tot = sum(flat)
        used = 0
        for i, p in enumerate(flat):  # per part, in execution order (sim.py:381)
            a = int(round(dur)) - used if i == len(flat) - 1 else max(1, int(round(dur * p / tot)))
            a = max(1, a)
            used += a
            update_latency_feedback(fb, p, a)
        for job in batch:
            job.state = JobState.COMPLETED
            job.completion_us = end_us
            if queue.running is job:
                queue.running = None
            true_dl = job.deadline_us + sched_margin_us
            records.append(JobRecord(job.id, job.arrival_us, job.size, job.accuracy_slo,
                                     job.assigned.effective_accuracy, end_us, False,
                                     end_us > true_dl))
            if end_us > true_dl:
                stats.late += job.size

    while pos < len(pending) or len(queue) or inflight:
        now = now_us()
        # arrivals due
        arrived = False
        while pos < len(pending) and pending[pos][1].arrival_us <= now:
            jid, tpl = pending[pos]
            pos += 1
            if selector is not None:
                cands, pack = fcache.lookup(tpl.size, tpl.accuracy_slo)
            else:
                cands, pack = candidates_with_rounding(matrix, tpl.size, tpl.accuracy_slo), None
            job = Job(jid, tpl.arrival_us, tpl.size, tpl.accuracy_slo, tpl.deadline_us - sched_margin_us, cands)
            job.pack = pack
            if not cands:
                job.state = JobState.DROPPED
                drop(job)
                stats.dropped_admit += job.size
                continue
            job.assigned_idx = len(cands) - 1
            queue.admit(job)
            since_opt += 1
            arrived = True
        while inflight and inflight[0][2].done():  # non-blocking completion checks
            finish()
        if refresher is not None and selector is not None:
            if len(inflight) >= depth or not len(queue):
                refresher.advance()  # host slack: the GPU queue is full (or nothing to form)
            res = refresher.poll()
            if res is not None:  # hot-swap between two formations
                cost, profile, matrix = res.cost, res.profile, res.matrix
                fcache = res.fcache
                selector.cost = cost.device_table()
                stats.refreshes.append(res)
            elif refresher.due(now / 1e6):
                refresher.start(now / 1e6)
        if policy is not Policy.NONE and since_opt > 0 and len(queue) and not policy_at_dispatch and \
                (since_opt >= watermark or not inflight):
            run_policy(now_us())
        while len(inflight) < depth and len(queue):
            t = now_us()
            if inflight and inflight[-1][0][-1].est_finish_us is not None:
                fin = inflight[-1][0][-1].est_finish_us
                if cost is not None and fin - t > lead_us and \
                        sum(j.size for j in queue._jobs) < cap:
                    break  # let the batch grow; dispatch closer to the GPU freeing up
                t = max(t, fin)
            if policy_at_dispatch and policy is not Policy.NONE and since_opt > 0:
                queue.running = inflight[-1][0][-1] if inflight else None
                run_policy(now_us())
                if not len(queue):
                    break
            if not dispatch(t):
                break
        if not inflight and not len(queue) and pos < len(pending):
            # idle until the next arrival
            wait = pending[pos][1].arrival_us - now_us()
            if wait > 200:
                time.sleep((wait - 100) / 1e6)
    torch.cuda.synchronize()
    stats.wall_s = time.perf_counter() - t0
    if refresher is not None:
        refresher.close()
    if selector is not None:
        stats.policy_launches = selector.launches
        stats.policy_device_us = selector.device_us
        stats.policy_kernel_us = selector.kernel_us
        if record_formations:
            stats.formations = selector.records
    log = MetricsLog(window_us, tuple(sorted(records, key=lambda r: r.id)))
    return log, stats


def serve_realtime(*args, **kwargs):
    """Real-time serving (``_serve_realtime``) with Python's cyclic garbage
    collector paused for the window: a full collection over the per-request
    objects of a 20k req/s stream stalls the host loop for milliseconds, which
    at a 15 ms deadline shows up as a ~1 % SLO-miss floor independent of the
    offered rate.  Refcounting still frees everything acyclic; one collection
    runs before and after."""
    import gc
    was = gc.isenabled()
    gc.collect()
    gc.disable()
    try:
        return _serve_realtime(*args, **kwargs)
    finally:
        if was:
            gc.enable()
        gc.collect()
