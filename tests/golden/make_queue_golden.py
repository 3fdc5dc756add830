"""Golden fixtures for the COUPLED queue policy (multi-job EDF scopes), by
running the REAL reference (modserve) read-only from /root/reference:

    python tests/golden/make_queue_golden.py      # build container only

``queue_policy_cases.json``: random EDF queues of 2-40 jobs with frontiers
from real matrices, tight/loose deadlines, running jobs and latency factors;
each case records the reference ``apply_policy(OPTIMIZED)``
(scheduler.py:382-425: detect_violation -> compute_budget ->
reassign_optimized MCKP on the 1 ms grid -> drops -> try_upgrade) outcome:
every job's final candidate index, -1 when dropped.  The device coupled
policy kernel (ms_policy_apply) must reproduce all of them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from modserve import (  # noqa: E402
    FeedbackState, Job, JobQueue, JobState, Policy, SynthSpec, apply_policy, build_matrix,
    candidates_with_rounding, demo_profile, recommended_alphas, synth_profile,
)

HERE = Path(__file__).resolve().parent
MS = 1000


def main():
    rng = np.random.default_rng(20231019)
    profiles = [("demo", demo_profile())]
    for n_mod, max_batch, seed in [(2, 3, 1), (3, 4, 0), (4, 3, 2)]:
        profiles.append((f"synth_k{n_mod}_b{max_batch}_s{seed}",
                         synth_profile(SynthSpec(n_modalities=n_mod, max_batch=max_batch), seed)))
    cases = []
    for pname, p in profiles:
        m = build_matrix(p, range(1, 7), recommended_alphas(p))
        for _ in range(110):
            n_jobs = int(rng.integers(2, 41))
            factor = float(rng.choice([0.5, 0.93, 1.0, 1.2, 2.5])) if rng.random() < 0.6 \
                else float(rng.uniform(0.4, 2.6))
            fb = FeedbackState(factor=factor)
            now = int(rng.integers(0, 5_000)) * MS + int(rng.integers(0, 1000))
            q = JobQueue()
            jobs = []
            # deadline pressure: tight queues force downgrades, drops and upgrades
            slack = float(rng.uniform(0.15, 1.3))
            t = now
            for i in range(n_jobs):
                size = int(rng.integers(1, 7))
                slo = round(float(rng.uniform(p.min_accuracy, p.max_accuracy)), 4)
                cands = candidates_with_rounding(m, size, slo)
                if not cands:
                    continue
                t += int(fb.estimate_us(cands[-1].latency_us) * slack) + int(rng.integers(0, 2000))
                deadline = t + int(rng.integers(-5_000, 5_000))
                job = Job(id=i + 1, arrival_us=min(now, deadline) - 1, size=size, accuracy_slo=slo,
                          deadline_us=deadline, candidates=list(cands))
                job.assigned_idx = len(cands) - 1 if rng.random() < 0.8 else int(rng.integers(len(cands)))
                q.admit(job)
                jobs.append(job)
            running_finish = None
            if rng.random() < 0.5:
                running_finish = now + int(rng.integers(-20_000, 80_000))
                run_job = Job(id=999, arrival_us=0, size=1, accuracy_slo=0.0, deadline_us=10**12,
                              candidates=list(jobs[0].candidates))
                run_job.state = JobState.RUNNING
                run_job.est_finish_us = running_finish
                q.running = run_job
            order = [j.id for j in q.jobs()]  # EDF order
            init = {j.id: j.assigned_idx for j in jobs}
            dropped = {j.id for j in apply_policy(Policy.OPTIMIZED, q, now, fb)}
            by_id = {j.id: j for j in jobs}
            cases.append({
                "profile": pname, "now_us": now, "running_finish_us": running_finish, "factor": factor,
                "jobs": [{"id": jid, "deadline_us": by_id[jid].deadline_us, "assigned": init[jid],
                          "lat_us": [c.latency_us for c in by_id[jid].candidates],
                          "credit": [c.credit for c in by_id[jid].candidates],
                          "acc": [c.effective_accuracy for c in by_id[jid].candidates]}
                         for jid in order],
                "expected": [-1 if jid in dropped else by_id[jid].assigned_idx for jid in order],
            })
    (HERE / "queue_policy_cases.json").write_text(json.dumps(cases))
    n_drop = sum(sum(1 for e in c["expected"] if e < 0) for c in cases)
    n_changed = sum(sum(1 for j, e in zip(c["jobs"], c["expected"]) if e >= 0 and e != j["assigned"])
                    for c in cases)
    print(f"{len(cases)} queues, {sum(len(c['jobs']) for c in cases)} jobs, {n_drop} dropped, "
          f"{n_changed} reassigned")


if __name__ == "__main__":
    main()
