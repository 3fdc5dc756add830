"""Generate golden fixtures by running the REAL reference (modserve).

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It imports ``modserve`` read-only from /root/reference/pkg/src and writes
small JSON fixtures next to this script.  The fixtures pin:

* ``policy_cases.json``  — one-job ``apply_policy(OPTIMIZED)`` outcomes
  (scheduler.py:382-425) on frontiers from real matrices, with budgets near
  candidate boundaries, latency factors 0.5-2.5 and running jobs; the device
  policy kernel must reproduce every choice.
* ``frontier_cases.json`` — ``candidates_with_rounding`` (scheduler.py:138)
  outputs, including rounded-up sizes.
* ``matrices/*.json`` + ``profiles/*.yaml`` — reference ``build_matrix`` /
  ``save_matrix`` (strategy.py:441, :573) documents for synthetic profiles.
* ``sim_logs.json`` — reference ``run()`` (sim.py:400) per-job records for
  small workloads under all four policies.
* ``grouping_cases.json`` — assigned strategies' parts for real jobs, used
  by the request->part grouping tests.
"""

from __future__ import annotations

import json
import sys
from dataclasses import asdict
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from modserve import (  # noqa: E402
    FeedbackState, Job, JobQueue, JobState, Policy, SimConfig, SynthSpec,
    WorkloadSpec, apply_policy, build_matrix, candidates_with_rounding,
    demo_profile, generate_jobs, matrix_for_jobs, recommended_alphas, run,
    save_matrix, save_profile, synth_profile,
)

HERE = Path(__file__).resolve().parent
MS = 1000


def _profiles():
    out = [("demo", demo_profile())]
    for n_mod, max_batch, seed in [(2, 3, 1), (3, 4, 0), (3, 4, 5), (4, 3, 2), (3, 2, 7)]:
        p = synth_profile(SynthSpec(n_modalities=n_mod, max_batch=max_batch), seed)
        out.append((f"synth_k{n_mod}_b{max_batch}_s{seed}", p))
    return out


def policy_cases(rng):
    cases = []
    factors = [0.5, 0.93, 1.0, 1.2, 2.5]
    for pname, p in _profiles():
        m = build_matrix(p, range(1, 7), recommended_alphas(p))
        for _ in range(420):
            size = int(rng.integers(1, 7))
            slo = round(float(rng.uniform(p.min_accuracy, p.max_accuracy)), 4)
            cands = candidates_with_rounding(m, size, slo)
            if not cands:
                continue
            factor = float(factors[int(rng.integers(len(factors)))]) if rng.random() < 0.7 \
                else float(rng.uniform(0.4, 2.6))
            fb = FeedbackState(factor=factor)
            now = int(rng.integers(0, 5_000)) * MS + int(rng.integers(0, 1000))
            running_finish = None
            if rng.random() < 0.4:
                running_finish = now + int(rng.integers(-50_000, 200_000))
            dispatch = max(now, running_finish) if running_finish is not None else now
            mode = rng.random()
            if mode < 0.5:
                # within +-1.5 ms of a random candidate's estimate
                c = cands[int(rng.integers(len(cands)))]
                budget = fb.estimate_us(c.latency_us) + int(rng.integers(-1500, 1501))
            elif mode < 0.8:
                budget = int(rng.integers(-20_000, 1 + 2 * fb.estimate_us(cands[-1].latency_us)))
            else:
                budget = fb.estimate_us(cands[int(rng.integers(len(cands)))].latency_us) \
                    + int(rng.integers(-3, 4)) * MS
            deadline = dispatch + budget
            arrival = min(now, deadline) - 1
            job = Job(id=1, arrival_us=arrival, size=size, accuracy_slo=slo,
                      deadline_us=deadline, candidates=list(cands))
            job.assigned_idx = len(cands) - 1
            q = JobQueue()
            q.admit(job)
            if running_finish is not None:
                run_job = Job(id=99, arrival_us=0, size=1, accuracy_slo=slo,
                              deadline_us=10**12, candidates=list(cands))
                run_job.state = JobState.RUNNING
                run_job.est_finish_us = running_finish
                q.running = run_job
            drops = apply_policy(Policy.OPTIMIZED, q, now, fb)
            choice = -1 if drops else job.assigned_idx
            cases.append({
                "profile": pname,
                "lat_us": [c.latency_us for c in cands],
                "credit": [c.credit for c in cands],
                "deadline_us": deadline,
                "now_us": now,
                "running_finish_us": running_finish,
                "dispatch_us": dispatch,
                "factor": factor,
                "expected": choice,
            })
    return cases


def _cand_doc(c):
    return {"parts": [list(pt) for pt in c.strategy.parts], "job_size": c.strategy.job_size,
            "latency_us": c.latency_us, "effective_accuracy": c.effective_accuracy,
            "credit": c.credit}


def frontier_cases(rng):
    cases = []
    for pname, p in _profiles():
        for sizes in ([1, 2, 3, 4], [1, 2, 4, 6]):
            m = build_matrix(p, sizes, recommended_alphas(p))
            for _ in range(25):
                size = int(rng.integers(1, 8))
                slo = round(float(rng.uniform(p.min_accuracy - 0.05, p.max_accuracy + 0.02)), 4)
                cands = candidates_with_rounding(m, size, slo)
                cases.append({"profile": pname, "sizes": sizes, "size": size, "slo": slo,
                              "candidates": [_cand_doc(c) for c in cands]})
    return cases


def write_profiles_and_matrices():
    (HERE / "profiles").mkdir(exist_ok=True)
    (HERE / "matrices").mkdir(exist_ok=True)
    for pname, p in _profiles():
        save_profile(p, HERE / "profiles" / f"{pname}.yaml")
        m = build_matrix(p, range(1, 9), recommended_alphas(p))
        save_matrix(m, HERE / "matrices" / f"{pname}.json")


def sim_logs():
    runs = []
    specs = [
        ("demo", demo_profile(), WorkloadSpec(kind="constant", qps=33, duration_s=12, seed=1), 1.0),
        ("demo", demo_profile(), WorkloadSpec(kind="constant", qps=20, duration_s=10, seed=4), 1.4),
        ("synth_k3_b4_s0", synth_profile(SynthSpec(n_modalities=3, max_batch=4), 0),
         WorkloadSpec(kind="constant", qps=40, duration_s=10, seed=2, deadline_ms=400.0), 1.0),
        ("synth_k3_b4_s0", synth_profile(SynthSpec(n_modalities=3, max_batch=4), 0),
         WorkloadSpec(kind="constant", qps=60, duration_s=8, seed=3, deadline_ms=300.0), 0.8),
    ]
    for pname, p, spec, d in specs:
        jobs = generate_jobs(spec, p)
        m = matrix_for_jobs(p, jobs)
        for policy in Policy:
            cfg = SimConfig(profile=p, matrix=m, policy=policy, discrepancy=d, seed=spec.seed)
            log = run(cfg, jobs)
            runs.append({
                "profile": pname,
                "spec": {k: v for k, v in asdict(spec).items()},
                "discrepancy": d,
                "policy": policy.value,
                "jobs": [asdict(j) for j in jobs],
                "records": [asdict(r) for r in log.records],
                "violation_ratio": log.violation_ratio(),
            })
    return runs


def main():
    rng = np.random.default_rng(20231018)
    write_profiles_and_matrices()
    pc = policy_cases(rng)
    (HERE / "policy_cases.json").write_text(json.dumps(pc))
    fc = frontier_cases(rng)
    (HERE / "frontier_cases.json").write_text(json.dumps(fc))
    sl = sim_logs()
    (HERE / "sim_logs.json").write_text(json.dumps(sl))
    n_drop = sum(1 for c in pc if c["expected"] == -1)
    print(f"policy cases {len(pc)} ({n_drop} drops); frontier cases {len(fc)}; sim runs {len(sl)}")


if __name__ == "__main__":
    main()
