"""Coupled OPTIMIZED policy: host mirror (numpy MCKP) vs one device launch
(ms_policy_apply), on the reference-generated EDF queues, by queue length."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from queue_cases import build_queue, load_cases  # noqa: E402

from paper_2310_18481_b200.policy import DevicePolicy, Policy, apply_policy  # noqa: E402

cases = load_cases()
for grid in (1000, 20):
    pol = DevicePolicy(grid_us=grid)
    rows = {}
    for case in cases:
        n = len(case["jobs"])
        b = "2-10" if n <= 10 else "11-25" if n <= 25 else "26-40"
        q1, _, fb1 = build_queue(case)
        q2, _, fb2 = build_queue(case)
        t0 = time.perf_counter()
        apply_policy(Policy.OPTIMIZED, q1, case["now_us"], fb1, grid_us=grid)
        t1 = time.perf_counter()
        pol.apply(q2, case["now_us"], fb2)
        t2 = time.perf_counter()
        rows.setdefault(b, []).append(((t1 - t0) * 1e6, (t2 - t1) * 1e6))
    for b, v in rows.items():
        v = np.array(v)
        print(f"grid {grid:4d} us, {b:5s} jobs ({len(v):3d} queues): host median {np.median(v[:, 0]):8.0f} us "
              f"p90 {np.percentile(v[:, 0], 90):8.0f} | device median {np.median(v[:, 1]):6.0f} us "
              f"p90 {np.percentile(v[:, 1], 90):6.0f}")

# the batched TBN server's regime: marginal-cost frontiers (100s of us),
# 15 ms deadlines, 20 us knapsack quantum
from paper_2310_18481_b200.planner import build_matrix, recommended_alphas  # noqa: E402
from paper_2310_18481_b200.policy import FeedbackState, Job, JobQueue, candidates_with_rounding  # noqa: E402
from paper_2310_18481_b200.profiler import TBN_ACCURACY, PassCostModel, marginal_profile  # noqa: E402

enc = [[400 + 55 * n for n in range(96)], [410 + 62 * n for n in range(96)], [420 + 68 * n for n in range(96)]]
pa = [(1, 577), (4, 881), (8, 1358), (16, 2203), (24, 2848), (32, 3642), (48, 5046), (96, 9183)]
prof = marginal_profile(PassCostModel(enc, [30.0] * 96, 15, pass_all_us=pa), ("rgb", "flow", "audio"),
                        TBN_ACCURACY, 8)
mat = build_matrix(prof, range(1, 25), recommended_alphas(prof))
rng = np.random.default_rng(0)
pol = DevicePolicy(grid_us=20)
for n_jobs in (8, 32, 64, 128):
    th, td = [], []
    for rep in range(20):
        def mk():
            q = JobQueue()
            r2 = np.random.default_rng(rep * 1000 + n_jobs)
            for i in range(n_jobs):
                size = int(min(24, max(1, round(r2.normal(1, 6)))))
                slo = round(float(r2.uniform(prof.min_accuracy, prof.max_accuracy)), 4)
                cands = candidates_with_rounding(mat, size, slo)
                dl = 100_000 + int(r2.uniform(1_000, 15_000))
                j = Job(i + 1, 99_000, size, slo, dl, cands)
                j.assigned_idx = len(cands) - 1
                q.admit(j)
            return q
        q1, q2 = mk(), mk()
        t0 = time.perf_counter()
        d1 = apply_policy(Policy.OPTIMIZED, q1, 100_000, FeedbackState(1.0), grid_us=20)
        t1 = time.perf_counter()
        d2 = pol.apply(q2, 100_000, FeedbackState(1.0))
        t2 = time.perf_counter()
        assert [j.assigned_idx for j in q1.jobs()] == [j.assigned_idx for j in q2.jobs()]
        assert sorted(j.id for j in d1) == sorted(j.id for j in d2)
        th.append((t1 - t0) * 1e6)
        td.append((t2 - t1) * 1e6)
    print(f"TBN serving regime, {n_jobs:3d} queued jobs: host median {np.median(th):8.0f} us | "
          f"device median {np.median(td):6.0f} us (bit-identical)")
