"""Where the refresh-loop test's late requests come from: 4 s at 12k req/s
with the pass cost model 25 % optimistic, late requests per 250 ms window
(by arrival), refresh swap times, and the same run without the refresher /
without skew.

    python tools/refresh_diag.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_18481_b200 as ms  # noqa: E402
from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402
from paper_2310_18481_b200.policy import Policy  # noqa: E402
from paper_2310_18481_b200.profiler import TBN_ACCURACY, PassCostModel, marginal_profile, profile_pass_costs  # noqa: E402
from paper_2310_18481_b200.realtime import serve_realtime  # noqa: E402
from paper_2310_18481_b200.refresh import ProfileRefresher  # noqa: E402

model = build_tbn_model(max_req=96, n_slots=192)
true = profile_pass_costs(model, reps=2)
mods = ("rgb", "flow", "audio")
for name, scale, use_ref in (("skew+refresh", 0.75, True), ("skew only", 0.75, False), ("true+refresh", 1.0, True),
                             ("true only", 1.0, False), ("skew+refresh", 0.75, True)):
    cost = PassCostModel(true.enc_us, true.head_us, true.compact_us,
                         pass_all_us=[(n, scale * t) for n, t in true.pass_all])
    prof = marginal_profile(cost, mods, TBN_ACCURACY, max_batch=8)
    matrix = ms.build_matrix(prof, range(1, 25), ms.recommended_alphas(prof))
    ref = ProfileRefresher(cost, mods, TBN_ACCURACY, 8, range(1, 25), matrix.alphas, period_s=0.5) if use_ref else None
    spec = ms.WorkloadSpec(kind="poisson", qps=12000, duration_s=4, deadline_ms=15, seed=9)
    jobs = [ms.JobTemplate(j.arrival_us, min(j.size, 24), j.accuracy_slo, j.deadline_us)
            for j in ms.generate_jobs(spec, prof)]
    log, st = serve_realtime(model, prof, matrix, jobs, cost=cost, policy=Policy.NONE, selection="pass",
                             max_pass_us=3000, refresher=ref)
    late = np.zeros(16)
    tot = np.zeros(16)
    for r in log.records:
        b = min(15, r.arrival_us // 250_000)
        tot[b] += r.size
        if r.dropped or r.violated:
            late[b] += r.size
    print(f"{name}: violation {log.violation_ratio():.4f} passes {st.passes} factor_end {cost.factor:.3f}")
    print("   late per 250ms:", late.astype(int).tolist())
    if use_ref:
        for r in st.refreshes:
            print(f"   swap at {r.at_s:.2f}s build {r.build_s:.2f}s knots {[round(t) for _, t in r.knots_before][:4]} -> "
                  f"{[round(t) for _, t in r.knots_after][:4]}")
