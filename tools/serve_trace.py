"""Real-time serving near the SLO limit with per-pass diagnostics: where do
late requests come from?  Writes gpurun_out/serve_trace.json.

    python tools/serve_trace.py --rate 8000 --seconds 4
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--rate", type=float, default=8000)
ap.add_argument("--seconds", type=float, default=4)
ap.add_argument("--deadline-ms", type=float, default=15)
ap.add_argument("--profile", default="marginal")
ap.add_argument("--margin-ms", type=float, default=3.0)
ap.add_argument("--grid-us", type=int, default=20)
ap.add_argument("--policy", default="optimized")
ap.add_argument("--at-dispatch", type=int, default=1)
ap.add_argument("--device-policy", type=int, default=0)
ap.add_argument("--selection", default="policy")
ap.add_argument("--pass-frac", type=float, default=0.0)
a = ap.parse_args()
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402
from paper_2310_18481_b200.planner import build_matrix, recommended_alphas  # noqa: E402
from paper_2310_18481_b200.profiler import (TBN_ACCURACY, marginal_profile, profile_model,  # noqa: E402
                                            profile_pass_costs)
from paper_2310_18481_b200.realtime import serve_realtime  # noqa: E402
from paper_2310_18481_b200.policy import DevicePolicy, Policy  # noqa: E402

names = ("rgb", "flow", "audio")
model = build_tbn_model(max_req=96, n_slots=192)
model.warm_graphs()
prof = profile_model(model, names, TBN_ACCURACY, max_batch=8, reps=3)
cost = profile_pass_costs(model, reps=3)
sprof = marginal_profile(cost, names, TBN_ACCURACY, 8) if a.profile == "marginal" else prof
matrix = build_matrix(sprof, range(1, 25), recommended_alphas(sprof))
jobs = bench.make_jobs(sprof, a.rate, a.seconds, a.deadline_ms, 7)
from paper_2310_18481_b200.serving import JobTemplate  # noqa: E402
jobs = [JobTemplate(j.arrival_us, min(j.size, 24), j.accuracy_slo, j.deadline_us) for j in jobs]
cost.factor = 1.0
log, st = serve_realtime(model, sprof, matrix, jobs, cost=cost, trace=True, sched_margin_us=int(a.margin_ms * 1000),
                         policy_grid_us=a.grid_us, policy=Policy(a.policy), policy_at_dispatch=bool(a.at_dispatch),
                         device_policy=DevicePolicy(max_jobs=1024, max_cand=64, grid_us=a.grid_us) if a.device_policy
                         else None, selection=a.selection,
                         max_pass_us=a.pass_frac * a.deadline_ms * 1000 if a.pass_frac else None)
late = [r for r in log.records if r.violated]
served = [r for r in log.records if not r.dropped]
fa = sprof.combo_accuracy(sprof.all_modalities_mask)
print(f"selection={a.selection} pass_frac={a.pass_frac} {a.policy} at_dispatch={a.at_dispatch} dev={a.device_policy} grid {a.grid_us} us margin {a.margin_ms} ms: downgraded share {sum(r.size for r in served if r.achieved_accuracy < fa) / max(1, sum(r.size for r in served)):.3f}")
print(f"rate {a.rate}: violation {log.violation_ratio():.4f} passes {st.passes} req/pass {st.requests / st.passes:.1f} "
      f"late {st.late} drops {st.dropped_policy}/{st.dropped_dispatch}/{st.dropped_admit} "
      f"policy {st.policy_host_us / max(1, st.policy_runs):.0f}us x{st.policy_runs} wall {st.wall_s:.2f}s")
job_pass = {}
for tr in st.trace:
    for j in tr["jobs"]:
        job_pass[j] = tr
rec = {r.id: r for r in log.records}
gaps = []
for a_, b_ in zip(st.trace, st.trace[1:]):
    if "end_us" in a_ and "start_us" in b_:
        gaps.append(b_["start_us"] - a_["end_us"])
print("device gap between passes (us): p50 %.0f p99 %.0f max %.0f" % tuple(np.percentile(gaps, [50, 99, 100])))
durs = [t["end_us"] - t["start_us"] for t in st.trace if "end_us" in t]
print("pass us: p50 %.0f p99 %.0f max %.0f" % tuple(np.percentile(durs, [50, 99, 100])))
lags = [t["host_us"] - t["dispatch_us"] for t in st.trace]
print("host dispatch lag (us): p50 %.0f p99 %.0f max %.0f" % tuple(np.percentile(lags, [50, 99, 100])))
seen = [t["seen_us"] - t["end_us"] for t in st.trace if "seen_us" in t]
print("completion noticed after (us): p50 %.0f p99 %.0f max %.0f" % tuple(np.percentile(seen, [50, 99, 100])))
out = []
for r in late[:40]:
    tr = job_pass.get(r.id)
    out.append({"id": r.id, "arr": r.arrival_us, "size": r.size, "done": r.completion_us, "dropped": r.dropped,
                "pass": tr})
    if tr and "end_us" in tr:
        print(f"late job {r.id} size {r.size} arr {r.arrival_us / 1e3:.1f}ms dispatch {tr['dispatch_us'] / 1e3:.1f} "
              f"host {tr['host_us'] / 1e3:.1f} start {tr['start_us'] / 1e3:.1f} end {tr['end_us'] / 1e3:.1f} "
              f"n {tr['n']} est {tr['est_us']} queue {tr['queue']}/{tr['queued_req']}")
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/serve_trace.json").write_text(json.dumps({"trace": st.trace, "late": out}))

# mask composition of the served passes (for profiling a representative pass)
comp = [t["counts"] for t in st.trace if "counts" in t]
if comp:
    c = np.array(comp)
    print("per-pass modality counts (rgb, flow, audio): mean", np.round(c.mean(0), 1).tolist(),
          "p50 n", float(np.median([t["n"] for t in st.trace])))
