"""The drop-in boundary: the reference's public API, re-implemented host-side,
reproduces the reference byte-for-byte (matrices, frontiers, policies, whole
simulation logs) and its published golden scenarios."""

import json
from dataclasses import asdict
from pathlib import Path

import numpy as np
import pytest

import paper_2310_18481_b200 as ms
from paper_2310_18481_b200 import (FeedbackState, Job, JobQueue, JobState, JobTemplate, Policy,
                                   SimConfig, apply_policy, build_matrix, candidates_for_job,
                                   candidates_with_rounding, compute_budget, demo_profile,
                                   detect_violation, load_matrix, load_profile, next_dispatch,
                                   reassign_optimized, recommended_alphas, run, save_matrix,
                                   save_profile, solve_offline, try_upgrade)
from paper_2310_18481_b200.planner import Strategy, all_modalities_strategy, effective_accuracy
from paper_2310_18481_b200.planner import strategy_latency_ms

GOLDEN = Path(__file__).resolve().parent / "golden"
MS = 1000
A, V, AV = 1, 2, 3

# modserve/__init__.py:9-31
REFERENCE_API = """JobRecord MetricsLog Summary WindowStats accuracy_histogram export read_log summarize
window_stats ModalityCombo ModelProfile ProfileError SynthSpec count_strategies demo_profile
enumerate_combos load_profile save_profile scale_latency synth_profile FeedbackState Job JobQueue
JobState Policy ScheduleEstimate apply_policy build_schedule_estimate candidates_with_rounding
compute_budget detect_violation next_dispatch reassign_aggressive reassign_optimized
reassign_random try_upgrade update_latency_feedback JobTemplate SimConfig SimError WorkloadError
WorkloadSpec all_modalities_capacity_qps generate_jobs load_scenario load_trace map_trace_to_qps
matrix_for_jobs run Candidate MatrixCell MatrixError SolverError Strategy StrategyMatrix
all_modalities_strategy brute_force_offline build_matrix candidates_for_job default_alpha_grid
distinct_effective_accuracies effective_accuracy load_matrix recommended_alphas save_matrix
solve_offline strategy_latency_ms strategy_latency_us validate_matrix""".split()


def test_every_reference_name_is_exported():
    missing = [n for n in REFERENCE_API if not hasattr(ms, n)]
    assert not missing


@pytest.mark.parametrize("path", sorted((GOLDEN / "profiles").glob("*.yaml")), ids=lambda p: p.stem)
def test_matrix_documents_byte_identical(path, tmp_path):
    prof = load_profile(path)
    out = tmp_path / "m.json"
    save_matrix(build_matrix(prof, range(1, 9), recommended_alphas(prof)), out)
    assert out.read_text() == (GOLDEN / "matrices" / f"{path.stem}.json").read_text()
    # and the reference document loads + validates against our profile
    load_matrix(GOLDEN / "matrices" / f"{path.stem}.json", prof)
    save_profile(prof, tmp_path / "p.yaml")
    assert load_profile(tmp_path / "p.yaml") == prof


def test_frontier_lookups_match_reference():
    cases = json.loads((GOLDEN / "frontier_cases.json").read_text())
    mats = {}
    for c in cases:
        key = (c["profile"], tuple(c["sizes"]))
        if key not in mats:
            prof = load_profile(GOLDEN / "profiles" / f"{c['profile']}.yaml")
            mats[key] = build_matrix(prof, c["sizes"], recommended_alphas(prof))
        got = candidates_with_rounding(mats[key], c["size"], c["slo"])
        assert [{"parts": [list(p) for p in g.strategy.parts], "job_size": g.strategy.job_size,
                 "latency_us": g.latency_us, "effective_accuracy": g.effective_accuracy,
                 "credit": g.credit} for g in got] == c["candidates"]


def test_whole_simulations_match_reference_logs():
    runs = json.loads((GOLDEN / "sim_logs.json").read_text())
    profs = {"demo": demo_profile(),
             "synth_k3_b4_s0": ms.synth_profile(ms.SynthSpec(n_modalities=3, max_batch=4), 0)}
    for r in runs:
        p = profs[r["profile"]]
        jobs = [JobTemplate(**j) for j in r["jobs"]]
        log = run(SimConfig(profile=p, matrix=ms.matrix_for_jobs(p, jobs), policy=Policy(r["policy"]),
                            discrepancy=r["discrepancy"], seed=r["spec"]["seed"]), jobs)
        assert [asdict(x) for x in log.records] == r["records"], (r["profile"], r["policy"])


# ---------------------------------------------------------------- Appendix B goldens


@pytest.fixture(scope="module")
def demo_matrix():
    p = demo_profile()
    return build_matrix(p, [1, 2], recommended_alphas(p))


def make_job(m, jid, arrival_ms, size, slo, deadline_ms):
    c = candidates_for_job(m, size, slo)
    j = Job(jid, arrival_ms * MS, size, slo, deadline_ms * MS, c)
    j.assigned_idx = len(c) - 1
    return j


def test_effective_accuracy_and_latency_goldens():
    d = demo_profile()
    assert effective_accuracy(Strategy.make([(A, 1), (V, 1)]), d) == 0.685
    assert effective_accuracy(Strategy.make([(AV, 2)]), d) == 0.80
    assert effective_accuracy(Strategy.make([(A, 1), (AV, 1)]), d) == 0.735
    assert strategy_latency_ms(Strategy.make([(AV, 1), (A, 1)]), d) == 80.0
    assert all_modalities_strategy(d, 5).parts == ((AV, 1), (AV, 2), (AV, 2))


def test_solver_goldens():
    d = demo_profile()
    assert solve_offline(d, 2, 0.71).parts == ((A, 1), (AV, 1))
    assert solve_offline(d, 2, 0.0).parts == ((A, 2),)
    assert solve_offline(d, 2, 0.80).parts == ((AV, 2),)
    assert solve_offline(d, 2, 0.81) is None
    for size in range(1, 7):
        for alpha in (0.0, 0.6, 0.7, 0.72, 0.75, 0.8):
            assert ms.brute_force_offline(d, size, alpha) == solve_offline(d, size, alpha)


def test_frontier_goldens(demo_matrix):
    f = candidates_for_job(demo_matrix, 2, 0.71)
    assert [(c.latency_ms, c.effective_accuracy) for c in f] == [(80.0, 0.735), (90.0, 0.75), (120.0, 0.8)]
    assert (candidates_for_job(demo_matrix, 2, 0.65)[0].latency_ms,
            candidates_for_job(demo_matrix, 2, 0.65)[0].effective_accuracy) == (40.0, 0.67)
    assert candidates_for_job(demo_matrix, 2, 0.85) == []


def test_rescue_scenario_goldens(demo_matrix):
    q = JobQueue()
    j2 = make_job(demo_matrix, 2, 10, 2, 0.71, 140)
    j3 = make_job(demo_matrix, 3, 20, 2, 0.65, 150)
    q.admit(j2)
    q.admit(j3)
    fb = FeedbackState()
    assert detect_violation(q, 20 * MS, fb) is j3
    budget, scope = compute_budget(q, j3, 20 * MS)
    assert budget == 130 * MS and scope == [j2, j3]
    sel = reassign_optimized(scope, budget, 20 * MS, fb)
    j2.assigned_idx, j3.assigned_idx = sel
    assert (j2.assigned.latency_ms, j2.assigned.effective_accuracy) == (80.0, 0.735)
    assert (j3.assigned.latency_ms, j3.assigned.effective_accuracy) == (50.0, 0.685)
    assert j2.assigned.credit + j3.assigned.credit == 28_400


def test_cascading_violators_and_upgrade_goldens(demo_matrix):
    q = JobQueue()
    jobs = [make_job(demo_matrix, 1, 0, 2, 0.65, 130), make_job(demo_matrix, 2, 0, 2, 0.71, 260),
            make_job(demo_matrix, 3, 0, 2, 0.65, 300)]
    for j in jobs:
        q.admit(j)
    assert apply_policy(Policy.OPTIMIZED, q, 0, FeedbackState()) == []
    assert {j.id: (j.assigned.latency_ms, j.assigned.effective_accuracy) for j in jobs} == \
        {1: (120.0, 0.8), 2: (90.0, 0.75), 3: (90.0, 0.75)}
    q = JobQueue()
    a, b = make_job(demo_matrix, 1, 0, 2, 0.71, 90), make_job(demo_matrix, 2, 0, 2, 0.65, 130)
    a.assigned_idx = b.assigned_idx = 0
    q.admit(a)
    q.admit(b)
    try_upgrade(q, 0, FeedbackState())
    assert (a.assigned.latency_ms, b.assigned.latency_ms) == (90.0, 40.0)


def test_dispatch_drop_golden(demo_matrix):
    q = JobQueue()
    j = make_job(demo_matrix, 1, 0, 2, 0.65, 130)
    q.admit(j)
    job, drops = next_dispatch(q, 50 * MS, FeedbackState(factor=2.5))
    assert job is None and drops == [j] and j.state is JobState.DROPPED


def test_sim_golden_timeline():
    p = demo_profile()
    m = build_matrix(p, [1, 2], recommended_alphas(p))
    jobs = [JobTemplate(0, 1, 0.67, 20 * MS), JobTemplate(10 * MS, 2, 0.71, 140 * MS),
            JobTemplate(20 * MS, 2, 0.65, 150 * MS)]
    cfg = SimConfig(profile=p, matrix=m, policy=Policy.OPTIMIZED, optimizer_overhead_ms=0.0, seed=1)
    by = {r.id: r for r in run(cfg, jobs).records}
    assert (by[1].completion_us, by[2].completion_us, by[3].completion_us) == (20 * MS, 100 * MS, 150 * MS)
    assert (by[1].achieved_accuracy, by[2].achieved_accuracy, by[3].achieved_accuracy) == (0.67, 0.735, 0.685)
    none = SimConfig(profile=p, matrix=m, policy=Policy.NONE, optimizer_overhead_ms=0.0, seed=1)
    assert {r.id: r for r in run(none, jobs).records}[3].violated


def test_poisson_workload_and_percentiles():
    p = demo_profile()
    spec = ms.WorkloadSpec(kind="poisson", qps=200, duration_s=5, seed=3, deadline_ms=300)
    jobs = ms.generate_jobs(spec, p)
    assert jobs == ms.generate_jobs(spec, p)
    assert abs(sum(j.size for j in jobs) / 5 - 200) < 40
    assert all(j.deadline_us - j.arrival_us == 300 * MS for j in jobs)
    log = run(SimConfig(profile=p, matrix=ms.matrix_for_jobs(p, jobs), policy=Policy.AGGRESSIVE), jobs)
    pct = log.jct_percentiles_us((50, 99))
    assert pct[50] <= pct[99]


def test_run_replicas_round_robin_ids():
    p = demo_profile()
    spec = ms.WorkloadSpec(kind="constant", qps=30, duration_s=4, seed=2)
    jobs = ms.generate_jobs(spec, p)
    m = ms.matrix_for_jobs(p, jobs)
    cfgs = [SimConfig(profile=p, matrix=m, policy=Policy.OPTIMIZED, seed=1) for _ in range(3)]
    merged = ms.run_replicas(cfgs, jobs)
    assert [r.id for r in merged.records] == list(range(1, len(jobs) + 1))
    assert [(r.arrival_us, r.size) for r in merged.records] == [(j.arrival_us, j.size) for j in jobs]
    one = run(cfgs[0], jobs[1::3])
    assert [r.completion_us for r in one.records] == [r.completion_us for r in merged.records[1::3]]


def test_request_masks_follow_canonical_parts():
    from oracle.selection import parts_for_requests
    from paper_2310_18481_b200.executor import request_masks
    rng = np.random.default_rng(1)
    for _ in range(200):
        parts = sorted((int(rng.integers(1, 8)), int(rng.integers(1, 5))) for _ in range(rng.integers(1, 5)))
        total = sum(b for _, b in parts)
        size = int(rng.integers(1, total + 1))
        assert request_masks(parts, size).tolist() == parts_for_requests(parts, size)[0].tolist()


def test_coupled_queue_policy_matches_reference_goldens():
    """Host mirror of apply_policy(OPTIMIZED) on 440 multi-job EDF queues
    (2-40 jobs, drops, MCKP reassignments, upgrades) generated by the real
    reference (tests/golden/make_queue_golden.py)."""
    from queue_cases import build_queue, load_cases, outcome
    from paper_2310_18481_b200.policy import Policy, apply_policy
    cases = load_cases()
    assert len(cases) >= 400
    for case in cases:
        q, jobs, fb = build_queue(case)
        dropped = apply_policy(Policy.OPTIMIZED, q, case["now_us"], fb)
        assert outcome(jobs, dropped) == case["expected"], case["profile"]
