"""Rebuild the reference-generated coupled-policy cases
(tests/golden/queue_policy_cases.json, make_queue_golden.py) as host-mirror
JobQueues: jobs in EDF order with the reference frontiers (latency, credit,
effective accuracy), the running job's estimated finish and the factor."""

import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "queue_policy_cases.json"


def load_cases():
    return json.loads(GOLDEN.read_text())


def build_queue(case):
    from paper_2310_18481_b200.planner import Candidate
    from paper_2310_18481_b200.policy import FeedbackState, Job, JobQueue, JobState
    q = JobQueue()
    jobs = []
    for jd in case["jobs"]:
        cands = [Candidate(None, lat, acc, cr) for lat, acc, cr in zip(jd["lat_us"], jd["acc"], jd["credit"])]
        j = Job(jd["id"], min(case["now_us"], jd["deadline_us"]) - 1, 1, 0.0, jd["deadline_us"], cands)
        j.assigned_idx = jd["assigned"]
        q.admit(j)
        jobs.append(j)
    if case["running_finish_us"] is not None:
        r = Job(999, 0, 1, 0.0, 10**12, list(jobs[0].candidates))
        r.state = JobState.RUNNING
        r.est_finish_us = case["running_finish_us"]
        q.running = r
    assert [j.id for j in q.jobs()] == [jd["id"] for jd in case["jobs"]]  # EDF order preserved
    return q, jobs, FeedbackState(factor=case["factor"])


def outcome(jobs, dropped):
    ids = {j.id for j in dropped}
    return [-1 if j.id in ids else j.assigned_idx for j in jobs]
