"""Golden fixtures for the device pass-formation kernel (ms_pass_select).

    python tests/golden/make_pass_golden.py       # CPU only, deterministic

Pass formation is the batched executor's policy step (an extension: the
reference never batches across jobs), so its fixtures come from
the ORACLE restatement (oracle/selection.py pass_select) driven over
realistic queues: a virtual-time batched server on the B200 serving profile
measured in round 1 (``serving/tbn_b200_serving.yaml``, the reference YAML
format, frontiers from the product's matrix builder which is byte-identical
to the reference's build_matrix on the committed matrices) with the pass
costs of a measured cost model, Poisson arrivals from light load to 3x
overload, EWMA factors 0.8-1.3, pass caps 96 / 48 / 1024, with and without a
pass-length cap -- plus edge cases (head only, infeasible head, 2,000-job
queues past the kernel's shared-memory staging, one-knot tables, equal
deadlines).  Every problem's packed inputs and the oracle's answer go into
``pass_cases.npz``; the GPU test replays all of them through the C-ABI.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import selection  # noqa: E402
from paper_2310_18481_b200.batcher import FrontierCache  # noqa: E402
from paper_2310_18481_b200.planner import build_matrix, recommended_alphas  # noqa: E402
from paper_2310_18481_b200.registry import load_profile  # noqa: E402
from paper_2310_18481_b200.serving import WorkloadSpec, generate_jobs  # noqa: E402

HERE = Path(__file__).resolve().parent
K = 3
# measured round-1 cost model (bench pass_all knots, us) and encoder work shares
KNOTS_US = [(1, 412.0), (2, 455.0), (3, 497.0), (4, 540.0), (6, 640.0), (8, 745.0), (12, 960.0),
            (16, 1170.0), (24, 1640.0), (32, 2150.0), (48, 3180.0), (64, 4260.0), (96, 6400.0)]
W = [int(round(x * 1024)) for x in (0.2957, 0.3232, 0.3811)]


def table(knots=KNOTS_US, w=W):
    u = [n * 1024 for n, _ in knots]
    t = np.maximum.accumulate([int(round(v * 1000)) for _, v in knots]).tolist()
    return list(w), u, t


class Problems:
    def __init__(self):
        self.groups = {}  # (cap, max_pass_ns, table key) -> list of problems

    def add(self, cap, max_pass_ns, tab, jobs, now, factor):
        w, u, t = tab
        out = selection.pass_select(jobs, now, w, u, t, factor, cap, max_pass_ns)
        key = (cap, max_pass_ns, tuple(w), tuple(u), tuple(t))
        self.groups.setdefault(key, []).append((jobs, now, factor, out))
        return out

    def save(self, path):
        arrs = {}
        for gi, (key, probs) in enumerate(sorted(self.groups.items(), key=lambda kv: kv[0][:2])):
            cap, mp, w, u, t = key
            sizes, dls, ncs, ccs, rms, offs, nj, nows, facs = [], [], [], [], [], [], [], [], []
            res_m, res_n, res_c, res_e, res_ch, res_mask = [], [], [], [], [], []
            joff = 0
            for jobs, now, factor, (m, ch, est, counts, masks) in probs:
                offs.append(joff)
                nj.append(len(jobs))
                nows.append(now)
                facs.append(factor)
                for s, d, cc, mk in jobs:
                    sizes.append(s)
                    dls.append(d)
                    ncs.append(len(cc))
                    ccs.append(np.asarray(cc, np.int16).reshape(-1, K))
                    rms.append(np.asarray(mk, np.uint16).reshape(-1))
                joff += len(jobs)
                res_m.append(m)
                res_n.append(len(masks))
                res_c.append(counts)
                res_e.append(est)
                full = np.full(len(jobs), -1, np.int32)
                full[:m] = ch
                res_ch.append(full)
                res_mask.append(np.asarray(masks, np.uint16))
            p = f"g{gi}_"
            arrs.update({p + "cfg": np.array([cap, mp], np.int64), p + "w": np.array(w, np.int32),
                         p + "u": np.array(u, np.int64), p + "t": np.array(t, np.int64),
                         p + "job_off": np.array(offs, np.int32), p + "n_jobs": np.array(nj, np.int32),
                         p + "now": np.array(nows, np.int64), p + "factor": np.array(facs, np.float64),
                         p + "size": np.array(sizes, np.int32), p + "deadline": np.array(dls, np.int64),
                         p + "n_cand": np.array(ncs, np.int32), p + "cand_counts": np.concatenate(ccs),
                         p + "req_masks": np.concatenate(rms), p + "res_members": np.array(res_m, np.int32),
                         p + "res_requests": np.array(res_n, np.int32),
                         p + "res_counts": np.array(res_c, np.int32).reshape(-1, K),
                         p + "res_est": np.array(res_e, np.int64), p + "res_choice": np.concatenate(res_ch),
                         p + "res_mask": np.concatenate(res_mask) if res_mask else np.zeros(0, np.uint16)})
        arrs["n_groups"] = np.array(len(self.groups))
        np.savez_compressed(path, **arrs)
        return sum(len(v) for v in self.groups.values())


def as_job(tpl, fc):
    cands, pack = fc.lookup(tpl.size, tpl.accuracy_slo)
    if pack is None:
        return None
    return (tpl.size, tpl.deadline_us, pack.counts, pack.masks.reshape(pack.n_cand, tpl.size))


def serve(probs, fc, tab, rate, seconds, seed, cap, max_pass_ns, deadline_ms, rng, fastest_us):
    """Virtual-time batched server forming every pass with the oracle."""
    tpls = [t for t in generate_jobs(WorkloadSpec(kind="poisson", qps=rate, duration_s=1,
                                                  deadline_ms=deadline_ms, seed=seed), PROFILE)]
    tpls = [t for t in tpls if t.size <= 24 and t.arrival_us < seconds * 1_000_000]
    queue = []  # EDF (deadline, seq, job)
    free = 0
    i = 0
    seq = 0
    factor = 1.0
    made = 0
    while i < len(tpls) or queue:
        now = free if queue else max(free, tpls[i].arrival_us)
        while i < len(tpls) and tpls[i].arrival_us <= now:
            j = as_job(tpls[i], fc)
            if j is not None:
                seq += 1
                queue.append((j[1], seq, j))
            i += 1
        if not queue:
            continue
        queue.sort(key=lambda e: (e[0], e[1]))
        while queue and now + fastest_us > queue[0][0]:  # next_dispatch drop rule
            queue.pop(0)
        if not queue:
            continue
        jobs = [e[2] for e in queue]
        m, ch, est, counts, masks = probs.add(cap, max_pass_ns, tab, jobs, now, factor)
        made += 1
        del queue[:m]
        obs = est / 1000.0 * float(rng.uniform(0.85, 1.25))
        factor = 0.8 * factor + 0.2 * (obs / max(1.0, est / 1000.0 / factor))
        factor = float(np.clip(factor, 0.8, 1.3))
        free = now + int(obs)
    return made


def main():
    global PROFILE
    PROFILE = load_profile(HERE / "serving" / "tbn_b200_serving.yaml")
    matrix = build_matrix(PROFILE, range(1, 25), recommended_alphas(PROFILE))
    fc = FrontierCache(matrix, K)
    rng = np.random.default_rng(20261017)
    probs = Problems()
    tab = table()
    fastest = PROFILE.part_latency_us(4, 1)
    total = 0
    for rate, cap, mp, seed in [(8000, 96, 3_000_000, 1), (18000, 96, 3_000_000, 2), (24000, 96, 3_000_000, 3),
                                (30000, 96, 3_000_000, 4), (60000, 96, 3_000_000, 5), (24000, 96, -1, 6),
                                (45000, 48, -1, 7), (20000, 1024, 4_500_000, 8)]:
        total += serve(probs, fc, tab, rate, 0.3, seed, cap, mp, 15.0, rng, fastest)
    # edge cases
    tpls = generate_jobs(WorkloadSpec(kind="poisson", qps=50000, duration_s=1, deadline_ms=15.0, seed=11), PROFILE)
    jobs_all = [j for j in (as_job(t, fc) for t in tpls if t.size <= 24) if j is not None]
    jobs_all.sort(key=lambda j: j[1])
    one = table(KNOTS_US[:1])
    for q in (1, 2, 3, 5):  # tiny queues, one-knot table
        probs.add(96, -1, one, jobs_all[:q], jobs_all[0][1] - 14_000, 1.0)
        probs.add(96, 3_000_000, tab, jobs_all[:q], jobs_all[0][1] - 14_000, 1.0)
    probs.add(96, 3_000_000, tab, jobs_all[:40], jobs_all[0][1] + 1000, 1.0)  # head already late
    probs.add(96, 3_000_000, tab, jobs_all[:2000], jobs_all[0][1] - 14_500, 1.0)  # > smem staging
    probs.add(1024, -1, tab, jobs_all[:2000], jobs_all[0][1] - 14_500, 0.97)
    for f in (0.5, 0.999, 1.0005, 2.0, 3.7):
        probs.add(96, 3_000_000, tab, jobs_all[100:160], jobs_all[100][1] - 13_000, f)
    same = [(s, jobs_all[0][1], cc, mk) for s, _, cc, mk in jobs_all[:30]]  # equal deadlines
    probs.add(96, -1, tab, same, jobs_all[0][1] - 9_000, 1.0)
    n = probs.save(HERE / "pass_cases.npz")
    print(f"{n} pass formations ({total} from serving runs) -> pass_cases.npz")


if __name__ == "__main__":
    main()
