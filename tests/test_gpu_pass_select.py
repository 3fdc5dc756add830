"""The device pass-formation kernel (ms_pass_select) on the B200, bit-exact
against the oracle restatement (oracle/selection.py pass_select):

* every committed formation (tests/golden/pass_cases.npz: >= 2,400 problems
  from virtual-time serving runs and edge cases), batched, from device
  memory and from pinned (mapped) host memory -- members, choices,
  per-modality counts, the pass estimate and the per-request masks;
* >= 1,000 formations recorded from a REAL wall-clock serving run on the
  TBN model (the bench's path), replayed through the oracle.
"""

import numpy as np
import pytest

from oracle import selection as orc
import pass_cases as pc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_2310_18481_b200 import build, device
    build.build()
    device.lib()
    return device


def _run_group(dev, g, pinned=False):
    def put(a, dt):
        t = torch.as_tensor(np.ascontiguousarray(a)).to(dt)
        return t.pin_memory() if pinned else t.cuda()

    n_prob = len(g["job_off"])
    n_jobs = len(g["size"])
    cap, mp = (int(x) for x in g["cfg"])
    coff = np.concatenate([[0], np.cumsum(g["n_cand"])[:-1]]).astype(np.int32)
    moff = np.concatenate([[0], np.cumsum(g["n_cand"].astype(np.int64) * g["size"])[:-1]]).astype(np.int32)
    ins = [put(g["job_off"], torch.int32), put(g["n_jobs"], torch.int32), put(g["now"], torch.int64),
           put(g["factor"], torch.float64), put(g["size"], torch.int32), put(g["deadline"], torch.int64),
           put(g["n_cand"], torch.int32), put(coff, torch.int32), put(moff, torch.int32),
           put(g["cand_counts"].reshape(-1), torch.int16), put(g["req_masks"].view(np.int16), torch.int16)]
    choice = put(np.full(n_jobs, -7, np.int32), torch.int32)
    summ = put(np.zeros(n_prob * dev.PASS_SUMMARY, np.int32), torch.int32)
    est = put(np.zeros(n_prob, np.int64), torch.int64)
    mask = torch.full((n_prob, cap), -1, dtype=torch.int16, device="cuda")
    cost = dev.PassCost.make(g["w"], g["u"], g["t"])
    dev.pass_select(n_prob, *[t.data_ptr() for t in ins], cost, cap, mp, choice.data_ptr(), summ.data_ptr(),
                    est.data_ptr(), mask.data_ptr(), cap)
    torch.cuda.synchronize()
    return (choice.cpu().numpy(), summ.cpu().numpy().reshape(n_prob, -1), est.cpu().numpy(),
            mask.cpu().numpy().view(np.uint16))


def _compare(g, out):
    choice, summ, est, mask = out
    bad = 0
    for i in range(len(g["job_off"])):
        m, ch, e, counts, masks = pc.expected(g, i)
        j0, q = int(g["job_off"][i]), int(g["n_jobs"][i])
        ok = (summ[i, 0] == m and summ[i, 1] == len(masks) and summ[i, 2:2 + pc.K].tolist() == counts
              and est[i] == e and choice[j0:j0 + m].tolist() == ch and (choice[j0 + m:j0 + q] == -1).all()
              and mask[i, :len(masks)].tolist() == masks)
        bad += not ok
    return bad


def test_pass_select_replays_committed_formations(dev):
    total = bad = 0
    for g in pc.groups():
        bad += _compare(g, _run_group(dev, g))
        total += len(g["job_off"])
    assert total >= 2000
    assert bad == 0, f"{bad} of {total} formations differ from the oracle"


def test_pass_select_reads_pinned_host_memory(dev):
    """The serving loop hands the kernel its pinned staging buffers (mapped
    host memory, no memcpy): same answers."""
    for g in pc.groups()[:3]:
        assert _compare(g, _run_group(dev, g, pinned=True)) == 0


def test_served_formations_replay_bit_exact(dev):
    """A real wall-clock serving run of the TBN model (the bench's path, pass
    cap 96): every pass formed on the device during the run is replayed
    through the oracle -- >= 1,000 formations, zero mismatches."""
    import paper_2310_18481_b200 as ms
    from paper_2310_18481_b200.batcher import unpack_jobs
    from paper_2310_18481_b200.executor import build_tbn_model
    from paper_2310_18481_b200.policy import Policy
    from paper_2310_18481_b200.profiler import TBN_ACCURACY, marginal_profile, profile_pass_costs
    from paper_2310_18481_b200.realtime import serve_realtime
    model = build_tbn_model(max_req=96, n_slots=192)
    cost = profile_pass_costs(model, reps=2)
    prof = marginal_profile(cost, ("rgb", "flow", "audio"), TBN_ACCURACY, max_batch=8)
    matrix = ms.build_matrix(prof, range(1, 25), ms.recommended_alphas(prof))
    table = cost.device_table()
    w, u, t = table.table()
    n_form = 0
    for qps, seed in ((4000, 1), (20000, 2), (30000, 3)):
        spec = ms.WorkloadSpec(kind="poisson", qps=qps, duration_s=2, deadline_ms=15, seed=seed)
        jobs = [ms.JobTemplate(j.arrival_us, min(j.size, 24), j.accuracy_slo, j.deadline_us)
                for j in ms.generate_jobs(spec, prof)]
        cost.factor = 1.0
        log, st = serve_realtime(model, prof, matrix, jobs, cost=cost, policy=Policy.NONE, selection="pass",
                                 max_pass_us=0.2 * 15_000, record_formations=True)
        assert st.policy_launches == st.passes == len(st.formations)
        for rec in st.formations:
            got = orc.pass_select(unpack_jobs(rec, 3), rec["now_us"], w, u, t, rec["factor"], 96, 3_000_000)
            m, ch, est, counts, masks = got
            assert (m, ch, est, counts, len(masks)) == (rec["members"], rec["choices"].tolist(), rec["est_ns"],
                                                         list(rec["counts"]), rec["requests"])
        n_form += len(st.formations)
        served = [r for r in log.records if not r.dropped]
        assert all(r.achieved_accuracy >= r.accuracy_slo for r in served)
    assert n_form >= 1000, n_form


def test_refresh_loop_hot_swaps_matrix_without_slo_dip(dev, tmp_path):
    """a serving run whose cost model starts 25 % optimistic
    re-profiles itself from its own passes' CUDA-event times, rebuilds the
    serving profile + matrix on the device in the background and swaps them
    in mid-run: >= 1 swap, the re-fitted knots move toward the measured
    passes, the run stays >= 99 % on time, and every swapped matrix is
    byte-identical to a host-DP rebuild of its profile with a matching
    fingerprint (strategy.py:505-520)."""
    import paper_2310_18481_b200 as ms
    from paper_2310_18481_b200.executor import build_tbn_model
    from paper_2310_18481_b200.planner import build_matrix, save_matrix
    from paper_2310_18481_b200.policy import Policy
    from paper_2310_18481_b200.profiler import (TBN_ACCURACY, PassCostModel, marginal_profile,
                                                profile_pass_costs)
    from paper_2310_18481_b200.realtime import serve_realtime
    from paper_2310_18481_b200.refresh import ProfileRefresher
    model = build_tbn_model(max_req=96, n_slots=192)
    true = profile_pass_costs(model, reps=2)
    skew = PassCostModel(true.enc_us, true.head_us, true.compact_us, pass_all_us=[(n, 0.75 * t) for n, t in true.pass_all])
    mods = ("rgb", "flow", "audio")
    prof = marginal_profile(skew, mods, TBN_ACCURACY, max_batch=8)
    matrix = ms.build_matrix(prof, range(1, 25), ms.recommended_alphas(prof))
    ref = ProfileRefresher(skew, mods, TBN_ACCURACY, 8, range(1, 25), matrix.alphas, period_s=0.5)
    spec = ms.WorkloadSpec(kind="poisson", qps=12000, duration_s=4, deadline_ms=15, seed=9)
    jobs = [ms.JobTemplate(j.arrival_us, min(j.size, 24), j.accuracy_slo, j.deadline_us)
            for j in ms.generate_jobs(spec, prof)]
    log, st = serve_realtime(model, prof, matrix, jobs, cost=skew, policy=Policy.NONE, selection="pass",
                             max_pass_us=3000, refresher=ref)
    assert len(st.refreshes) >= 1
    assert log.violation_ratio() <= 0.01, log.violation_ratio()
    for r in st.refreshes:
        assert r.matrix.profile_fingerprint == r.profile.fingerprint()
        save_matrix(r.matrix, tmp_path / "dev.json")
        save_matrix(build_matrix(r.profile, range(1, 25), matrix.alphas), tmp_path / "host.json")
        assert (tmp_path / "dev.json").read_bytes() == (tmp_path / "host.json").read_bytes()
    # the busiest knot moved toward the measured pass time
    last = dict(st.refreshes[-1].knots_after)
    moved = [n for n, t in skew.pass_all if last[n] != t]
    assert moved
    for n in moved:
        assert abs(last[n] - true.pass_all_us(n)) < abs(0.75 * true.pass_all_us(n) - true.pass_all_us(n))
