"""Host-side serving logic that needs no GPU: the batched pass cost model,
the marginal (batched) latency table fed to the reference scheduler, and the
knapsack-quantum extension of the reference's OPTIMIZED policy."""

import numpy as np
import pytest

from paper_2310_18481_b200.planner import build_matrix, recommended_alphas
from paper_2310_18481_b200.policy import Policy, apply_policy
from paper_2310_18481_b200.profiler import TBN_ACCURACY, PassCostModel, marginal_profile

ENC = [[400 + 55 * n for n in range(96)], [410 + 62 * n for n in range(96)], [420 + 68 * n for n in range(96)]]
PASS = [(1, 577), (4, 881), (8, 1358), (16, 2203), (24, 2848), (32, 3642), (48, 5046), (96, 9183)]


def _cost():
    return PassCostModel(ENC, [30.0] * 96, 15.0, pass_all_us=PASS)


def test_pass_cost_model_interpolates_whole_passes():
    c = _cost()
    assert abs(sum(c.work_w) - 1.0) < 1e-12
    for n, t in PASS:  # all-modality passes reproduce the measured points
        assert abs(c.raw_us((n, n, n), n) - t) < 1e-6
    # a single-modality pass costs its work share; monotone in every count
    assert c.raw_us((24, 0, 0), 24) < c.raw_us((24, 24, 0), 24) < c.raw_us((24, 24, 24), 24)
    c.observe((24, 24, 24), 24, 2 * PASS[4][1])  # EWMA of observed / estimated
    assert abs(c.factor - 1.2) < 1e-12 and abs(c.estimate_us((24, 24, 24), 24) - 1.2 * PASS[4][1]) < 1e-6


def test_marginal_profile_is_a_valid_reference_table():
    prof = marginal_profile(_cost(), ("rgb", "flow", "audio"), TBN_ACCURACY, max_batch=8)
    lat = np.array(prof.latency_us)
    assert lat.dtype.kind == "i" and lat.min() >= 1
    assert np.all(np.diff(lat, axis=1) >= 0)  # load_profile's monotonicity (profile.py:136-140)
    # a superset of modalities costs more at every batch size
    assert np.all(lat[6] > lat[0]) and np.all(lat[6] > lat[2])
    m = build_matrix(prof, range(1, 13), recommended_alphas(prof))
    assert m.sizes[-1] == 12


def test_fine_knapsack_grid_downgrades_where_the_1ms_grid_drops():
    """With sub-millisecond (marginal) part costs the reference's 1 ms grid
    prices every candidate at one grid unit: a violating queue can only be
    fixed by drops.  A finer quantum lets the same MCKP downgrade instead."""
    from paper_2310_18481_b200.planner import Candidate
    from paper_2310_18481_b200.policy import FeedbackState, Job, JobQueue

    def queue():
        q = JobQueue()
        for i in range(6):
            cands = [Candidate(None, 300, 0.55, 5500), Candidate(None, 900, 0.66, 6600)]
            j = Job(i + 1, 0, 1, 0.5, 2_700 + 10 * i, cands)
            j.assigned_idx = 1
            q.admit(j)
        return q

    q1 = queue()
    d1 = apply_policy(Policy.OPTIMIZED, q1, 0, FeedbackState())
    q2 = queue()
    d2 = apply_policy(Policy.OPTIMIZED, q2, 0, FeedbackState(), grid_us=50)
    assert len(d1) > len(d2) == 0
    assert any(j.assigned_idx == 0 for j in q2.jobs())


def test_refresher_refit_scales_knots_toward_observations():
    """The refresh loop's re-fit (refresh.py): knots with enough nearby
    observations take the median observed/modelled ratio; the others take
    the median ratio of all observations; the result is non-decreasing."""
    from paper_2310_18481_b200.profiler import PassCostModel
    from paper_2310_18481_b200.refresh import ProfileRefresher
    enc = [[100.0 + i for i in range(96)]] * 3
    cost = PassCostModel(enc, [20.0] * 96, 10.0, pass_all_us=[(1, 400.0), (8, 800.0), (32, 2000.0), (96, 6000.0)])
    r = ProfileRefresher(cost, ("a", "b", "c"), (0.5,) * 7, 8, range(1, 9), (0.0, 0.5), min_obs=4)
    for _ in range(10):  # observed 20 % slower near n = 8 (work 8)
        r.observe([8, 8, 8], 8, 960.0)
    obs = r._obs
    for _ in range(10):  # and 10 % slower near n = 32
        r.observe([32, 32, 32], 32, 2200.0)
    knots, g = r.refit(obs)
    assert dict(knots)[8] == pytest.approx(960.0)
    assert dict(knots)[32] == pytest.approx(2200.0)
    assert g == pytest.approx(1.15)
    assert dict(knots)[1] == pytest.approx(460.0) and dict(knots)[96] == pytest.approx(6900.0)
    assert all(b[1] >= a[1] for a, b in zip(knots, knots[1:]))
    r.close()


def test_frontier_cache_warm_matches_lookups():
    """FrontierCache.warm (filled off the serving thread on a matrix swap)
    holds exactly the frontiers candidates_for_job returns for any SLO."""
    import numpy as np

    import paper_2310_18481_b200 as ms
    from paper_2310_18481_b200.batcher import FrontierCache
    prof = ms.synth_profile(ms.SynthSpec(n_modalities=3, max_batch=4), seed=0)
    matrix = ms.build_matrix(prof, range(1, 7), ms.recommended_alphas(prof))
    fc = FrontierCache(matrix, 3)
    fc.warm()
    n = len(fc._cache)
    assert n >= 6 * len(matrix.alphas)
    rng = np.random.default_rng(0)
    for _ in range(300):
        size = int(rng.integers(1, 7))
        slo = float(rng.uniform(0.3, 1.0))
        cands, _ = fc.lookup(size, slo)
        assert cands == ms.candidates_for_job(matrix, size, slo)
    assert len(fc._cache) == n  # no miss after warm()


def test_refresher_helper_process_rebuild_matches_host():
    """The refresh rebuild runs in a helper process: its profile/matrix are
    the ones an in-process marginal_profile + build_matrix produce, and the
    cooperative cache fill ends in a swap (poll) with factor continuity."""
    import time

    from paper_2310_18481_b200.planner import build_matrix, save_matrix
    from paper_2310_18481_b200.profiler import PassCostModel, marginal_profile
    from paper_2310_18481_b200.refresh import ProfileRefresher
    enc = [[100.0 + 3 * i for i in range(96)]] * 3
    cost = PassCostModel(enc, [20.0] * 96, 10.0, pass_all_us=[(1, 400.0), (8, 800.0), (32, 2000.0), (96, 6000.0)])
    cost.factor = 1.3
    acc = (0.55, 0.6, 0.7, 0.5, 0.65, 0.62, 0.75)
    r = ProfileRefresher(cost, ("a", "b", "c"), acc, 8, range(1, 9), (0.0, 0.5, 0.6, 0.7), min_obs=4, period_s=0.0)
    try:
        assert not r.due(0.0)
        for _ in range(10):
            r.observe([8, 8, 8], 8, 1040.0)  # 1.3x the model at n = 8
        assert r.due(1.0)
        r.start(1.0)
        res = None
        t0 = time.time()
        while res is None and time.time() - t0 < 60:
            r.advance(4)
            res = r.poll()
            time.sleep(0.01)
        assert res is not None
        assert res.matrix.profile_fingerprint == res.profile.fingerprint()
        ref_prof = marginal_profile(res.cost, ("a", "b", "c"), acc, 8, name=r.name)
        assert ref_prof.fingerprint() == res.profile.fingerprint()
        import tempfile
        from pathlib import Path
        with tempfile.TemporaryDirectory() as d:
            save_matrix(res.matrix, Path(d) / "a.json")
            save_matrix(build_matrix(ref_prof, range(1, 9), (0.0, 0.5, 0.6, 0.7)), Path(d) / "b.json")
            assert (Path(d) / "a.json").read_bytes() == (Path(d) / "b.json").read_bytes()
        assert res.absorbed == pytest.approx(1.3)
        assert res.cost.factor == pytest.approx(1.0)  # 1.3 / 1.3: the knots took the bias
        assert r.cost is res.cost
    finally:
        r.close()
