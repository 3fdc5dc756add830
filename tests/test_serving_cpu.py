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
    observations take the median observed/modelled ratio; the others keep
    their time; the result is non-decreasing."""
    from paper_2310_18481_b200.profiler import PassCostModel
    from paper_2310_18481_b200.refresh import ProfileRefresher
    enc = [[100.0 + i for i in range(96)]] * 3
    cost = PassCostModel(enc, [20.0] * 96, 10.0, pass_all_us=[(1, 400.0), (8, 800.0), (32, 2000.0), (96, 6000.0)])
    r = ProfileRefresher(cost, ("a", "b", "c"), (0.5,) * 7, 8, range(1, 9), (0.0, 0.5), min_obs=4)
    for _ in range(10):  # observed 20 % slower near n = 8 (work 8)
        r.observe([8, 8, 8], 8, 960.0)
    obs = r._obs
    knots = r.refit(obs)
    assert dict(knots)[8] == pytest.approx(960.0)
    assert dict(knots)[1] == 400.0 and dict(knots)[96] == 6000.0
    assert all(b[1] >= a[1] for a, b in zip(knots, knots[1:]))
