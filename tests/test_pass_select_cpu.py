"""Pass formation (the batched executor's policy step) on the CPU: the
oracle restatement against its committed fixtures and its own invariants,
the host packing, and the C-ABI's argument checks (no GPU needed)."""

import ctypes

import numpy as np
import pytest

from oracle import selection as orc
import pass_cases as pc


def test_oracle_reproduces_committed_formations():
    n = 0
    for g in pc.groups():
        w, u, t = g["w"].tolist(), g["u"].tolist(), g["t"].tolist()
        cap, mp = (int(x) for x in g["cfg"])
        for i in range(len(g["job_off"])):
            got = orc.pass_select(pc.problem_jobs(g, i), int(g["now"][i]), w, u, t, float(g["factor"][i]), cap, mp)
            assert got == pc.expected(g, i), i
            n += 1
    assert n >= 1000


def test_formation_invariants():
    """Members' deadlines, the cap and the pass-length cap hold whenever the
    head alone did; choices never go below the fastest candidate; the masks
    are the chosen candidates' masks in member order."""
    checked = 0
    for g in pc.groups():
        w, u, t = g["w"].tolist(), g["u"].tolist(), g["t"].tolist()
        cap, mp = (int(x) for x in g["cfg"])
        for i in range(len(g["job_off"])):
            jobs = pc.problem_jobs(g, i)
            now, f = int(g["now"][i]), float(g["factor"][i])
            m, ch, est, counts, masks = orc.pass_select(jobs, now, w, u, t, f, cap, mp)
            assert 1 <= m <= len(jobs)
            assert sum(j[0] for j in jobs[:m]) <= max(cap, jobs[0][0])
            exp_masks = [int(x) for j, c in zip(jobs[:m], ch) for x in j[3][c]]
            assert masks == exp_masks
            assert counts == [sum((mk >> k) & 1 for mk in masks) for k in range(len(w))]
            assert est == orc.pass_estimate_ns(counts, w, u, t, f)
            head_ok = now * 1000 + orc.pass_estimate_ns(list(jobs[0][2][0]), w, u, t, f) <= jobs[0][1] * 1000
            if head_ok and m > 1:
                assert now * 1000 + est <= min(j[1] for j in jobs[:m]) * 1000
                assert mp < 0 or est <= mp
            checked += 1
    assert checked >= 1000


def test_tiny_formation_by_hand():
    # two modalities, work 512/1024 per request; knots 1 req -> 100 us, 3 req -> 300 us
    w, u, t = [512, 512], [1024, 3072], [100_000, 300_000]
    # job A (size 1): candidates {m1}, {m1+m2}; job B (size 1): {m2}, {m1+m2}
    a = (1, 1000, np.array([[1, 0], [1, 1]]), np.array([[1], [3]]))
    b = (1, 1000, np.array([[0, 1], [1, 1]]), np.array([[2], [3]]))
    # now = 0, deadlines 1000 us: everything fits -> both top
    assert orc.pass_select([a, b], 0, w, u, t, 1.0, 96, -1) == (2, [1, 1], 200_000, [2, 2], [3, 3])
    # deadline 150 us: fastest pair = work 1024 -> 100 us; A top -> 1536 -> 150 us ok; then B top -> 200 us no
    a2, b2 = (1, 150, a[2], a[3]), (1, 150, b[2], b[3])
    assert orc.pass_select([a2, b2], 0, w, u, t, 1.0, 96, -1) == (2, [1, 0], 150_000, [1, 2], [3, 2])
    # cap 1: only the head
    assert orc.pass_select([a, b], 0, w, u, t, 1.0, 1, -1)[0] == 1
    # a queued job that can still make it after an all-fastest pass constrains the upgrades
    c = (1, 260, a[2], a[3])
    m, ch, est, counts, masks = orc.pass_select([a, b, c], 0, w, u, t, 1.0, 2, -1)
    assert m == 2 and est + orc.pass_estimate_ns([1, 0], w, u, t, 1.0) <= 260_000


def test_estimate_matches_round_half_even():
    w, u, t = [1024], [1024, 2048], [1000, 1001]
    # raw at u=1536: 1000 + 1*512//1024 = 1000; *2.5 = 2500 exactly
    assert orc.pass_estimate_ns([1], w, u, t, 2.5) == 2500
    assert orc.pass_estimate_ns([1], [1], [1, 2], [1, 2], 2.5) == 2  # round(2.5) half-even
    assert orc.pass_raw_ns(10 * 1024, [1024, 2048], [1000, 2000]) == 10_000  # extrapolated


def test_frontier_pack_layout():
    from paper_2310_18481_b200.batcher import FrontierCache
    from paper_2310_18481_b200.planner import build_matrix, recommended_alphas
    from paper_2310_18481_b200.registry import load_profile
    prof = load_profile(pc.GOLDEN / "serving" / "tbn_b200_serving.yaml")
    m = build_matrix(prof, range(1, 7), recommended_alphas(prof))
    fc = FrontierCache(m, 3)
    for size in range(1, 7):
        for slo in (0.38, 0.5, 0.6, 0.65, 0.66):
            cands, pack = fc.lookup(size, slo)
            from paper_2310_18481_b200.policy import candidates_with_rounding
            ref = candidates_with_rounding(m, size, slo)
            assert [c.strategy for c in cands] == [c.strategy for c in ref]
            if not cands:
                assert pack is None
                continue
            assert pack.masks.shape == (len(cands) * size,) and pack.counts.shape == (len(cands), 3)
            for ci, c in enumerate(cands):
                exp, _ = orc.parts_for_requests(c.strategy.parts, size)
                assert pack.masks[ci * size:(ci + 1) * size].tolist() == exp.tolist()
                assert pack.counts[ci].tolist() == [int(((exp >> k) & 1).sum()) for k in range(3)]


def test_abi_pass_select_rejects_bad_arguments():
    from paper_2310_18481_b200 import build, device
    build.build()
    L = device.lib()
    assert ctypes.sizeof(device.PassCost) == 552
    cost = device.PassCost.make([300, 330, 390], [1024, 2048], [400_000, 450_000])
    dummy = ctypes.c_void_p(16)
    args = [1] + [dummy] * 11 + [ctypes.byref(cost), 96, -1] + [dummy] * 4 + [96, None, None]
    bad = list(args)
    bad[13] = 0  # cap
    assert L.ms_pass_select(*bad) == 1 and b"cap" in L.ms_last_error()
    bad = list(args)
    bad[19] = 8  # out_mask_ld < cap
    assert L.ms_pass_select(*bad) == 1
    dec = device.PassCost.make([1, 1, 1], [2048, 1024], [1, 2])
    bad = list(args)
    bad[12] = ctypes.byref(dec)
    assert L.ms_pass_select(*bad) == 1 and b"knots" in L.ms_last_error()
    bad = list(args)
    bad[5] = None
    assert L.ms_pass_select(*bad) == 1 and b"null" in L.ms_last_error()
    assert L.ms_pass_select(0, *args[1:]) == 0  # nothing to do, no CUDA call
