"""The oracle is pinned to the real reference before it is trusted.

Golden vectors come from ``tests/golden/make_golden.py`` (run against the
reference ``modserve`` in the build container; committed as fixtures).
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import selection as orc

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_policy_closed_form_matches_every_reference_case():
    cases = json.loads((GOLDEN / "policy_cases.json").read_text())
    assert len(cases) > 2000
    assert sum(c["expected"] == -1 for c in cases) > 100  # the drop branches are exercised
    bad = [c for c in cases
           if orc.policy_select_one(c["lat_us"], c["deadline_us"], c["dispatch_us"], c["factor"])
           != c["expected"]]
    assert not bad, bad[:3]


def test_policy_cases_cover_running_jobs_and_ms_grid_quirk():
    cases = json.loads((GOLDEN / "policy_cases.json").read_text())
    assert any(c["running_finish_us"] is not None and c["running_finish_us"] > c["now_us"] for c in cases)
    # budget within one millisecond above a fitting estimate but dropped by the 1 ms grid
    quirk = 0
    for c in cases:
        est0 = orc.estimate_us(c["lat_us"][0], c["factor"])
        b = c["deadline_us"] - c["dispatch_us"]
        if c["expected"] == -1 and 0 < b and est0 <= b:
            quirk += 1
    assert quirk > 0


def test_round_half_even_estimates():
    assert orc.estimate_us(5, 0.5) == 2  # 2.5 -> 2 (half to even)
    assert orc.estimate_us(7, 0.5) == 4  # 3.5 -> 4
    assert orc.estimate_us(100_000, 1.2) == 120_000


def test_feedback_ewma_goldens():
    f = orc.feedback_update(1.0, 100, 200)
    assert f == pytest.approx(1.2)
    for _ in range(200):
        f = orc.feedback_update(f, 100, 200)
    assert f == pytest.approx(2.0, rel=1e-9)


def test_frontier_restatement_matches_reference_cases():
    from paper_2310_18481_b200.planner import load_matrix
    from paper_2310_18481_b200.registry import load_profile, scaled_accuracy
    cases = json.loads((GOLDEN / "frontier_cases.json").read_text())
    checked = 0
    for c in cases:
        if c["size"] not in c["sizes"]:
            continue  # rounded sizes are covered by the host-API test
        prof = load_profile(GOLDEN / "profiles" / f"{c['profile']}.yaml")
        from paper_2310_18481_b200.planner import build_matrix, recommended_alphas
        m = build_matrix(prof, c["sizes"], recommended_alphas(prof))
        cells = [(scaled_accuracy(a), m.cells[(c["size"], a)].strategy,
                  m.cells[(c["size"], a)].latency_us, m.cells[(c["size"], a)].credit)
                 for a in m.alphas if m.cells[(c["size"], a)] is not None]
        got = orc.frontier(cells, scaled_accuracy(c["slo"]))
        exp = [(tuple(map(tuple, e["parts"])), e["latency_us"], e["credit"]) for e in c["candidates"]]
        assert [(k.parts, lat, cr) for k, lat, cr in got] == exp
        checked += 1
    assert checked > 50


def test_grouping_rules_pinned_to_reference_canonical_order():
    # all_modalities_strategy(demo, 5) -> ((AV,1),(AV,2),(AV,2)) (test_strategy.py:36-38)
    perm, offs, chunks = orc.group_free_masks(np.array([3, 3, 3, 3, 3]), max_batch=2)
    assert [(m, n) for m, _, n in chunks] == [(3, 1), (3, 2), (3, 2)]
    masks, spans = orc.parts_for_requests(((1, 1), (3, 1)), 2)
    assert masks.tolist() == [1, 3] and spans == [(1, 0, 1), (3, 1, 2)]
    # rounded-up strategy covering more requests than the job has (builder
    # contract, not in the reference): the most-modality parts are filled
    # first, so the row left over is the least-informed subset's
    masks, spans = orc.parts_for_requests(((1, 2), (3, 2)), 3)
    assert masks.tolist() == [3, 3, 1]


def test_compaction_restatement_properties():
    rng = np.random.default_rng(0)
    masks = rng.integers(1, 16, size=500)
    idx, inv, counts = orc.compact(masks, 4)
    for k in range(4):
        assert np.all(np.diff(idx[k]) > 0)  # stable (ascending)
        assert np.all(inv[k][idx[k]] == np.arange(counts[k]))
        assert counts[k] == int(((masks >> k) & 1).sum())
    perm, offs, chunks = orc.group_free_masks(masks, 4)
    assert np.all(np.diff(masks[perm]) >= 0)
    assert sum(n for _, _, n in chunks) == len(masks)
    assert orc.dropped_modalities(0b0101, 3) == 0b010


def test_oracle_bninception_table_is_pinned():
    """The oracle's own BN-Inception table: Ioffe & Szegedy's printed widths
    reproduce SURVEY Appendix C's analytic MACs (2.032 / 2.307 / 2.551 GMAC
    per frame, 69 convs); the TSN widths the models use differ only in
    4c/4d's 1x1 and match the product's independent table and FLOP count."""
    from oracle import bninception as bni
    from paper_2310_18481_b200 import encoders as enc
    got = [round(bni.macs(c, s, bni.IOFFE) / 1e9, 3) for c, s in ((3, 224), (10, 224), (1, 256))]
    assert got == [2.032, 2.307, 2.551]
    assert len(bni.convs(3, bni.IOFFE)) == len(bni.convs(3, bni.TSN)) == 69
    assert {b for b in bni.ORDER if bni.IOFFE[b] != bni.TSN[b]} == {"4c", "4d"}
    for m in enc.TBN_MODALITIES:
        assert bni.macs(m.channels, m.size) == enc.bninception_macs(m.channels, m.size)


def test_oracle_weights_match_the_model_definition():
    import torch
    from oracle import bninception as bni
    from oracle.forward import fusion_weights
    from paper_2310_18481_b200 import encoders as enc
    ow = bni.weights(10, 102)
    pw = enc.bninception_weights(10, 224, 102)
    assert list(ow) == list(pw)
    for k in ow:
        assert torch.equal(ow[k][0], pw[k][0]) and torch.equal(ow[k][1], pw[k][1]), k
    for a, b in zip(fusion_weights(3, 1024, 199), enc.fusion_weights(3, 1024, 199)):
        assert torch.equal(a, b)
    for (a, b), (c, d) in zip(bni.dense_weights((1024, 1024, 1024), 201), enc.mlp_weights((1024, 1024, 1024), 201)):
        assert torch.equal(a, c) and torch.equal(b, d)
