"""End-to-end masked forward on the B200 vs the frozen CPU oracle.

Modality grouping (which requests each encoder saw) is bit-exact; logits
are within the north_star tolerance: rtol 2e-2 (scale-relative max error)
and >= 99.9 % top-1 agreement, near-ties (oracle top-2 gap below the
tolerance) excepted.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 2e-2


def _check_logits(got, ref):
    got, ref = got.float().cpu(), ref.float().cpu()
    scale = ref.abs().max().item()
    err = (got - ref).abs().max().item()
    assert err <= RTOL * scale, (err, scale)
    top_g, top_r = got.argmax(1), ref.argmax(1)
    srt = ref.sort(1, descending=True).values
    gap = srt[:, 0] - srt[:, 1]
    agree = (top_g == top_r) | (gap <= RTOL * scale)
    assert agree.float().mean().item() >= 0.999
    return err / scale, (top_g == top_r).float().mean().item()


@pytest.fixture(scope="module")
def built():
    from paper_2310_18481_b200 import build
    build.build()


def test_mlp_model_c1_vs_oracle(built):
    """configs[0]: 3 modality MLP towers, 256 requests, masks uniform over the 7 combos."""
    from oracle.forward import OracleMLP
    from paper_2310_18481_b200.executor import build_mlp_model
    dims = (1024, 1024, 1024)
    model = build_mlp_model(dims, max_req=256, n_slots=256)
    rng = np.random.default_rng(0)
    masks = rng.integers(1, 8, size=256)
    slots = rng.permutation(256)
    logits = model.forward(slots, masks).clone()
    torch.cuda.synchronize()
    assert tuple(model.counts.cpu().tolist()) == model.counts_for(masks)
    orc = OracleMLP(dims, (201, 202, 203), 299)
    inputs = [p[torch.as_tensor(slots).long().cuda(), :d].float().cpu() for p, d in zip(model.pools, dims)]
    ref = orc.logits(inputs, torch.as_tensor(masks))
    rel, agree = _check_logits(logits, ref)
    print(f"MLP C1: max rel err {rel:.2e}, top-1 agreement {agree:.4f}")


def test_tbn_model_masked_forward_vs_oracle(built):
    """configs[1] shapes at a CPU-sized batch: every combo once, some twice."""
    from oracle.forward import OracleTBN
    from paper_2310_18481_b200.encoders import TBN_MODALITIES
    from paper_2310_18481_b200.executor import build_tbn_model
    model = build_tbn_model(max_req=10, n_slots=12)
    masks = np.array([7, 1, 2, 4, 3, 5, 6, 7, 1, 6])
    slots = np.array([0, 3, 5, 7, 11, 2, 9, 1, 4, 6])
    logits = model.forward(slots, masks).clone()
    torch.cuda.synchronize()
    # grouping bit-exact
    idx = model.idx[: 3 * len(masks)].view(3, -1).cpu().numpy()
    for k in range(3):
        exp = np.flatnonzero((masks >> k) & 1)
        assert np.array_equal(idx[k, : len(exp)], exp)
    orc = OracleTBN(TBN_MODALITIES, (101, 102, 103), 199, 3)
    sl = torch.as_tensor(slots).long().cuda()
    clips = [p[sl].cpu() for p in model.pools]
    ref = orc.logits(clips, torch.as_tensor(masks))
    rel, agree = _check_logits(logits, ref)
    print(f"TBN: max rel err {rel:.2e}, top-1 agreement {agree:.4f}")


def test_tbn_graph_replay_matches_eager(built):
    from paper_2310_18481_b200.executor import build_tbn_model
    model = build_tbn_model(max_req=8, n_slots=8)
    masks = np.array([7, 3, 5, 1, 2, 7, 4, 6])
    slots = np.arange(8)
    model.use_graphs = False
    a = model.forward(slots, masks).clone()
    model.use_graphs = True
    b = model.forward(slots, masks).clone()
    c = model.forward(slots, masks).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(b, c)


def test_tbn_pdl_and_branch_lanes_bitwise_stable(built):
    """Programmatic dependent launch and the concurrent Inception branch
    lanes change only scheduling: logits are bitwise identical with PDL off
    (serial launches), on (eager) and on (CUDA graph with lane fork/join)."""
    from paper_2310_18481_b200 import device as dv
    from paper_2310_18481_b200.executor import build_tbn_model
    model = build_tbn_model(max_req=12, n_slots=12)
    rng = np.random.default_rng(3)
    masks = rng.integers(1, 8, size=12)
    slots = rng.permutation(12)
    prev = dv.set_pdl(False)
    try:
        model.use_graphs = False
        a = model.forward(slots, masks).clone()
        dv.set_pdl(True)
        b = model.forward(slots, masks).clone()
        model.use_graphs = True
        c = model.forward(slots, masks).clone()
        d = model.forward(slots, masks).clone()
    finally:
        dv.set_pdl(prev)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(b, c) and torch.equal(c, d)


def test_realtime_serving_batched_and_host_io(built):
    """Wall-clock serving on the device: every request accounted for, each
    completed job met its accuracy floor, batching merged jobs, and the
    host-IO path copied only the present modalities' clips."""
    import paper_2310_18481_b200 as ms
    from paper_2310_18481_b200.executor import build_tbn_model
    from paper_2310_18481_b200.profiler import TBN_ACCURACY, profile_model, profile_pass_costs
    from paper_2310_18481_b200.realtime import HostClips, serve_realtime
    model = build_tbn_model(max_req=16, n_slots=32)
    prof = profile_model(model, ("rgb", "flow", "audio"), TBN_ACCURACY, max_batch=4, reps=2)
    matrix = ms.build_matrix(prof, range(1, 9), ms.recommended_alphas(prof))
    cost = profile_pass_costs(model, reps=2)
    spec = ms.WorkloadSpec(kind="poisson", qps=1500, duration_s=1, deadline_ms=20, seed=5)
    jobs = [ms.JobTemplate(j.arrival_us, min(j.size, 8), j.accuracy_slo, j.deadline_us)
            for j in ms.generate_jobs(spec, prof)]
    log, st = serve_realtime(model, prof, matrix, jobs, cost=cost)
    assert len(log.records) == len(jobs)
    assert sum(r.size for r in log.records) == sum(j.size for j in jobs)
    assert all(r.achieved_accuracy >= r.accuracy_slo for r in log.records if not r.dropped)
    assert st.passes < len([r for r in log.records if not r.dropped])  # jobs were merged
    log2, st2 = serve_realtime(model, prof, matrix, jobs, cost=cost, host_clips=HostClips(model))
    assert len(log2.records) == len(jobs)
    n_req = sum(j.size for j in jobs)
    full = sum(model.row_bytes) * n_req
    assert 0 < st2.h2d_bytes <= full + (2 + 4 * model.K) * n_req  # only present modalities are transferred
    assert st2.h2d_bytes % 2 == 0 and st2.d2h_bytes > 0


def test_realtime_pass_selection_meets_slos(built):
    """Batched pass-level selection (per-request accuracy argmax under the
    formed pass's deadline): every served request meets its accuracy floor,
    an idle GPU keeps every job at its most accurate candidate, and an
    overloaded one drops modalities instead of missing deadlines."""
    import paper_2310_18481_b200 as ms
    from paper_2310_18481_b200.executor import build_tbn_model
    from paper_2310_18481_b200.policy import Policy
    from paper_2310_18481_b200.profiler import TBN_ACCURACY, marginal_profile, profile_pass_costs
    from paper_2310_18481_b200.realtime import serve_realtime
    model = build_tbn_model(max_req=32, n_slots=32)
    cost = profile_pass_costs(model, reps=2)
    prof = marginal_profile(cost, ("rgb", "flow", "audio"), TBN_ACCURACY, max_batch=4)
    matrix = ms.build_matrix(prof, range(1, 9), ms.recommended_alphas(prof))

    def run(qps, seed):
        spec = ms.WorkloadSpec(kind="poisson", qps=qps, duration_s=1, deadline_ms=15, seed=seed)
        jobs = [ms.JobTemplate(j.arrival_us, min(j.size, 8), j.accuracy_slo, j.deadline_us)
                for j in ms.generate_jobs(spec, prof)]
        cost.factor = 1.0
        log, st = serve_realtime(model, prof, matrix, jobs, cost=cost, policy=Policy.NONE, selection="pass",
                                 max_pass_us=0.25 * 15_000)
        assert len(log.records) == len(jobs)
        served = [r for r in log.records if not r.dropped]
        assert all(r.achieved_accuracy >= r.accuracy_slo for r in served)
        return log, served

    log, served = run(200, 3)  # light load: top accuracy, on time
    top = prof.combo_accuracy(prof.all_modalities_mask)
    assert log.violation_ratio() == 0.0
    assert sum(r.size for r in served if r.achieved_accuracy >= top - 1e-9) >= 0.95 * sum(r.size for r in served)
    # 1.4x what all-modality passes of <= 32 requests can serve (measured pass cost)
    overload = 1.4 * 32 / (cost.pass_all_us(32) * 1e-6)
    log, served = run(overload, 4)
    dropped = sum(r.size for r in served if r.achieved_accuracy < top - 1e-9)
    total = sum(r.size for r in served)
    assert dropped > 0.2 * total, (dropped, total, log.violation_ratio())
    assert log.violation_ratio() < 0.15, (dropped, total, log.violation_ratio())


def _oracle_rows(orc, model, rows_per_mod, masks, pick):
    """Oracle logits for the requests ``pick`` (each request's logits depend
    only on its own clips): rows_per_mod[k][i] = pool row of request i."""
    clips = [p.cpu()[torch.as_tensor(np.asarray(r)[pick]).long()] for p, r in zip(model.pools, rows_per_mod)]
    return orc.logits(clips, torch.as_tensor(np.asarray(masks)[pick]))


@pytest.fixture(scope="module")
def tbn96(built):
    from paper_2310_18481_b200.executor import build_tbn_model
    return build_tbn_model(max_req=96, n_slots=192)


def test_tbn_bench_operating_point_passes_vs_oracle(tbn96):
    """The bench's operating configuration (max_req 96: 2-SM pair tiles,
    split-K, halo/K32 convs, per-count CUDA graphs with concurrent branch
    lanes): a full 96-request mixed pass and a 61-request pass with the
    served modality mix (all rgb, ~60 % flow, ~40 % audio), both through the
    graphs; grouping bit-exact, logits vs the oracle on 32 sampled requests
    of each (covering every combo present)."""
    from oracle.forward import OracleTBN
    from paper_2310_18481_b200.encoders import TBN_MODALITIES
    model = tbn96
    orc = OracleTBN(TBN_MODALITIES, (101, 102, 103), 199, 3)
    rng = np.random.default_rng(11)
    mixed = rng.integers(1, 8, size=96)
    served = 1 | (rng.random(61) < 0.6) * 2 | (rng.random(61) < 0.4) * 4
    for masks in (mixed, served):
        n = len(masks)
        slots = rng.permutation(model.n_slots)[:n]
        logits = model.forward(slots, masks).clone()
        torch.cuda.synchronize()
        idx = model.idx[: 3 * n].view(3, n).cpu().numpy()
        for k in range(3):
            exp = np.flatnonzero((masks >> k) & 1)
            assert np.array_equal(idx[k, : len(exp)], exp)
        pick = np.sort(np.concatenate([np.flatnonzero(masks == m)[:2] for m in range(1, 8)] +
                                       [rng.permutation(n)[:32]]))[:32]
        pick = np.unique(pick)
        ref = _oracle_rows(orc, model, [slots] * 3, masks, pick)
        rel, agree = _check_logits(logits[pick], ref)
        print(f"TBN n={n}: max rel err {rel:.2e}, top-1 agreement {agree:.4f} on {len(pick)} rows")


def test_tbn_ring_path_host_io_logits_vs_oracle(tbn96):
    """The e2e host-IO path exactly as the server runs it: a pass formed on
    the device (ms_pass_select writes the masks into the mask ring), each
    modality's clips DMA'd into its pool ring at the ring base, compaction in
    ring mode; distinct data in every host row, so a wrong row map fails.
    Logits vs the oracle on the rows actually copied."""
    from oracle.forward import OracleTBN
    from oracle import selection as orc_sel
    from paper_2310_18481_b200 import device as dv
    from paper_2310_18481_b200.batcher import DevicePassSelector
    from paper_2310_18481_b200.encoders import TBN_MODALITIES
    model = tbn96
    ns = model.n_slots
    g = torch.Generator().manual_seed(5)
    host = []
    for p in model.pools:  # fresh, distinct host rows (pinned)
        h = (torch.randint(0, 256, p.shape, generator=g, dtype=torch.uint8) if p.dtype == torch.uint8 else
             torch.randn(p.shape, generator=g).to(p.dtype))
        host.append(h.pin_memory())
    # one formation: three jobs whose fastest candidates use different modalities
    cost = dv.PassCost.make([300, 330, 390], [1024, 96 * 1024], [400_000, 6_400_000])
    sel = DevicePassSelector(3, cost, 96, -1, model.mask_ring)

    class J:
        def __init__(self, size, dl, masks):
            from paper_2310_18481_b200.batcher import FrontierPack
            self.deadline_us = dl
            self.pack = FrontierPack.__new__(FrontierPack)
            m = np.asarray(masks, np.uint16)
            self.pack.size, self.pack.n_cand = size, m.shape[0]
            self.pack.masks = m.reshape(-1)
            self.pack.counts = np.stack([((m >> k) & 1).sum(1) for k in range(3)], 1).astype(np.int16)

    jobs = [J(20, 50_000, [[1] * 20, [3] * 20, [7] * 20]), J(25, 50_000, [[4] * 25, [5] * 25]),
            J(30, 50_000, [[2] * 30, [6] * 10 + [7] * 20])]
    bases = [ns - 7, 3, ns - 40]  # wrap-around on rgb and audio
    r = sel.select(jobs, 0, 1.0, slot=0)
    w, u, t = cost.table()
    ref_sel = orc_sel.pass_select([(j.pack.size, j.deadline_us, j.pack.counts,
                                    j.pack.masks.reshape(j.pack.n_cand, j.pack.size)) for j in jobs],
                                  0, w, u, t, 1.0, 96, -1)
    assert (r.members, r.choices.tolist(), r.est_ns, list(r.counts)) == ref_sel[:4]
    masks = np.asarray(ref_sel[4])
    cs = torch.cuda.Stream()
    model.ring_upload(host, r.counts, bases, cs)
    torch.cuda.current_stream().wait_stream(cs)
    model.run_ring(r.requests, r.counts, 0, bases)
    logits = model.head.logits[: r.requests].clone()
    torch.cuda.synchronize()
    assert np.array_equal(model.mask_ring[0, : r.requests].cpu().numpy().view(np.uint16), masks)
    # request i's modality-k row: (base_k + position of i among modality-k requests) % ns
    rows = []
    for k in range(3):
        has = (masks >> k) & 1
        pos = np.cumsum(has) - 1
        rows.append(np.where(has == 1, (bases[k] + pos) % ns, 0))
    orc = OracleTBN(TBN_MODALITIES, (101, 102, 103), 199, 3)
    pick = np.unique(np.concatenate([np.flatnonzero(masks == m)[:4] for m in range(1, 8)]))
    clips = [h[torch.as_tensor(rr[pick]).long()] for h, rr in zip(host, rows)]
    ref = orc.logits(clips, torch.as_tensor(masks[pick].astype(np.int64)))
    rel, agree = _check_logits(logits[pick], ref)
    print(f"ring host-IO pass: {r.requests} requests, counts {r.counts}, rel err {rel:.2e} on {len(pick)} rows")
