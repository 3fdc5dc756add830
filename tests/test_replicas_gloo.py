"""Multi-GPU path on CPU: world_size 2 with the gloo backend.

The path shards as independent replicas: rank r serves jobs
r, r+G, ... of one global stream with its own queue/feedback/executor and no
data-path collective.  Each rank here runs the host serving loop on its
shard; rank 0 gathers the records (plumbing only) and checks the merged log
against the single-process ``run_replicas`` and the bench aggregation rules
(sum of requests, max of times).
"""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2310_18481_b200 as ms
    p = ms.demo_profile()
    spec = ms.WorkloadSpec(kind="poisson", qps=40, duration_s=6, seed=11, deadline_ms=400)
    jobs = ms.generate_jobs(spec, p)
    m = ms.matrix_for_jobs(p, jobs)
    cfg = ms.SimConfig(profile=p, matrix=m, policy=ms.Policy.OPTIMIZED, seed=1)
    log = ms.run(cfg, jobs[rank::world])
    recs = [((r.id - 1) * world + rank + 1, r.completion_us, r.violated, r.size) for r in log.records]
    gathered = [None] * world
    dist.all_gather_object(gathered, recs)
    ok = torch.tensor([sum(s for *_, v, s in recs if not v)], dtype=torch.float64)
    t = torch.tensor([float(max((c or 0) for _, c, _, _ in recs))], dtype=torch.float64)
    dist.all_reduce(ok, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        merged = sorted(x for g in gathered for x in g)
        ref = ms.run_replicas([cfg] * world, jobs)
        out.put((merged, [(r.id, r.completion_us, r.violated, r.size) for r in ref.records],
                 ok.item(), sum(r.size for r in ref.records if not r.violated), t.item(),
                 max((r.completion_us or 0) for r in ref.records)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, ref, ok, ref_ok, tmax, ref_tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert merged == ref
    assert ok == ref_ok and tmax == ref_tmax
