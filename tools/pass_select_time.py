"""Latency of one ms_pass_select launch (a single formation), CUDA events on
the launching stream: inputs in HBM vs pinned (mapped) host memory, on an
idle GPU and while TBN encoder passes occupy every SM.

    python tools/pass_select_time.py > gpurun_out/pass_select_time.txt
"""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import pass_cases as pc  # noqa: E402
from paper_2310_18481_b200 import build, device as dv  # noqa: E402


def main():
    build.build()
    g = [x for x in pc.groups() if int(x["cfg"][0]) == 96 and int(x["cfg"][1]) > 0][0]
    coff = np.concatenate([[0], np.cumsum(g["n_cand"])[:-1]]).astype(np.int32)
    moff = np.concatenate([[0], np.cumsum(g["n_cand"].astype(np.int64) * g["size"])[:-1]]).astype(np.int32)
    cost = dv.PassCost.make(g["w"], g["u"], g["t"])

    def bufs(pinned):
        def put(a, dt):
            t = torch.as_tensor(np.ascontiguousarray(a)).to(dt)
            return t.pin_memory() if pinned else t.cuda()
        ins = [put(g["job_off"], torch.int32), put(g["n_jobs"], torch.int32), put(g["now"], torch.int64),
               put(g["factor"], torch.float64), put(g["size"], torch.int32), put(g["deadline"], torch.int64),
               put(g["n_cand"], torch.int32), put(coff, torch.int32), put(moff, torch.int32),
               put(g["cand_counts"].reshape(-1), torch.int16), put(g["req_masks"].view(np.int16), torch.int16)]
        outs = [put(np.zeros(len(g["size"]), np.int32), torch.int32),
                put(np.zeros(len(g["job_off"]) * dv.PASS_SUMMARY, np.int32), torch.int32),
                put(np.zeros(len(g["job_off"]), np.int64), torch.int64)]
        return ins, outs

    mask = torch.zeros(len(g["job_off"]), 96, dtype=torch.int16, device="cuda")
    st = torch.cuda.Stream(priority=-1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    probs = [i for i in range(len(g["job_off"])) if g["res_members"][i] >= 4][:200]
    qs = [int(g["n_jobs"][i]) for i in probs]
    print(f"{len(probs)} formations (>= 4 members), queue mean {np.mean(qs):.1f} max {max(qs)}")

    clock = torch.zeros(2, dtype=torch.int64).pin_memory()

    def run(pinned, busy=None):
        ins, outs = bufs(pinned)
        ts = []
        ks = []
        for i in probs:
            p = [t.data_ptr() for t in ins]
            # one problem: offset the per-problem arrays
            p[0] += 4 * i
            p[1] += 4 * i
            p[2] += 8 * i
            p[3] += 8 * i
            if busy is not None:
                busy()
            with torch.cuda.stream(st):
                e0.record(st)
                dv.pass_select(1, *p, cost, 96, int(g["cfg"][1]), outs[0].data_ptr(),
                               outs[1].data_ptr() + 4 * dv.PASS_SUMMARY * i, outs[2].data_ptr() + 8 * i,
                               mask[i].data_ptr(), 96, stream=st, out_clock=clock.data_ptr())
                e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
            ks.append((int(clock[1]) - int(clock[0])) / 1000)
        torch.cuda.synchronize()
        print(f"   kernel-resident (globaltimer): mean {np.mean(ks):.2f} us, p50 {np.median(ks):.2f}, "
              f"p90 {np.percentile(ks, 90):.2f}")
        return np.array(ts)

    for pinned in (False, True):
        t = run(pinned)
        print(f"idle GPU, inputs in {'pinned host' if pinned else 'HBM'}: mean {t.mean():.1f} us, "
              f"p50 {np.median(t):.1f}, p90 {np.percentile(t, 90):.1f}")
    from paper_2310_18481_b200.executor import build_tbn_model
    model = build_tbn_model(max_req=96, n_slots=192)
    model.warm_graphs(96)
    rng = np.random.default_rng(0)
    masks = rng.integers(1, 8, size=96)

    def busy():
        model.forward(rng.integers(0, 192, size=96), masks)  # ~6 ms of encoder work queued

    for pinned in (False, True):
        t = run(pinned, busy)
        print(f"busy GPU (TBN 96-request pass in flight), inputs in {'pinned host' if pinned else 'HBM'}: "
              f"mean {t.mean():.1f} us, p50 {np.median(t):.1f}, p90 {np.percentile(t, 90):.1f}")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def batched():
    """All problems of the group in ONE launch (for ncu source-level stall sampling)."""
    build.build()
    g = [x for x in pc.groups() if int(x["cfg"][0]) == 96 and int(x["cfg"][1]) > 0][0]
    coff = np.concatenate([[0], np.cumsum(g["n_cand"])[:-1]]).astype(np.int32)
    moff = np.concatenate([[0], np.cumsum(g["n_cand"].astype(np.int64) * g["size"])[:-1]]).astype(np.int32)
    cost = dv.PassCost.make(g["w"], g["u"], g["t"])
    put = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
    ins = [put(g["job_off"], torch.int32), put(g["n_jobs"], torch.int32), put(g["now"], torch.int64),
           put(g["factor"], torch.float64), put(g["size"], torch.int32), put(g["deadline"], torch.int64),
           put(g["n_cand"], torch.int32), put(coff, torch.int32), put(moff, torch.int32),
           put(g["cand_counts"].reshape(-1), torch.int16), put(g["req_masks"].view(np.int16), torch.int16)]
    n = len(g["job_off"])
    outs = [put(np.zeros(len(g["size"]), np.int32), torch.int32), put(np.zeros(n * dv.PASS_SUMMARY, np.int32), torch.int32),
            put(np.zeros(n, np.int64), torch.int64)]
    mask = torch.zeros(n, 96, dtype=torch.int16, device="cuda")
    for _ in range(3):
        dv.pass_select(n, *[t.data_ptr() for t in ins], cost, 96, int(g["cfg"][1]), outs[0].data_ptr(),
                       outs[1].data_ptr(), outs[2].data_ptr(), mask.data_ptr(), 96)
    torch.cuda.synchronize()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "batched":
    batched()
