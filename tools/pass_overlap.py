"""Is a served-mix pass throughput- or latency-bound?  Device time of each
modality's encoder graph alone (served counts 61/36/24), of pairs run
concurrently, and of the whole pass (compaction + 3 encoders + head).

    python tools/pass_overlap.py
"""
import itertools
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=96, n_slots=192)
e0, e1 = dv.Event(), dv.Event()
counts = (61, 36, 24)
n = 61
rng = np.random.default_rng(0)
masks = np.zeros(n, dtype=np.int16)
for k, c in enumerate(counts):
    masks[rng.permutation(n)[:c]] |= 1 << k
masks[masks == 0] = 1
slots = np.arange(n)
for _ in range(3):
    m.forward(slots, masks)
torch.cuda.synchronize()
graphs = {k: m._graph(("enc", k, counts[k]), m.encoders[k].program(counts[k]).run) for k in range(3)}
main = torch.cuda.current_stream()


def run_set(ks):
    ev = dv.Event()
    ev.record()
    evs = []
    for k in ks:
        side = m._side[k]
        side.wait_event(m._ev_c) if False else None
        side.wait_stream(main)
        with torch.cuda.stream(side):
            graphs[k].replay()
        x = torch.cuda.Event()
        x.record(side)
        evs.append(x)
    for x in evs:
        main.wait_event(x)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_us(e1))
    return float(np.median(ts))


names = ("rgb", "flow", "audio")
for r in (1, 2, 3):
    for ks in itertools.combinations(range(3), r):
        t = timed(lambda: run_set(ks))
        print(f"{'+'.join(names[k] for k in ks):16s} {t:8.1f} us", flush=True)
print(f"{'whole pass':16s} {timed(lambda: m.forward(slots, masks)):8.1f} us")
