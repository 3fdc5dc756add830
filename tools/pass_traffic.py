"""DRAM traffic and per-launch times of ONE served-mix TBN pass (graphs,
modality streams, exactly as serving runs it), captured by ncu between
cudaProfilerStart/Stop:

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/pass_traffic.csv python tools/pass_traffic.py
    python tools/pass_traffic.py --summarize gpurun_out/pass_traffic.csv > profiles/r02_pass_traffic.json
"""
import collections
import csv
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
COUNTS = (61, 36, 24)


def run():
    import torch
    from paper_2310_18481_b200 import build
    build.build()
    from paper_2310_18481_b200.executor import build_tbn_model
    m = build_tbn_model(max_req=96, n_slots=192)
    n = max(COUNTS)
    rng = np.random.default_rng(0)
    masks = np.zeros(n, dtype=np.int16)
    for k, c in enumerate(COUNTS):
        masks[rng.permutation(n)[:c]] |= 1 << k
    masks[masks == 0] = 1
    assert m.counts_for(masks) == COUNTS, m.counts_for(masks)
    for _ in range(3):
        m.forward(rng.integers(0, 192, size=n), masks)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    m.forward(rng.integers(0, 192, size=n), masks)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(json.dumps({"counts": COUNTS, "flop": m.flops(masks)}))


def summarize(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ii, ki, mi, vi, ui = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3,
             "ms": 1e6, "msecond": 1e6}
    for r in data:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        names[r[ii]] = r[ki].split("(")[0]
    tot_b = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
    tot_t = sum(v.get("gpu__time_duration.sum", 0) for v in per.values())
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, v in per.items():
        x = by[names[i]]
        x[0] += 1
        x[1] += v.get("gpu__time_duration.sum", 0)
        x[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    out = {"counts": list(COUNTS), "launches": len(per), "dram_bytes": int(tot_b),
           "serialized_kernel_ns": int(tot_t), "source": "ncu --profile-from-start off, one served-mix pass",
           "by_kernel": {k: {"n": n, "ns": int(t), "dram_bytes": int(b)}
                         for k, (n, t, b) in sorted(by.items(), key=lambda kv: -kv[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarize":
        summarize(sys.argv[2])
    else:
        run()
