"""configs[4]: 4-modality synthetic sweep — batch 1..1024, masks uniform over
all 15 modality subsets — of the HBM-bound hot-path kernels vs the HBM
roofline:

* policy step (ms_policy_select): N jobs x C=16 candidates;
  bytes = N * (12 C + 16)
* compaction (ms_compact: index + 4 gathers) in two regimes:
  "feat" = 1024-d bf16 feature rows (2 KB, latency regime),
  "clip" = TBN-clip-sized rows (rgb 3x224x224x3 bf16, 903 KB, HBM regime);
  bytes = sum over present (request, modality) of row read + row write
          + 2N (masks) + 4 sum N_k (indices)
* fusion (masked concat FC1 4x1024->512 + head 512->397):
  bytes = sum present 1024*2 + N*397*4 + weight bytes

Each point: CUDA-event median over reps after warm-up.  Writes
gpurun_out/c5_sweep.json and a markdown table.

    python tools/sweep_c5.py [--max-n 1024]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--max-n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import FusionHead  # noqa: E402

peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
    else {"hbm_gbs": 6650.0}
HBM = peaks["hbm_gbs"]
K = 4
L = dv.lib()
e0, e1 = dv.Event(), dv.Event()


def timed(fn, reps=a.reps, inner=20):
    """Device time per launch: ``inner`` launches captured in one CUDA graph,
    replayed between two events (no host enqueue gaps), median over reps."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(inner):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / inner)
    return float(np.median(ts))


Ns = [1 << i for i in range(0, int(np.log2(a.max_n)) + 1)]
rng = np.random.default_rng(0)
out = {"hbm_gbs": HBM, "policy": [], "compact_feat": [], "compact_clip": [], "fusion": []}

# ---------------------------------------------------------------- policy
C = 16
for n in Ns:
    lat = np.sort(rng.integers(1_000, 200_000, size=(n, C)), axis=1).astype(np.int64) + np.arange(C)
    lat_d = torch.as_tensor(lat).cuda()
    nc = torch.full((n,), C, dtype=torch.int32, device="cuda")
    dl = torch.as_tensor(rng.integers(0, 300_000, size=n).astype(np.int64)).cuda()
    ch = torch.empty(n, dtype=torch.int32, device="cuda")
    us = timed(lambda: L.ms_policy_select(lat_d.data_ptr(), None, nc.data_ptr(), C, dl.data_ptr(), 0, 1.0, n,
                                          ch.data_ptr(), dv.stream_ptr()))
    b = n * (12 * C + 16)
    out["policy"].append({"n": n, "us": us, "bytes": b, "gbs": b / us / 1e3, "frac": b / us / 1e3 / HBM})


# ------------------------------------------------------------ compaction
def compaction(regime, row_elems):
    slots = min(a.max_n, 1024)
    pools = [torch.randn(slots, row_elems, device="cuda").to(torch.bfloat16) for _ in range(K)]
    dst = [torch.empty(a.max_n, row_elems, dtype=torch.bfloat16, device="cuda") for _ in range(K)]
    X = (ctypes.c_void_p * K)(*[p.data_ptr() for p in pools])
    G = (ctypes.c_void_p * K)(*[d.data_ptr() for d in dst])
    rows = (dv.RowDesc * K)(*[dv.RowDesc(1, 1, row_elems, row_elems, 0) for _ in range(K)])
    idx = torch.empty(K * a.max_n, dtype=torch.int32, device="cuda")
    inv = torch.empty(K * a.max_n, dtype=torch.int32, device="cuda")
    cnt = torch.empty(K, dtype=torch.int32, device="cuda")
    offs = torch.empty((1 << K) + 1, dtype=torch.int32, device="cuda")
    perm = torch.empty(a.max_n, dtype=torch.int32, device="cuda")
    res = []
    for n in Ns:
        masks = rng.integers(1, 16, size=n).astype(np.int16)
        m_d = torch.as_tensor(masks).cuda()
        sl = torch.as_tensor(rng.integers(0, slots, size=n).astype(np.int32)).cuda()
        us = timed(lambda: L.ms_compact(m_d.data_ptr(), n, K, X, rows, sl.data_ptr(), G, idx.data_ptr(),
                                        inv.data_ptr(), cnt.data_ptr(), offs.data_ptr(), perm.data_ptr(),
                                        dv.stream_ptr()))
        present = sum(int(((masks.astype(np.int64) >> k) & 1).sum()) for k in range(K))
        b = present * row_elems * 2 * 2 + 2 * n + 4 * present
        res.append({"n": n, "us": us, "bytes": b, "gbs": b / us / 1e3, "frac": b / us / 1e3 / HBM,
                    "row_bytes": row_elems * 2})
    del pools, dst
    torch.cuda.empty_cache()
    return res


out["compact_feat"] = compaction("feat", 1024)
out["compact_clip"] = compaction("clip", 3 * 224 * 224 * 3)

# ----------------------------------------------------------------- fusion
head = FusionHead(K, a.max_n, 499, 1024)
feats = [torch.randn(a.max_n, 1024, device="cuda").to(torch.bfloat16) for _ in range(K)]
wbytes = head.w1.numel() * 2 + head.w2.numel() * 2 + (head.b1.numel() + head.b2.numel()) * 4
for n in Ns:
    masks = rng.integers(1, 16, size=n)
    inv = torch.full((K, n), -1, dtype=torch.int32)
    for k in range(K):
        sel = np.flatnonzero((masks >> k) & 1)
        inv[k, sel] = torch.arange(len(sel), dtype=torch.int32)
    inv = inv.cuda()
    prog = head.program(n, feats, inv)
    us = timed(prog.run)
    present = sum(int(((masks >> k) & 1).sum()) for k in range(K))
    b = present * 1024 * 2 + n * head.n_classes * 4 + wbytes
    out["fusion"].append({"n": n, "us": us, "bytes": b, "gbs": b / us / 1e3, "frac": b / us / 1e3 / HBM,
                          "tflops": head.flops(n) / us / 1e6})

Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/c5_sweep.json").write_text(json.dumps(out, indent=1))
lines = [f"# configs[4] C5 sweep (K=4, masks uniform over 15 combos), HBM peak {HBM:.0f} GB/s (measured)", ""]
for key in ("policy", "compact_feat", "compact_clip", "fusion"):
    lines += [f"## {key}", "", "| N | us | MB | GB/s | frac of HBM |", "|---|---|---|---|---|"]
    for r in out[key]:
        lines.append(f"| {r['n']} | {r['us']:.1f} | {r['bytes'] / 1e6:.3f} | {r['gbs']:.1f} | {r['frac']:.3f} |")
    lines.append("")
Path("gpurun_out/c5_sweep.md").write_text("\n".join(lines))
print("\n".join(lines))
