"""Per-CTA timeline of single GEMM launches (ms_gemm_plan_set_trace):
%globaltimer at entry, prologue done, PDL wait done, first TMA issued, first
data ready, last MMA commit, first accumulator ready, epilogue done.  Each
traced op runs in a CUDA graph right after its predecessor op (as in a pass).

    python tools/gemm_trace.py --n 32 --ops 3,20,21,22,47
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--mod", type=int, default=0)
ap.add_argument("--ops", default="3,20,21,22,47")
a = ap.parse_args()
import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

NAMES = ["entry", "prolog", "pdlwait", "tma0", "data0", "lastmma", "acc0", "epi_end", "ldtm0", "cvt0", "store0",
         "tile0end"]
NS = len(NAMES)
m = build_tbn_model(max_req=a.n, n_slots=a.n)
m.use_graphs = False
m.forward(np.arange(a.n), np.full(a.n, 7, dtype=np.int16))
torch.cuda.synchronize()
prog = m.encoders[a.mod].program(a.n)
def trace(i, kind, op, dbg):
    info = op.info()
    buf = torch.zeros(info["grid_x"] * NS, dtype=torch.int64, device="cuda")
    dv.check(dv.lib().ms_gemm_plan_set_trace(op.addr, buf.data_ptr()), "set_trace")
    dv.check(dv.lib().ms_gemm_plan_debug(op.addr, dbg), "debug")
    P = dv.Program()
    P.ops = [prog.ops[i - 1], (kind, op)] if i > 0 else [(kind, op)]
    P.keep = prog.keep
    P.seal()  # copies the plan (trace pointer + debug flags) by value
    dv.check(dv.lib().ms_gemm_plan_set_trace(op.addr, None), "set_trace")
    dv.check(dv.lib().ms_gemm_plan_debug(op.addr, 0), "debug")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.run(s)
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            P.run(s)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    t = buf.view(-1, NS).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)  # us
    span = np.nanmax(rel[:, 7])
    print(f"op {i}: {op.label} grid {info['grid_x']} stages {info['stages']} flops {op.flops / 1e9:.2f} G"
          f" debug {dbg} span {span:.1f} us")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        if np.all(np.isnan(col)):
            continue
        print(f"   {nm:8s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f}")


for i in [int(x) for x in a.ops.split(",")]:
    kind, op = prog.ops[i]
    if kind != "gemm" or getattr(op, "pair", False):
        print(f"op {i}: {kind} (skipped)")
        continue
    for dbg in (0, 1, 2):
        trace(i, kind, op, dbg)
