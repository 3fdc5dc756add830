"""Per-kernel floor of a dependent op chain in a CUDA graph: R copies of one
op (a late-stage pool, a 1-tile GEMM, a 7x7 conv) back to back, PDL on/off.

    python tools/launch_floor.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

R = 20
m = build_tbn_model(max_req=64, n_slots=64)
m.use_graphs = False
m.forward(np.arange(61), np.full(61, 7, dtype=np.int16))
torch.cuda.synchronize()
prog = m.encoders[0].program(61)
dev = torch.device("cuda")
A = torch.randn(128, 64, device=dev).to(torch.bfloat16)
W = torch.randn(64, 64, device=dev).to(torch.bfloat16)
b = torch.zeros(64, device=dev)
D = torch.empty(128, 64, device=dev, dtype=torch.bfloat16)
tiny = dv.plan_dense(A, W, b, D, BN=64, relu=True)
e0, e1 = dv.Event(), dv.Event()


def chain(ops, keep):
    P = dv.Program()
    P.ops = ops * R
    P.keep = keep
    P.seal()
    P.run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            P.run(s)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    ts = []
    for _ in range(7):
        e0.record()
        g.replay()
        e1.record()
        ts.append(e0.elapsed_us(e1) / R)
    return float(np.median(ts))


cases = [("gemm 1 tile M=128 N=64 K=64", [("gemm", tiny)], [A, W, b, D])]
for i in (48, 53, 54, 45, 46, 44, 21):
    kind, op = prog.ops[i]
    lab = op.label if kind == "gemm" else f"{kind} {op[1:6]}"
    cases.append((f"op {i} {lab}", [(kind, op)], prog.keep))
for pdl in (True, False):
    dv.set_pdl(pdl)
    for lab, ops, keep in cases:
        print(f"pdl={int(pdl)} {chain(ops, keep):7.2f} us/op  {lab}")
dv.set_pdl(True)
