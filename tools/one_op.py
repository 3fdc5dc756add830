"""Run one op of one encoder program (after a warm pass) inside a
cudaProfilerStart/Stop window, for `ncu --profile-from-start off`.

    ncu --profile-from-start off --set full -c 1 -o prof python tools/one_op.py --n 32 --mod 0 --op 20
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--mod", type=int, default=0)
ap.add_argument("--op", type=int, default=20)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mask", type=int, default=7)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.executor import build_tbn_model  # noqa: E402

m = build_tbn_model(max_req=a.n, n_slots=a.n)
m.use_graphs = False
masks = np.full(a.n, a.mask, dtype=np.int16)
m.forward(np.arange(a.n), masks)
torch.cuda.synchronize()
prog = m.encoders[a.mod].program(a.n)
kind, op = prog.ops[a.op]
P = dv.Program()
P.ops = [(kind, op)]
P.keep = prog.keep
P.seal()
P.run()
torch.cuda.synchronize()
print("op", kind, getattr(op, "label", ""), flush=True)
torch.cuda.profiler.start()
for _ in range(a.reps):
    P.run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
