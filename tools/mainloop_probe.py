"""What bounds the GEMM main loop: dense GEMMs (4 tiles per CTA, long K,
epilogue stores skipped via debug flag 1), single-SM vs CTA pair, BN 64 / 128
/ 256, pipeline depth 2..max (MS_MAX_STAGES).  If TF/s scales with stages the
loop is load-latency bound; flat means MMA- or bandwidth-bound.

    python tools/mainloop_probe.py
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

dev = torch.device("cuda")
e0, e1 = dv.Event(), dv.Event()
K = 4096
for BN in (64, 128, 256):
    M = 148 * 128 * 4
    A = (torch.randn(M, K, device=dev) * 0.1).to(torch.bfloat16)
    W = (torch.randn(BN, K, device=dev) * 0.1).to(torch.bfloat16)
    b = torch.zeros(BN, device=dev)
    D = torch.empty(M, BN, device=dev, dtype=torch.bfloat16)
    for pair in (False, True):
        row = []
        for st in (2, 3, 4, 6, 8, 12):
            os.environ["MS_MAX_STAGES"] = str(st)
            try:
                p = dv.plan_dense(A, W, b, D, BN=BN, relu=True, split_k=1, pair=pair)
            except Exception as ex:  # noqa: BLE001
                row.append(f"{st}:err")
                continue
            dv.check(dv.lib().ms_gemm_plan_debug(p.addr, 1), "debug")
            real = p.info()["stages"]
            for _ in range(3):
                p.run()
            ts = []
            for _ in range(5):
                e0.record()
                for _ in range(5):
                    p.run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_us(e1) / 5)
            t = float(np.median(ts))
            row.append(f"{real}:{2 * M * BN * K / t / 1e6:5.0f}")
        print(f"BN={BN:3d} {'pair  ' if pair else 'single'} stages:TF/s  " + "  ".join(row), flush=True)
os.environ.pop("MS_MAX_STAGES", None)
