"""Dense 1x1 GEMMs of the served TBN pass and the VQA towers: single-CTA plan
(as auto-selected without pairs) vs the same plan on CTA pairs, warm.

    python tools/pair_sweep.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pick_bn  # noqa: E402

e0, e1 = dv.Event(), dv.Event()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_us(e1) / reps


shapes = [(183 * 784, 192, 224, 1), (183 * 784, 256, 256, 1), (108 * 784, 192, 224, 1), (183 * 196, 576, 512, 1),
          (108 * 196, 576, 512, 1), (183 * 196, 576, 320, 1), (183 * 49, 1024, 832, 1), (183 * 49, 1024, 736, 1),
          (18912, 768, 3072, 2), (18912, 3072, 768, 0), (18912, 768, 2304, 0), (18912, 768, 768, 0)]
for M, K, N, act in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda") * 0.1
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    BN = pick_bn(N)
    fl = 2 * M * N * K
    p0 = dv.plan_dense(A, W, b, D, BN=BN, act=act, pair=False)
    p1 = dv.plan_dense(A, W, b, D, BN=BN, act=act, pair=True)
    pa = dv.plan_dense(A, W, b, D, BN=BN, act=act)
    t0, t1 = t(p0.run), t(p1.run)
    auto = "pair" if pa.info()["grid_x"] == p1.info()["grid_x"] and p1.info()["stages"] == pa.info()["stages"] else "single"
    print(f"M={M:6d} K={K:4d} N={N:4d} act={act} BN={BN}: single {t0:6.1f} us {fl / t0 / 1e6:5.0f} TF/s "
          f"(g{p0.info()['grid_x']} st{p0.info()['stages']}) | pair {t1:6.1f} us {fl / t1 / 1e6:5.0f} TF/s x{t0 / t1:4.2f} "
          f"| auto: {auto}", flush=True)
