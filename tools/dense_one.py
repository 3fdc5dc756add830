"""One served-shape 28^2 merged 1x1 GEMM (M = 183 * 784, K = 192, N = 224,
bias + ReLU) for an ncu capture:
    ncu --set full -k regex:gemm_tc -s 3 -c 1 python tools/dense_one.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402

M, K, N = 183 * 784, int(sys.argv[1]) if len(sys.argv) > 1 else 192, int(sys.argv[2]) if len(sys.argv) > 2 else 224
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
W = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
b = torch.randn(N, device="cuda") * 0.1
D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
p = dv.plan_dense(A, W, b, D, BN=N, relu=True)
for _ in range(5):
    p.run()
torch.cuda.synchronize()
print("ok", p.info())
