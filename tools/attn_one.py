import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2310_18481_b200 import device as dv
H, L, n = 12, 197, 32
qkv = torch.randn(n * L, 3 * H * 64, device="cuda").to(torch.bfloat16)
out = torch.empty(n * L, H * 64, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    dv.check(dv.lib().ms_attention(qkv.data_ptr(), 3 * H * 64, L, H, n, out.data_ptr(), H * 64, 0.125, dv.stream_ptr()), "a")
torch.cuda.synchronize()
