"""Per-tile timeline of the fused stem kernel (CTA 0, first 32 tiles):
producer issue / MMA ready / MMA issued / epilogue ready / epilogue done
(%globaltimer ns, relative to tile 0's MMA start).  Used to find that the
one-conv-row-per-handshake version was bound by the issuing warp's control
path (per-unit integer division, a lane-0 branch around every MMA), not by
the tensor core: 122 -> 85 us for 192 rgb frames."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
from paper_2310_18481_b200.encoders import pack_stem_weight  # noqa: E402

n, H = 192, 224
X = torch.randn(n, H + 6, H + 6, 4, device="cuda").to(torch.bfloat16)
w = (torch.randn(64, 3, 7, 7) * 0.05).to(torch.bfloat16)
b = torch.zeros(64, device="cuda")
Y = torch.empty(n * 56 * 56, 64, device="cuda", dtype=torch.bfloat16)
p = dv.plan_stem_pool(X, n, H, H, 7, 3, pack_stem_weight(w).cuda(), b, Y, ldy=64)
tr = torch.zeros(32 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    p.run()
dv.check(dv.lib().ms_gemm_plan_set_trace(p.addr, tr.data_ptr()), "trace")
p.run()
torch.cuda.synchronize()
t = tr.cpu().reshape(32, 8)
t0 = int(t[0, 0])
prev = None
for k in range(32):
    r = [(int(x) - t0) for x in t[k]]
    d = "" if prev is None else f"  dMMA {r[0] - prev[0]:5d}  dEPI {r[3] - prev[3]:5d}"
    print(f"tile {k:2d}: prod {r[4]:6d} mma_ready {r[0]:6d} issued {r[1]:6d} "
          f"epi_ready {r[2]:6d} epi_done {r[3]:6d}{d}")
    prev = r
