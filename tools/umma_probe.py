"""Probe: shifted K-major SW128 UMMA A-operand descriptors (base-offset
field) -- the addressing a halo-reusing 3x3 conv would need."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
import _probes  # noqa: E402

g = torch.Generator().manual_seed(0)
A = torch.randn(256, 64, generator=g).to(torch.bfloat16)
W = (torch.randn(64, 64, generator=g) * 0.1).to(torch.bfloat16)
Ad, Wd = A.cuda(), W.cuda()
D = torch.zeros(128, 64, device="cuda")
for sbo in (1024, 1280, 2048):
    for use_base in (0, 1):
        res = []
        for shift in (0, 1, 3, 7, 8, 10, 13):
            dv.check(_probes.lib().ms_debug_umma_shift(Ad.data_ptr(), Wd.data_ptr(), D.data_ptr(), shift, sbo, use_base,
                                                  dv.stream_ptr()), "probe")
            torch.cuda.synchronize()
            # expected: row m reads A row  shift + (m // 8) * (sbo // 128) + m % 8
            rows = torch.tensor([shift + (m // 8) * (sbo // 128) + m % 8 for m in range(128)])
            ok_rows = rows < 256
            ref = A[rows.clamp(max=255)].float() @ W.float().T
            err = (D.cpu() - ref)[ok_rows].abs().max().item()
            res.append(f"s{shift}:{'ok' if err < 1e-2 else 'BAD'}")
        print(f"sbo {sbo} base_offset {'on ' if use_base else 'off'}: " + " ".join(res), flush=True)
