"""Issue rate of back-to-back tcgen05.mma (M=128, K=16) whose SW128 A
descriptor starts r 128-B rows into the tile (the halo conv's tap views),
and with the 9 tap shifts of a pitch-16 / pitch-32 halo rotating."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
import _probes  # noqa: E402

cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
for mode, name in [(0, "SW128 aligned")] + [(4 + r, f"SW128 +{r} rows") for r in (1, 2, 3, 4, 8, 16, 17)] + \
        [(20, "taps pitch 16"), (21, "taps pitch 32")]:
    for n in (64, 96, 128, 192, 256):
        res = []
        for count in (72, 1080):
            dv.check(_probes.lib().ms_debug_umma_rate(mode, n, count, cyc.data_ptr(), dv.stream_ptr()), "rate")
            torch.cuda.synchronize()
            res.append(int(cyc.item()))
        per = (res[1] - res[0]) / (1080 - 72)
        ideal = 2 * 128 * n * 16 / 8192
        print(f"{name:18s} N={n:3d}: {per:7.1f} clk/MMA (ideal {ideal:5.1f}) -> {ideal / per:5.1%}", flush=True)
