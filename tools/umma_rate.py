"""Issue rate of back-to-back tcgen05.mma (M=128, K=16, one accumulator)
from one thread, by A-operand layout and width N: clocks per MMA and the
fraction of the dense bf16 tensor peak (8192 flop/clk/SM) it sustains."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_18481_b200 import build  # noqa: E402

build.build()
from paper_2310_18481_b200 import device as dv  # noqa: E402
import _probes  # noqa: E402

cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
names = {0: "SW128", 1: "interleave LBO16/SBO128", 2: "interleave LBO16/SBO112", 3: "interleave LBO128/SBO256"}
for mode in (0, 1, 2, 3):
    for n in (64, 128, 256):
        res = []
        for count in (64, 1024):
            dv.check(_probes.lib().ms_debug_umma_rate(mode, n, count, cyc.data_ptr(), dv.stream_ptr()), "rate")
            torch.cuda.synchronize()
            res.append(int(cyc.item()))
        per = (res[1] - res[0]) / (1024 - 64)
        ideal = 2 * 128 * n * 16 / 8192
        print(f"{names[mode]:26s} N={n:3d}: {per:7.1f} clk/MMA (ideal {ideal:5.1f}) -> {ideal / per:5.1%} of peak;"
              f" latency-ish {res[0] / 64:6.1f} clk/MMA at 64")
