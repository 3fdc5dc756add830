"""Offline strategy DP (strategy.py:139-177): host mirror (numpy, as the
reference) vs ms_strategy_dp on the GPU, K=4 synthetic profiles."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_18481_b200 import build  # noqa: E402

build.build()
import torch  # noqa: E402

from paper_2310_18481_b200.planner import DeviceTable, _Table  # noqa: E402
from paper_2310_18481_b200.registry import SynthSpec, synth_profile  # noqa: E402

prof = synth_profile(SynthSpec(n_modalities=4, max_batch=32), 0)
DeviceTable(prof, 8)  # warm (module load, allocator)
for S in (16, 32, 64, 128):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = DeviceTable(prof, S)
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    line = f"S={S:4d} width {d.lat.shape[1]:8d}: device {td * 1e3:9.1f} ms (incl. download of {d.lat.nbytes / 1e6:.0f} MB)"
    if S <= 32:
        t0 = time.perf_counter()
        h = _Table(prof, S)
        th = time.perf_counter() - t0
        assert np.array_equal(d.lat, h.lat) and np.array_equal(d.cnt, h.cnt)
        line += f" | host numpy {th * 1e3:9.1f} ms (identical)"
    print(line, flush=True)
