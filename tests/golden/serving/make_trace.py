"""Writes bursty_trace.csv: a 120 s synthetic request trace in the reference's
trace format (``epoch_seconds,count`` per line, sim.py:92-104) -- a slow
sinusoidal base plus 14 random 1-3 s bursts (seed 2023).  The configs[3]
bench line maps it to [min_qps, max_qps] with map_trace_to_qps (sim.py:
107-125) and searches the peak rate."""
from pathlib import Path

import numpy as np


def main():
    rng = np.random.default_rng(2023)
    t0 = 1_700_000_000
    base = 100 + 20 * np.sin(np.arange(120) / 9.0)
    bursts = np.zeros(120)
    for c in rng.choice(120, 14, replace=False):
        w = int(rng.integers(1, 4))
        bursts[c:c + w] += rng.uniform(60, 140)
    cnt = np.maximum(0, base + bursts + rng.normal(0, 8, 120)).round().astype(int)
    lines = ["# bursty synthetic request trace (epoch_seconds,count): sinusoidal base + 14 random 1-3 s bursts",
             "# made by tests/golden/serving/make_trace.py (seed 2023); map_trace_to_qps scales it"]
    lines += [f"{t0 + i},{c}" for i, c in enumerate(cnt)]
    (Path(__file__).resolve().parent / "bursty_trace.csv").write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
