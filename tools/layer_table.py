"""Join an ncu launch list (eager profile_pass run) with the pass op list to
get per-launch achieved TFLOP/s.  Usage: layer_table.py launches.csv pass_ops.json [reps]"""
import json
import sys

sys.path.insert(0, "tools")
from launches import load  # noqa: E402

L = [(n.split("(")[0], t) for n, t in load(sys.argv[1]) if n.startswith("mosel::")]
ops = json.load(open(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
per = len(L) // reps
last = L[(reps - 1) * per:]
rows = []
for (kind, label, fl), (kname, ns) in zip(ops, last):
    rows.append((ns / 1e3, kind, label, fl, fl / (ns * 1e-9) / 1e12 if fl else 0.0, kname))
tot = sum(r[0] for r in rows)
gem = [r for r in rows if r[1] == "gemm"]
print(f"pass: {tot:.1f} us total, {len(rows)} launches; GEMM {sum(r[0] for r in gem):.1f} us, "
      f"{sum(r[3] for r in gem) / 1e9:.1f} GFLOP -> {sum(r[3] for r in gem) / (sum(r[0] for r in gem) * 1e-6) / 1e12:.0f} TFLOP/s")
for r in sorted(rows, key=lambda r: -r[0])[:40]:
    print(f"{r[0]:8.1f} us {r[4]:7.1f} TF/s  {r[1]:8s} {r[2]}")
