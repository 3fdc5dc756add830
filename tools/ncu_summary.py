"""Summarise ncu --set full reports (raw page) into a markdown table.

    python tools/ncu_summary.py out.md rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    for d in data:
        yield {h: (v, u) for h, v, u in zip(hdr, d, units)}


def main():
    out = sys.argv[1]
    lines = ["| kernel | " + " | ".join(n for _, n in METRICS) + " |",
             "|---" * (len(METRICS) + 1) + "|"]
    for rep in sys.argv[2:]:
        for d in rows(rep):
            name = d.get("Kernel Name", ("?", ""))[0].split("(")[0]
            cells = []
            for m, _ in METRICS:
                v, u = d.get(m, ("n/a", ""))
                cells.append(f"{v} {u}".strip())
            lines.append(f"| {name} | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
