"""Summarise an `ncu --set full` report (or a gpu__time_duration launch list)
into the markdown tables committed under profiles/.

    python profiles/summarize.py full  gpurun_out/prof_r1.ncu-rep  > profiles/r1_ncu_full.md
    python profiles/summarize.py list  gpurun_out/launches.csv     > profiles/r1_launches.md
"""
import collections
import csv
import io
import re
import subprocess
import sys

FULL = [("gpu__time_duration.sum", "time"), ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"), ("dram__bytes_read.sum", "dram rd"),
        ("dram__bytes_write.sum", "dram wr"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def short(name):
    return re.sub(r"\(.*", "", name).replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(h for _, h in FULL) + " |")
    print("|---" * (len(FULL) + 1) + "|")
    for r in rows[2:]:
        cells = []
        for m, _ in FULL:
            if m in hdr:
                i = hdr.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        print(f"| {short(r[hdr.index('Kernel Name')])} | " + " | ".join(cells) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[short(d["Kernel Name"])][0] += 1
            agg[short(d["Kernel Name"])][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | share | avg us |")
    print("|---|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% | {v / c / 1e3:.1f} |")


if __name__ == "__main__":
    (full if sys.argv[1] == "full" else launches)(sys.argv[2])
