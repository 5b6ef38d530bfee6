"""Aggregate ncu per-instruction warp-stall samples of one kernel by CUDA source
line, using the line table that `nvdisasm -g` prints for the kernel's cubin.

    python profiles/stall_by_line.py <report.ncu-rep> <kernel regex> <object.o> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, kernel_re):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    table, cur, infn, loc = {}, None, False, None
    for ln in dis.splitlines():
        m = re.match(r"^(\S+):\s*$", ln)
        if m and not ln.startswith("."):
            infn = re.search(kernel_re, m.group(1)) is not None
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and loc:
            table[int(m.group(1), 16)] = loc
    return table


def main():
    rep, kre, obj = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(obj, kre)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    seen, data = set(), []
    for r in rows[2:]:
        if r[0] in seen or not r[0].startswith("0x"):
            continue
        seen.add(r[0])
        data.append((int(r[0], 16), int(r[i_s] or 0), r[1]))
    base = min(a for a, _, _ in data)
    agg = collections.Counter()
    for a, n, _ in data:
        agg[table.get(a - base, ("?", 0))] += n
    tot = sum(agg.values())
    src = {}
    for (f, l), n in agg.most_common(top):
        print(f"{n:7d} {100 * n / tot:5.1f}%  {f}:{l}")
    print("total samples", tot)


if __name__ == "__main__":
    main()
