"""Per-source-line warp-stall / instruction shares of one kernel in an ncu report.

ncu's CUDA source page carries no metrics for our .so (no embedded source), so
this maps the SASS page's addresses onto source lines with nvdisasm -g of a
locally compiled cubin of the same file (same nvcc, same flags).

  python scripts/ncu_lines.py REPORT.ncu-rep LAUNCH_SKIP csrc/dbscan.cu components_kernelILb0 [N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    rep, skip, src, fn_pat = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
    src = os.path.abspath(src)
    with tempfile.TemporaryDirectory() as td:
        cub = os.path.join(td, "k.cubin")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                        "-std=c++17", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
                        "-cubin", "-o", cub, src], check=True, capture_output=True)
        dis = subprocess.run(["nvdisasm", "-g", cub], check=True, capture_output=True,
                             text=True).stdout
    fn = ln = None
    off2line = {}
    base = os.path.basename(src)
    for l in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        f = re.search(r'File "([^"]+)", line (\d+)', l)
        if f and f.group(1).endswith(base):
            ln = int(f.group(2))
        o = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if o and fn and fn_pat in fn and ln:
            off2line[int(o.group(1), 16)] = ln
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", skip, "--launch-count", "1"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    b0 = int(rows[2][0], 16)
    stall, inst = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        try:
            off = int(r[0], 16) - b0
        except (ValueError, IndexError):
            continue
        L = off2line.get(off, -1)
        stall[L] += float(r[si] or 0)
        inst[L] += float(r[ei] or 0)
    ts, ti = sum(stall.values()) or 1, sum(inst.values()) or 1
    lines = open(src).read().split("\n")
    print(f"{rows[0][1][:100]}")
    print(" line  stall%  inst%  source")
    for L, v in stall.most_common(top):
        s = lines[L - 1].strip()[:80] if L > 0 else "(unmapped)"
        print(f"{L:5d} {100 * v / ts:6.1f} {100 * inst[L] / ti:6.1f}  {s}")


if __name__ == "__main__":
    main()
