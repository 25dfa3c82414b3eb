"""Per-kernel summary of an ncu --set full report (dev tool; output -> profiles/).

usage: python scripts/ncu_report.py REPORT.ncu-rep [top_stall_lines]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u = r[0], r[1]
idx = {n: i for i, n in enumerate(h)}
want = [
    ("duration", "gpu__time_duration.sum"),
    ("dram read", "dram__bytes_read.sum"),
    ("dram write", "dram__bytes_write.sum"),
    ("dram throughput % peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 throughput % peak", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput % peak", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe active % (realtime)",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor mem active %", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("issue active %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("warps active % peak", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("registers/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("dyn smem/block", "launch__shared_mem_per_block_dynamic"),
]
for row in r[2:]:
    print("=" * 100)
    print(row[idx["Kernel Name"]][:120])
    for label, m in want:
        if m in idx:
            print(f"  {label:34s} {row[idx[m]]:>16s} {u[idx[m]]}")
    if "dram__bytes_read.sum" in idx:
        def val(m):
            v = float(row[idx[m]].replace(",", ""))
            unit = u[idx[m]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        print(f"  {'dram traffic (read+write) bytes':34s} {val('dram__bytes_read.sum') + val('dram__bytes_write.sum'):16.4e}")
# top stall sites of each kernel (SASS)
for k in range(len(r) - 2):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(k),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    if len(rows) < 3:
        continue
    hdr = rows[1]
    ix = {n: i for i, n in enumerate(hdr)}
    key = "Warp Stall Sampling (All Samples)"
    if key not in ix:
        continue

    def f(v):
        try:
            return float(v)
        except ValueError:
            return None
    # the source page lists each SASS line once per view: keep one copy
    seen, data = set(), []
    for x in rows[2:]:
        if len(x) >= len(hdr) - 1 and f(x[ix[key]]) is not None and tuple(x) not in seen:
            seen.add(tuple(x))
            data.append(x)
    tot = sum(f(x[ix[key]]) for x in data) or 1.0
    stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
    print("=" * 100)
    print("top stall sites:", rows[0][1][:100] if len(rows[0]) > 1 else k)
    for x in sorted(data, key=lambda x: -f(x[ix[key]]))[:top]:
        s = f(x[ix[key]])
        best = sorted(((f(x[ix[n]]) or 0, n) for n in stalls), reverse=True)[:2]
        print(f"  {100 * s / tot:5.1f}%  {x[ix['Source']].strip()[:64]:64s} "
              f"{[(n[6:], int(c)) for c, n in best]}")
