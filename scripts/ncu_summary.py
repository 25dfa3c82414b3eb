"""Summarise an ncu report: key metrics + top stall sites (dev tool)."""
import csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct", "tensor_subpipe_imma_cycles_active_realtime",
        "sm__inst_executed.sum.per_cycle_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
for i, name in enumerate(h):
    if any(name == w or name.startswith(w) for w in want) and not name.endswith((".max", ".min")):
        print(f"{name:80s} {u[i]:>10s} {v[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
idx = {n: i for i, n in enumerate(hdr)}
data = rows[2:]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[idx[key]] or 0) for x in data)
stalls = [n for n in hdr if n.startswith("stall_") and "Not Issued" not in n]
print("stall samples", tot)
for x in sorted(data, key=lambda x: -float(x[idx[key]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    s = float(x[idx[key]] or 0)
    top = sorted(((float(x[idx[n]] or 0), n) for n in stalls), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {x[idx['Source']][:70]:70s} {[(n[6:], int(c)) for c, n in top]}")
