"""Summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool)."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
agg = collections.OrderedDict()
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("bm::<unnamed>::", "").replace("void ", "")
    v = float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1)
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{len(data)} launches, {tot/1e6:.2f} ms total device time (serialised, cold-cache)")
print(f"{'ms':>9} {'n':>4} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v[0]/1e6:9.3f} {v[1]:4d} {100*v[0]/tot:5.1f}%  {k}")
