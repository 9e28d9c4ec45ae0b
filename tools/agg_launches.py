"""Aggregate an ncu --csv gpu__time_duration launch list by kernel name (ms)."""
import collections, csv, sys
agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(d["Metric Unit"], 1e-6)
    k = d["Kernel Name"][:70]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v[1]:9.3f} ms {v[0]:5d}  {k}")
print(f"{tot:9.3f} ms total")
