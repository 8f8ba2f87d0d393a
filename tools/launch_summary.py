"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
total / count / mean per kernel, ms."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}[d["Metric Unit"]]
    name = d["Kernel Name"][:70]
    tot[name] += v * scale
    cnt[name] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v:9.3f} ms {cnt[k]:6d} x {1e3 * v / cnt[k]:8.1f} us  {k}")
print(f"{sum(tot.values()):9.3f} ms total, {sum(cnt.values())} launches")
