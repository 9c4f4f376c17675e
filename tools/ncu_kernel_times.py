"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` log: per kernel
name, count and mean/min duration in microseconds."""
import csv, collections, re, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i
        break
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) <= iv or not r[iv]:
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("cveb::", "").replace("<unnamed>::", "")
    v = float(r[iv].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
             "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[iu], 1.0)
    agg[name].append(v * scale)
for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
    print(f"{k:45s} n={len(v):5d} mean={sum(v)/len(v):10.2f} us  min={min(v):10.2f} us  total={sum(v)/1e3:9.3f} ms")
