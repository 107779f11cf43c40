"""Mean device time per kernel name from an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:72]].append(float(d["Metric Value"].replace(",", "")))
    print(f"== {path}")
    for k, v in agg.items():
        print(f"{len(v):4d} x {sum(v) / len(v) / 1000:9.2f} us  {k}")
