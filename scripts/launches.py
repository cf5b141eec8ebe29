"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("kb::<unnamed>::", "")[:60]
    agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")) / 1000.0)
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v):9.2f} us  {k}")
