"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per kernel, launches and the
last and the longest launch's duration (us).  python scripts/launch_table.py gpurun_out/launches_X.csv [...]"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg.setdefault(d["Kernel Name"].split("(")[0][:60], []).append(float(d["Metric Value"].replace(",", "")))
    print(path)
    for k, v in agg.items():
        print(f"  {k:60s} n={len(v):3d} last={v[-1] / 1e3:9.1f} us  max={max(v) / 1e3:9.1f} us")
