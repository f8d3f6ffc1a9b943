"""Print an ncu `--metrics gpu__time_duration.sum --csv` launch list as
kernel / microseconds / grid (one line per launch)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "nsecond")
            us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
            print(f"{d['Kernel Name'][:44]:44s} {us:9.1f} us  grid {d.get('Grid Size')}")
