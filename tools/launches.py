"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, launches and mean/total device time.
    python tools/launches.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i0]
d = collections.OrderedDict()
for r in rows[i0 + 1:]:
    if len(r) < len(h):
        continue
    rec = dict(zip(h, r))
    if rec["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(rec["Metric Value"].replace(",", ""))
    unit = rec["Metric Unit"]
    v = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    name = rec["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    d.setdefault(name, []).append(v)
tot = sum(sum(v) for v in d.values())
for k, v in d.items():
    print(f"{len(v):5d}  mean {sum(v) / len(v):9.4f} ms  total {sum(v):9.3f} ms  {100 * sum(v) / tot:5.1f}%  {k}")
