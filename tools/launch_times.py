"""Per-kernel device times of one short command under `ncu --metrics gpu__time_duration.sum` (serialised, cold cache):
python tools/launch_times.py <launches.csv>  ->  name, count, mean us"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
acc = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    name = r[kn].split("(")[0].replace("void unnamed>::", "").replace("unnamed>::", "")
    t = float(r[mv].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[mu], 1.0)
    acc.setdefault(name, []).append(t)
for name, ts in acc.items():
    print(f"{name:60s} n={len(ts):4d} mean {sum(ts) / len(ts):10.2f} us")
