"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
kn, mv = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > mv:
        d[r[kn][:70]].append(float(r[mv].replace(",", "")))
for k, v in d.items():
    print(f"{len(v):4d} x {sum(v) / len(v) / 1000:10.1f} us  {k}")
