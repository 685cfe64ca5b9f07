"""Print kernel name + metric values from `ncu --csv` output on stdin (one line per launch)."""
import csv
import sys

label = sys.argv[1] if len(sys.argv) > 1 else ""
rows = [r for r in csv.reader(sys.stdin) if r]
hdr = None
per = {}
for r in rows:
    if r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"][:34])
    per.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, k), m in per.items():
    print(label, k, " ".join(f"{n.split('.')[0]}={v}" for n, v in sorted(m.items())))
