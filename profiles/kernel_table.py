#!/usr/bin/env python
"""Mean per-launch time of every kernel in an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`).

  python profiles/kernel_table.py gpurun_out/launches.csv [--skip N]
"""
import csv
import io
import sys
from collections import OrderedDict


def table(path, skip=0):
    text = open(path).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(text)))
    per = OrderedDict()
    seen = 0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        seen += 1
        if seen <= skip:
            continue
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        name = r["Kernel Name"].split("(")[0]
        per.setdefault(name, []).append(us)
    total = sum(sum(v) for v in per.values())
    out = []
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append((name, len(v), sum(v) / len(v), sum(v) / total))
    return out


if __name__ == "__main__":
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    print("| kernel | launches | mean us | share |\n|---|---|---|---|")
    for name, n, mean, share in table(sys.argv[1], skip):
        print(f"| `{name}` | {n} | {mean:.1f} | {100 * share:.1f}% |")
