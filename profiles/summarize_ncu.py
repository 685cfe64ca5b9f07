#!/usr/bin/env python
"""Summarise ncu output into profiles/ (committed evidence).

  python profiles/summarize_ncu.py --launches gpurun_out/launches_rNN.csv \
      --full gpurun_out/prof_gemm_rNN.ncu-rep --tag rNN

Writes profiles/ncu_<tag>.md (launch list shares + full-capture metrics) and
profiles/ncu_gemm_summary.json (dram bytes per GEMM launch, read by bench.py
for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % (elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            ns = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            ns *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
            out.append((d["Kernel Name"].split("(")[0], ns))
    return out


def read_full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        m = OrderedDict(kernel=d.get("Kernel Name", "").split("(")[0])
        for key, label in FULL_METRICS:
            if key in d:
                m[label] = (d[key], units[hdr.index(key)])
        res.append(m)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [f"# ncu summary {a.tag}", "", a.note, ""]
    summary = {"source": f"profiles/ncu_{a.tag}.md"}
    if a.launches:
        launches = read_launches(a.launches)
        tot = {}
        cnt = {}
        for name, ns in launches:
            tot[name] = tot.get(name, 0.0) + ns
            cnt[name] = cnt.get(name, 0) + 1
        all_ns = sum(tot.values())
        lines += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised)", "",
                  "| kernel | launches | mean us | share of step |", "|---|---|---|---|"]
        for name in sorted(tot, key=lambda n: -tot[n]):
            lines.append(f"| `{name}` | {cnt[name]} | {tot[name] / cnt[name] / 1e3:.1f} | {tot[name] / all_ns:.1%} |")
        lines.append("")
    if a.full:
        full = read_full(a.full)
        lines += ["## `--set full` capture of the top kernel", ""]
        per = []
        for m in full:
            lines.append(f"### `{m['kernel']}`")
            for k, v in m.items():
                if k != "kernel":
                    lines.append(f"- {k}: {v[0]} {v[1]}")
            lines.append("")
            rd = float(m["DRAM read"][0].replace(",", "")) * TO_BYTES.get(m["DRAM read"][1], 1)
            wr = float(m["DRAM write"][0].replace(",", "")) * TO_BYTES.get(m["DRAM write"][1], 1)
            per.append(rd + wr)
        summary["dram_bytes_per_launch"] = per
        summary["dram_bytes_per_step"] = sum(per)
    with open(os.path.join(HERE, f"ncu_{a.tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.full:
        with open(os.path.join(HERE, "ncu_gemm_summary.json"), "w") as f:
            json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
