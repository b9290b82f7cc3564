"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) per kernel: launches, total/avg device time, share of the
step, DRAM bytes per launch.

usage: python tools/launch_summary.py LAUNCHES.csv [OUT.json]
"""
import collections
import csv
import json
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.strip()


def summarise(path):
    rows = collections.defaultdict(dict)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (int(r["ID"]), short(r["Kernel Name"]))
        v = float(r["Metric Value"].replace(",", ""))
        rows[key][r["Metric Name"]] = v
    agg = collections.OrderedDict()
    for (_, k), m in sorted(rows.items()):
        a = agg.setdefault(k, {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["time_ns"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_ns"] for a in agg.values())
    out = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_ns"]):
        out[k] = {"launches": a["launches"], "total_ms": round(a["time_ns"] / 1e6, 3),
                  "avg_us": round(a["time_ns"] / a["launches"] / 1e3, 2),
                  "share": round(a["time_ns"] / total, 4),
                  "dram_bytes_per_launch": int(a["dram_bytes"] / a["launches"]),
                  "dram_GBps": round(a["dram_bytes"] / max(a["time_ns"], 1), 1)}
    return {"total_ms": round(total / 1e6, 3), "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    txt = json.dumps(s, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)
