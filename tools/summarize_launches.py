"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel mean
duration and share of the step (our kernels only).  Usage: summarize_launches.py launches.csv"""
import collections
import csv
import json
import sys


def summarize(path):
    hdr, per = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        if "sfa::" not in name:
            continue
        short = name.split("(")[0].replace("sfa::<unnamed>::", "").replace("void ", "").replace("sfa::", "")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
        per.setdefault(short, []).append(float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0))
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot} for k, v in per.items()}


if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1]), indent=1))
