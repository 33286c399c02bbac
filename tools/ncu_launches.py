#!/usr/bin/env python
"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``).

    python tools/ncu_launches.py launches.csv [kernel-substring]

Prints per-kernel launch count, total / average duration and share of the
summed kernel time (ncu times are serialised and cold-cache: compare shares,
not absolute step times).
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def load(path):
    hdr, out = None, []
    with open(path) as fh:
        for r in csv.reader(fh):
            if r and r[0] == "ID":
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    d["us"] = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
                    out.append(d)
    return out


def main():
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rows:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += d["us"]
    tot = sum(v[1] for v in agg.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-64s n=%5d total=%10.1f us avg=%9.2f us share=%5.1f%%"
              % (k[:64], v[0], v[1], v[1] / v[0], 100 * v[1] / tot))
    print("launches %d, summed kernel time %.1f us" % (len(rows), tot))
    if len(sys.argv) > 2:
        for d in rows:
            if sys.argv[2] in d["Kernel Name"]:
                print(d["Kernel Name"][:70], d["Grid Size"], "%.2f us" % d["us"])


if __name__ == "__main__":
    try:
        main()
    except BrokenPipeError:
        pass
