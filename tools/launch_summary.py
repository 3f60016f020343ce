"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, mean duration and share of device time per kernel.

  python tools/launch_summary.py launches.csv [title]
"""
import csv
import sys
from collections import defaultdict


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "nsecond")
            us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
            agg[d["Kernel Name"]].append(us)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    if title:
        print(title)
    print("cold-cache serialised launches (ncu replays each kernel alone): compare SHARES, not absolute times")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} launches  mean {sum(v) / len(v):9.2f} us  share {100 * sum(v) / tot:5.1f}%  {name[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
