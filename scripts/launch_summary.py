"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches and total time per kernel, and each kernel's SHARE of the total
(the cold-cache serialised absolutes are not comparable to bench timings)."""
import csv
import io
import re
import sys
from collections import OrderedDict


def main(path, title=""):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", r["Kernel Name"]).strip()
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r["Metric Unit"], 1e-3)
        us = float(r["Metric Value"].replace(",", "")) * scale
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values()) or 1.0
    if title:
        print(title)
    print("cold-cache serialised launches: compare SHARES, not absolutes")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:60s} launches={n:5d} total={t:11.1f} us  per_launch={t / n:9.1f} us  share={100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
