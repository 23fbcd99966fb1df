"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, total and mean device time, share of the total."""
import csv
import sys
from collections import defaultdict


def main(path, skip_prefix=("at::",)):
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':52s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:52]:52s} {c:8d} {t:10.1f} {t / c:9.2f} {t / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
