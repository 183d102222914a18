"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        name = name.replace("void ", "").replace("tf::<unnamed>::", "").replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':60s} {'n':>4s} {'total us':>12s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:60]:60s} {len(v):4d} {sum(v):12.1f} {100 * sum(v) / tot:6.1f}%")
    print(f"{'TOTAL':60s} {'':4s} {tot:12.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
