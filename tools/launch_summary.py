"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import collections
import csv
import sys


def main(path, only_pgb=True):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        if only_pgb and "pgb" not in k and "CUB" not in k:
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(d["Metric Unit"], 1e-6)
        agg.setdefault(k, [0.0, 0])
        agg[k][0] += v
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"{'ms':>10s} {'n':>5s} {'share':>6s}  kernel")
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{v:10.3f} {n:5d} {v / tot * 100:5.1f}%  {k[:90]}")
    print(f"{tot:10.3f} total")


if __name__ == "__main__":
    main(sys.argv[1])
