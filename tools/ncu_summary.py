"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "second": 1e6, "s": 1e6}


def load(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", "ns"), 1e-3)
        name = d["Kernel Name"]
        name = name.split("(")[0].split("::")[-1]
        out.append((name, v))
    return out


if __name__ == "__main__":
    rows = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in rows:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot:.1f} us total")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.1f} us {v[0]:5d}x {v[1] / v[0]:9.2f} us/launch {100 * v[1] / tot:5.1f}%  {k}")
