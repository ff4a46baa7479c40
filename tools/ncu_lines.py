"""Warp-stall samples per CUDA source line of one kernel:
ncu -i report.ncu-rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur, agg, hdr = None, {}, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].strip():
        continue
    try:
        samples = int(r[4] or 0)
    except ValueError:
        continue
    key = (cur, r[0])
    agg.setdefault(key, [0, r[1]])
    agg[key][0] += samples
print("total samples", sum(v[0] for v in agg.values()))
for (f, line), (n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{n:6d} {f}:{line:<5} {src.strip()[:90]}")
