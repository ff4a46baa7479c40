"""Top stalled SASS lines of one kernel from `ncu --page source --csv` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {c: sum(int(d[c] or 0) for d in data) for c in stall_cols}
print(" ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for d in top:
    st = {c[6:]: int(d[c] or 0) for c in stall_cols if int(d[c] or 0)}
    print(f'{d["Warp Stall Sampling (All Samples)"]:>6} {d["Address"][-5:]} {d["Source"].strip()[:60]:60s} {st}')
