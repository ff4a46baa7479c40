"""Compare the per-iteration device checksums ([sums] lines, CMPC_DEBUG_SUMS=1) of concurrent
identical solves: the first (iteration, quantity) where a context differs from the majority."""
import collections
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith("[sums]")]
by_ctx = collections.defaultdict(list)
for l in lines:
    f = l.split()
    by_ctx[f[1]].append((int(f[2]), dict(zip(f[3::2], f[4::2]))))
runs = list(by_ctx.values())
print(len(runs), "contexts,", len(lines), "lines")
n = min(len(r) for r in runs)
for k in range(n):
    for q in ("omega", "M", "rhs", "L", "pv", "ps"):
        vals = collections.Counter(r[k][1][q] for r in runs)
        if len(vals) > 1:
            print(f"record {k} (iter {runs[0][k][0]}): {q} differs: {dict(vals)}")
            sys.exit(0)
print("all equal")
