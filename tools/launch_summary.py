"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel count / total / mean, and the first / last launches."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt, seq = defaultdict(float), defaultdict(int), []
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    name = name.replace("void ", "").split("(")[0].split("<")[0]
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
    seq.append((name, v))
for k in sorted(tot, key=lambda k: -tot[k]):
    print("%-40s n=%5d total=%10.1f us mean=%8.2f us" % (k, cnt[k], tot[k], tot[k] / cnt[k]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
print("first:", [(a[:14], round(b, 1)) for a, b in seq[:n]])
print("last:", [(a[:14], round(b, 1)) for a, b in seq[-n:]])
