"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel
(gpu__time_duration.sum is reported in ns; shares are of the summed kernel time)."""
import collections
import csv
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iV:
        continue
    key = re.sub(r"\(.*", "", r[iK]).replace("void ", "").replace("amdp::<unnamed>::", "")
    key = key.replace("unnamed>::", "")
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total_ms':>10s} {'share':>6s} {'avg_us':>8s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {n:8d} {t / 1e6:10.2f} {t / tot:6.3f} {t / n / 1e3:8.2f}")
print(f"total {tot / 1e6:.1f} ms over {sum(v[0] for v in agg.values())} launches")
