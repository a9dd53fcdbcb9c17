"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    print(f, "total ms", round(s / 1e6, 3))
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
        print(f"  {k:32s} {v / s * 100:6.2f}%  n={cnt[k]:5d}  avg_us={v / cnt[k] / 1e3:9.2f}")
