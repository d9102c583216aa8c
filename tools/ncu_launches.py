"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt, seq = collections.defaultdict(float), collections.Counter(), []
for r in data:
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    name = r[ki].split("(")[0].replace("void ", "")[:48]
    tot[name] += us
    cnt[name] += 1
    seq.append((name, us))
T = sum(tot.values())
print(f"{'total us':>10} {'share':>6} {'n':>5}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} {100 * v / T:5.1f}% {cnt[k]:5d}  {k}")
if len(sys.argv) > 2:
    for name, us in seq[: int(sys.argv[2])]:
        print(f"{us:9.1f} us  {name}")
