"""Summarise an ncu launch list (time + DRAM bytes) of one refine pass."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg.setdefault((r[idi], r[ki].split("(")[0][:60]), {})[r[mi]] = float(r[vi].replace(",", ""))
tot = sum(v.get("gpu__time_duration.sum", 0) for v in agg.values())
print(f"# refine pass: {tot / 1e3:.1f} us over {len(agg)} launches (ncu, serialised)")
byk = collections.defaultdict(lambda: [0.0, 0, 0.0])
for (_, k), v in agg.items():
    b = byk[k]
    b[0] += v.get("gpu__time_duration.sum", 0)
    b[1] += 1
    b[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
for k, (t, c, by) in sorted(byk.items(), key=lambda x: -x[1][0]):
    print(f"{t / 1e3:8.1f} us {c:4d}x {by / 1e9:7.3f} GB {by / (t + 1e-9):7.1f} GB/s  {k}")
