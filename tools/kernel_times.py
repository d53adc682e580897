"""Summarise an ncu launch list (gpu__time_duration.sum) by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1 + skip:]:
    if len(r) > vi:
        k = r[ki].split("(")[0][:70]
        agg[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:15]:
    print(f"{v / 1e3:10.1f} us  {cnt[k]:5d}x  {100 * v / tot:5.1f}%  {k}")
