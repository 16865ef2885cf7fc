"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list: per kernel count,
mean and share (development helper)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        try:
            agg[r[ki].split("(")[0].replace("void ", "").split("::")[-1]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:10.3f} us share={sum(v) / tot * 100:5.1f}%")
