"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
share, count and mean duration per kernel.  usage: launch_summary.py FILE [TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print(f"| kernel | launches | mean us | share |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {sum(v) / tot * 100:.1f}% |")
