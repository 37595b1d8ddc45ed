"""Hot SASS blocks of an ncu report (instructions executed, stall samples).
usage: python tools/sass_hot.py report.ncu-rep [min_pct]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
minp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(h) - 1:
        continue
    try:
        data.append((r[0], r[1], float(r[ie] or 0), float(r[ws] or 0)))
    except ValueError:
        pass
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data) or 1
print(f"total warp instructions {tot:.0f}, {len(data)} SASS lines")
blocks = []
cur = None
for a, s, v, st in data:
    if cur is None or abs(v - cur["v"]) > 0.02 * max(v, cur["v"], 1):
        cur = {"start": a, "v": v, "n": 0, "st": 0.0, "ops": collections.Counter()}
        blocks.append(cur)
    cur["n"] += 1
    cur["st"] += st
    cur["ops"][s.split()[1] if s.startswith("@") else s.split()[0]] += 1
for b in sorted(blocks, key=lambda b: -b["v"] * b["n"]):
    share = b["v"] * b["n"] / tot * 100
    if share < minp * 100:
        continue
    print(f"{b['start'][-5:]} n={b['n']:4d} exec/inst={b['v']:.0f} share={share:5.1f}% stall={b['st'] / tst * 100:5.1f}% "
          f"{dict(b['ops'].most_common(8))}")
