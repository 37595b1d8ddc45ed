"""Summarise a tools/gpu_quick.sh run: tests, step launch list, ncu headline, bench."""
import csv
import json
import subprocess
import sys

T = sys.argv[1] if len(sys.argv) > 1 else "q"
O = "gpurun_out"
print(open(f"{O}/t_{T}.log").read().strip().splitlines()[-2:])
rows = list(csv.reader(open(f"{O}/launch_{T}.csv")))
h = None
out = []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        out.append((int(d["ID"]), d["Kernel Name"][:50], float(d["Metric Value"])))
last = [o for o in out if o[0] >= out[-1][0] - 6]
for o in last:
    print(f"  {o[0]:3d} {o[1]:50s} {o[2] / 1000:8.1f} us")
r = subprocess.run(["ncu", "-i", f"{O}/ncu_{T}.ncu-rep", "--page", "details", "--csv"], capture_output=True, text=True)
rr = list(csv.reader(r.stdout.splitlines()))
if rr:
    hh = rr[0]
    for row in rr[1:]:
        d = dict(zip(hh, row))
        if d.get("Metric Name") in ("Duration", "L1/TEX Hit Rate", "Issue Slots Busy", "Achieved Active Warps Per SM",
                                    "L1/TEX Cache Throughput", "DRAM Throughput", "Registers Per Thread"):
            print("  ncu", d["Metric Name"], d["Metric Value"], d["Metric Unit"])
r = subprocess.run(["ncu", "-i", f"{O}/ncu_{T}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True)
rr = list(csv.reader(r.stdout.splitlines()))
if len(rr) > 2:
    d = dict(zip(rr[0], rr[2]))
    for k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"):
        print("  ncu", k, d.get(k))
try:
    b = json.loads(open(f"{O}/bench_{T}.json").read().strip().splitlines()[-1])
    print("bench value", b["value"], "ms/step", b["ms_per_step"], "gather ms", b["roofline"]["launch_ms"],
          "frac", b["roofline"]["frac"])
except Exception as e:
    print("bench:", open(f"{O}/bench_{T}.json").read()[-800:])
