"""Summarise ncu reports / launch lists into markdown for profiles/.
usage: python tools/summarize_ncu.py out.md rep1.ncu-rep [rep2 ...] [--launches launches.csv]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def main():
    args = sys.argv[1:]
    out = args.pop(0)
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        del args[i:i + 2]
    lines = []
    for rep in args:
        for hdr, units, r in raw(rep):
            name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            lines.append(f"### `{name[:100]}`  ({rep.split('/')[-1]})\n")
            lines.append("| metric | value | unit |\n|---|---|---|")
            for key, label in METRICS:
                if key in hdr:
                    i = hdr.index(key)
                    lines.append(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")
            stalls = []
            for i, k in enumerate(hdr):
                if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and r[i]:
                    try:
                        stalls.append((float(r[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            tot = sum(v for v, _ in stalls) or 1
            lines.append("\nTop stall reasons (PC samples): " +
                         ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in stalls[:6]) + "\n")
    if launches:
        rows = list(csv.reader(open(launches)))
        h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[h]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = defaultdict(list)
        for r in rows[h + 1:]:
            agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
        total = sum(sum(v) for v in agg.values())
        lines.append(f"### launch list `{launches.split('/')[-1]}` (cold-cache, serialised; compare shares)\n")
        lines.append("| kernel | launches | mean ns | share |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.0f} | {100 * sum(v) / total:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
