"""Top CUDA source lines of a k_qfit capture by warp-stall samples
(ncu -i REP --page source --csv --print-source cuda,sass) as markdown."""
import csv
import subprocess
import sys


def top(rep, k=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    R = [r for r in rows[3:] if len(r) > 7 and r[2] == "-" and r[4].strip().isdigit()]
    tot = sum(int(r[4]) for r in R)
    lines = [f"| line | stall samples | warp inst | source |", "|---|---|---|---|"]
    for r in sorted(R, key=lambda r: -int(r[4]))[:k]:
        src = r[1].strip()[:100].replace("|", "\\|")
        lines.append(f"| {r[0]} | {int(r[4]) / tot * 100:.1f}% | {r[7]} | `{src}` |")
    return tot, "\n".join(lines)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        tot, md = top(rep)
        print(f"### {rep.split('/')[-1]} ({tot} samples)\n\n{md}\n")
