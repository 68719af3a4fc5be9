"""Per-CUDA-source-line share of executed warp instructions (or stall samples) of one ncu
report.   python tools/ncu_lines.py <report.ncu-rep> [top] [inst|stall]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
col = 7 if len(sys.argv) <= 3 else {"inst": 7, "stall": 4}[sys.argv[3]]  # column: executed inst | stall samples
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, agg = None, None, {}
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        agg[(cur, int(r[0]), r[1][:80])] = int(r[col])
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total", "warp instructions" if col == 7 else "stall samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot * 100:5.1f}% {v:>11} {k[0]}:{k[1]} {k[2]}")
