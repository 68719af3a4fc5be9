"""Per-SASS-instruction shared-memory wavefronts of one ncu report (bank-conflict hunting).
   python tools/ncu_smem.py <report.ncu-rep> [top]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[start]
ci, wi, ii = hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("L1 Wavefronts Shared"), hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[start + 1:]:
    try:
        data.append((int(r[wi]), int(r[ci]), r[0][-5:], r[1][:60], int(r[ii]), int(r[si])))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total shared wavefronts", tot, "excessive", sum(d[1] for d in data))
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{d[0] / tot * 100:5.1f}% excess {d[1] / max(1, d[0]) * 100:4.0f}% {d[2]} {d[3]} inst={d[4]} "
          f"wf/inst={d[0] / max(1, d[4]):.1f} stall={d[5]}")
