"""Summarise ncu captures from gpurun_out/ into tracked files under profiles/.

  python tools/summarize_profiles.py <round-tag>

* r1_launches_<cfg>.csv  (ncu --metrics gpu__time_duration.sum,dram__bytes_*)
      -> profiles/<tag>_launches_<cfg>.txt: one row per launch (name, us, DRAM MB) and each
         kernel's share of the step
* r1_full_<k>.ncu-rep    (ncu --set full)
      -> profiles/<tag>_full_<k>.txt: duration, DRAM traffic, throughput %, occupancy, issue,
         pipe utilisation, top stall reasons, SASS evidence (UTMALDG/UBLKCP/MATCH)
      -> profiles/<tag>_traffic.json: per-kernel DRAM bytes per launch (bench.py reads this
         for roofline.traffic)
"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag, prefix="r1_launches_"):
    for path in sorted(glob.glob(os.path.join(OUT, prefix + "*.csv"))):
        cfg = path.rsplit("_", 1)[1].split(".")[0]
        rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
        hdr = rows[0]
        ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
        per = defaultdict(dict)
        names = {}
        for r in rows[1:]:
            per[r[iid]][r[im]] = float(r[iv].replace(",", ""))
            names[r[iid]] = r[ik]
        lines = [f"# ncu launch list, config {cfg} (--clock-control none; cold-cache, serialised: compare shares)",
                 f"{'id':>4} {'us':>10} {'DRAM MB':>10}  kernel"]
        tot = defaultdict(float)
        for i in sorted(per, key=int):
            us = per[i].get("gpu__time_duration.sum", 0) / 1e3
            mb = (per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)) / 1e6
            nm = names[i].split("(")[0][:90]
            lines.append(f"{i:>4} {us:>10.2f} {mb:>10.2f}  {nm}")
            tot[nm] += us
        s = sum(tot.values())
        lines.append("")
        lines.append("# share of device time by kernel")
        for nm, us in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append(f"{us / s * 100:6.1f}%  {us:10.2f} us  {nm}")
        open(os.path.join(PROF, f"{tag}_launches_{cfg}.txt"), "w").write("\n".join(lines) + "\n")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def brief(path):
    """Summary lines + traffic dict of one `ncu --set full` report."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        return None, None
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    lines = [f"# ncu --set full --clock-control none: {d.get('Kernel Name', path)}"]
    for key, label in KEYS:
        if key in d:
            lines.append(f"{label:32s} {d[key]} {u.get(key, '')}")
    pipes = {kk.split("pipe_")[1].split(".")[0]: float(v) for kk, v in d.items()
             if kk.startswith("sm__inst_executed_pipe_") and kk.endswith(".avg.pct_of_peak_sustained_active") and v}
    lines.append("pipes (% of peak, active): " + ", ".join(f"{a}={b:.1f}" for a, b in
                                                         sorted(pipes.items(), key=lambda x: -x[1])[:8]))
    st = {kk.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for kk, v in d.items()
          if kk.startswith("smsp__pcsamp_warps_issue_stalled_") and not kk.endswith("not_issued") and v}
    tot = sum(st.values()) or 1
    lines.append("stall samples: " + ", ".join(f"{a}={b / tot * 100:.1f}%" for a, b in
                                              sorted(st.items(), key=lambda x: -x[1])[:8]))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    ev = {m: src.count(m) for m in ("UTMALDG", "UBLKCP", "SYNCS.ARRIVE.TRANS64", "MATCH.ANY", "LDS.128", "DADD")}
    lines.append("SASS evidence (static count in the kernel): " + ", ".join(f"{a}={b}" for a, b in ev.items()))
    traffic = None
    try:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb = float(d["dram__bytes_read.sum"]) * scale.get(u.get("dram__bytes_read.sum", "byte"), 1)
        wb = float(d["dram__bytes_write.sum"]) * scale.get(u.get("dram__bytes_write.sum", "byte"), 1)
        traffic = {"kernel": d.get("Kernel Name", path), "dram_bytes": rb + wb, "read": rb, "write": wb}
    except Exception:
        pass
    return lines, traffic


def full(tag, prefix="r1_full_"):
    traffic = {}
    for path in sorted(glob.glob(os.path.join(OUT, prefix + "*.ncu-rep"))):
        k = path.rsplit(prefix, 1)[1].split(".")[0]
        lines, tr = brief(path)
        if lines is None:
            continue
        open(os.path.join(PROF, f"{tag}_full_{k}.txt"), "w").write("\n".join(lines) + "\n")
        if tr:
            traffic[k] = tr
    json.dump(traffic, open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--brief":  # ad-hoc: print one report's summary
        for path in sys.argv[2:]:
            print("\n".join(brief(path)[0] or [path + ": no data"]) + "\n")
        sys.exit(0)
    tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
    src = sys.argv[2] if len(sys.argv) > 2 else "r1"  # gpurun_out/<src>_launches_*.csv, <src>_full_*.ncu-rep
    os.makedirs(PROF, exist_ok=True)
    launches(tag, src + "_launches_")
    full(tag, src + "_full_")
    print("\n".join(sorted(os.listdir(PROF))))
