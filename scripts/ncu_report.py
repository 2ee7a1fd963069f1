"""Summarise every kernel of an ncu --set full report into one text file (key counters + stalls).

usage: python scripts/ncu_report.py REPORT.ncu-rep OUT.txt "title"
"""
import csv
import subprocess
import sys

rep, out_path, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
res = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(res.splitlines()))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]
out = [f"# {title}", f"# ncu --set full --clock-control none; report {rep.split('/')[-1]}", ""]
for v in rows[2:]:
    name = v[h.index("Kernel Name")]
    out.append(f"## {name[:160]}")
    for k in keys:
        if k in h:
            i = h.index(k)
            out.append(f"  {k:66s} {v[i]} {units[i]}")
    try:
        dur = float(v[h.index("gpu__time_duration.sum")].replace(",", ""))
        du = units[h.index("gpu__time_duration.sum")]
        mb = sum(float(v[h.index(k)].replace(",", "")) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        scale = {"usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(du, 1e-6)
        out.append(f"  {'achieved DRAM GB/s (read+write / duration)':66s} {mb * 1e6 / (dur * scale) / 1e9:.0f}")
    except (ValueError, KeyError):
        pass
    st = [(k, float(v[i])) for i, k in enumerate(h) if "pcsamp_warps_issue_stalled" in k
          and not k.endswith("not_issued") and v[i].replace(".", "").isdigit() and float(v[i]) > 0]
    tot = sum(x for _, x in st) or 1.0
    out.append("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {x / tot:.0%}"
                                       for k, x in sorted(st, key=lambda t: -t[1])[:6]))
    out.append("")
open(out_path, "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
