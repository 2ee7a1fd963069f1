"""Write the committed profiling evidence under profiles/ from a gpurun capture.

usage: python scripts/profile_summary.py TAG ROUND
  reads gpurun_out/launches_TAG.csv (ncu --metrics gpu__time_duration.sum launch list of bench.py) and
  gpurun_out/prof_TAG.ncu-rep (ncu --set full of the k_stencil kernels); writes
  profiles/ROUND_launches.txt, profiles/ROUND_ncu_<kernel>.txt and profiles/ncu_summary.json (per-apply
  DRAM traffic of the matrix-free apply, read by bench.py's roofline.traffic).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], sys.argv[2]
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

# ---- launch list
rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv"))))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
         f"`python bench.py --steps 5 --warmup 1 --no-cpu --e2e-steps 1` (capture {tag}).",
         "# Cold-cache, serialised per-launch times: compare shares, not absolutes.",
         f"{'kernel':60s} {'n':>5s} {'mean_us':>10s} {'total_us':>11s} {'share':>7s}"]
for k, v in agg.items():
    lines.append(f"{k[-60:]:60s} {len(v):5d} {sum(v)/len(v):10.2f} {sum(v):11.1f} {sum(v)/tot:7.1%}")
open(os.path.join(out_dir, f"{rnd}_launches.txt"), "w").write("\n".join(lines) + "\n")


def page(rep, kern, p):
    res = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", "-k", f"regex:{kern}"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(res.splitlines()))


rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
summary = {}
traffic = 0.0
for kern in ["k_stencil_tma", "k_stencil_main", "k_stencil_items"]:
    raw = page(rep, kern, "raw")
    if len(raw) < 3:
        continue
    hh, units, v = raw[0], raw[1], raw[2]
    name = v[hh.index("Kernel Name")] if "Kernel Name" in hh else kern
    rec = {}
    out = [f"# ncu --set full --clock-control none ({tag}): {name}", ""]
    for k in keys:
        if k in hh:
            i = hh.index(k)
            rec[k] = v[i]
            out.append(f"{k:70s} {v[i]} {units[i]}")
    st = [(k, float(v[i])) for i, k in enumerate(hh) if "pcsamp_warps_issue_stalled" in k
          and not k.endswith("not_issued") and v[i].replace(".", "").isdigit() and float(v[i]) > 0]
    s_tot = sum(x for _, x in st) or 1.0
    out.append("")
    out.append("warp stall sampling:")
    for k, x in sorted(st, key=lambda t: -t[1])[:10]:
        out.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {x / s_tot:6.1%}")
    open(os.path.join(out_dir, f"{rnd}_ncu_{kern}.txt"), "w").write("\n".join(out) + "\n")

    def num(k):
        try:
            return float(rec.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    mb = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")  # MB as reported by ncu
    traffic += mb * 1e6
    summary[kern] = {"duration_us": num("gpu__time_duration.sum"), "dram_MB": mb}
js_path = os.path.join(out_dir, "ncu_summary.json")
js = json.load(open(js_path)) if os.path.exists(js_path) else {}
js["n128"] = {"round": rnd, "capture": tag, "kernels": summary, "dram_bytes_per_apply": traffic,
              "note": "sum over the apply's kernels of dram__bytes_read.sum + dram__bytes_write.sum from one "
                      "ncu --set full capture (cold cache; writes still resident in L2 at kernel end are not counted)"}
json.dump(js, open(js_path, "w"), indent=1)
print(json.dumps(js["n128"], indent=1))
