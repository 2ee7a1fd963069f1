"""Summarise one kernel of an ncu --set full report: key metrics, stall reasons, hottest SASS lines."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 20


def page(p):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", "-k", f"regex:{kern}"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(out.splitlines()))


raw = page("raw")
h, v = raw[0], raw[2]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
st = [(k, float(v[i])) for i, k in enumerate(h) if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")
      and v[i].replace(".", "").isdigit() and float(v[i]) > 0]
tot = sum(x for _, x in st)
for k, x in sorted(st, key=lambda t: -t[1])[:10]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {x / tot:6.1%}")
src = page("source")
if len(src) > 2:
    hh = src[1]
    si, ws, ie = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    rows = [r for r in src[2:] if r[ws].isdigit()]
    rows.sort(key=lambda r: -int(r[ws]))
    seen = set()
    n = 0
    for r in rows:
        key = (r[si], r[ws])
        if key in seen:
            continue
        seen.add(key)
        print(f"  {r[ws]:>6s} {r[ie]:>9s}  {r[si][:100]}")
        n += 1
        if n >= ntop:
            break
