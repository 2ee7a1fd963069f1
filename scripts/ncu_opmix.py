"""Executed-instruction mix (warp-level SASS instructions per opcode) of one kernel in an ncu report."""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"], capture_output=True,
                     text=True).stdout
src = list(csv.reader(out.splitlines()))
hh = src[1]
si, ie = hh.index("Source"), hh.index("Instructions Executed")
ws = hh.index("Warp Stall Sampling (All Samples)")
cnt = collections.Counter()
stall = collections.Counter()
seen = set()
for r in src[2:]:
    if len(r) != len(hh) or r == hh:
        break  # next kernel's table
    if not r[ie].isdigit():
        continue
    key = (r[0], r[si])
    if key in seen:
        continue
    seen.add(key)
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    cnt[op] += int(r[ie])
    stall[op] += int(r[ws]) if r[ws].isdigit() else 0
tot = sum(cnt.values())
ts = sum(stall.values()) or 1
print(f"total {tot}")
for op, c in cnt.most_common(30):
    print(f"  {op:10s} {c:10d} {c / tot:6.1%}   stall-samples {stall[op] / ts:6.1%}")
