"""Instruction mix of an ncu --page source --csv (SASS) export: warp instructions by opcode,
thread utilisation, and the stall samples by opcode."""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
thr = collections.Counter()
samp = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    mix[o] += n
    thr[o] += int(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
    samp[o] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += n
S = sum(samp.values())
print(f"total warp instructions {tot:,}")
for o, n in mix.most_common(25):
    print(f"  {o:10s} {n:14,d} {100*n/tot:5.1f}%  lanes {thr[o]/max(n,1):5.1f}  stall-samples {100*samp[o]/S:5.1f}%")
