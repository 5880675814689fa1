"""Per-kernel share of one FMM matvec from an ncu launch list (`--metrics
gpu__time_duration.sum --csv`): finds the sequences that start at the source preparation
kernel and tabulates one of them (ncu serialises launches and runs them cold, so only the
shares are comparable with bench.py's live phase times)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
rs = rows[1:]
name = lambda r: r[ik].split("(")[0].replace("void ", "").replace("ebem::", "")
starts = [i for i, r in enumerate(rs) if name(r).startswith("prepare_kernel")]
lens = collections.Counter(b - a for a, b in zip(starts, starts[1:]) if b - a > 10)
L = lens.most_common(1)[0][0]
# the bench line's matvec (p = 6: full-chain M2L kernel tc_pairs_fast_kernel<0, ...>: template
# arguments DRAIN, F16), not the p = 10 line (drained kernel, <1, ...>)
cands = [s for s, t in zip(starts, starts[1:]) if t - s == L and
         any("tc_pairs_fast_kernel<0" in name(r) for r in rs[s:t])]
cands = [s for s in cands if not any("fast_kernel<1" in name(r) for r in rs[s:s + L])] or cands
a = (cands or [s for s, t in zip(starts, starts[1:]) if t - s == L])[-1]
agg, tot = collections.OrderedDict(), 0.0
for r in rs[a:a + L]:
    v = float(r[iv]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[iu]]
    e = agg.setdefault(name(r)[:48], [0, 0.0])
    e[0] += 1
    e[1] += v
    tot += v
print(f"one matvec = {L} launches (launches {a}..{a + L - 1} of the list)\n")
print("| kernel | launches | us (ncu, serialised) | share |")
print("|---|---|---|---|")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {c} | {v:.0f} | {v / tot:.1%} |")
print(f"| total | {L} | {tot:.0f} | |")
