"""Regenerate profiles/<round>/SUMMARY.md from the files in that directory:
bench_latest.json (bench.py), launches_bench.csv (ncu launch list of the bench command),
hot_raw.csv (ncu --set full of the hot kernels), traffic.json, tree_build_launches.csv,
stress / gmres JSON lines."""
import json
import os
import subprocess
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01"
run = lambda *a: subprocess.run([sys.executable, *a], capture_output=True, text=True).stdout
b = json.load(open(os.path.join(d, "bench_latest.json")))
hot = run("tools/ncu_summary.py", os.path.join(d, "hot_raw.csv"))
if os.path.exists(os.path.join(d, "hot2_raw.csv")):
    hot += "\n" + run("tools/ncu_summary.py", os.path.join(d, "hot2_raw.csv"))
shares = run("tools/launch_shares.py", os.path.join(d, "launches_bench.csv"))
tr = json.load(open(os.path.join(d, "traffic.json")))["M2L"]
ph = "\n".join(f"| {p['name']} | {p['ms']:.3f} | {p['launches']} | {p['bound']} | {p['frac']:.2f} |"
               for p in b["phases"])
extra = []
for name, label in (("stress_config3.json", "configs[3] stress (D+S), 500k sources -> 1M grid targets"),
                    ("gmres_config4_blockjacobi.json", "configs[4] BEM GMRES, block-Jacobi"),
                    ("gmres_config4_noprecond.json", "configs[4] BEM GMRES, no preconditioner (the paper's)")):
    p = os.path.join(d, name)
    if os.path.exists(p):
        x = json.load(open(p))
        if "iterations" in x:
            extra.append(f"* {label}: {x['value']:.1f} s, {x['iterations']} iterations, residual "
                         f"{x['rel_residual']:.1e}, {x['ms_per_iteration']:.0f} ms/iteration (`{name}`)")
        else:
            extra.append(f"* {label}: {x['value']:.2f} ms, rel-L2 {x['rel_l2']:.1e} (`{name}`)")
def tree_table(path):
    import collections
    import csv
    if not os.path.exists(path):
        return ""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iu, iid = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        e = per.setdefault(r[iid], {"name": r[ik].split("(")[0].replace("void ", "").replace("ebem::", "")[:36]})
        e[r[im]] = float(r[iv]) * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "byte": 1, "Kbyte": 1e3,
                                   "Mbyte": 1e6, "Gbyte": 1e9}.get(r[iu], 1.0)
    items = list(per.values())
    starts = [i for i, it in enumerate(items) if it["name"].startswith("bbox_partial")]
    last = items[starts[-1]:] if starts else items   # the last build (operators cached)
    agg = collections.OrderedDict()
    for it in last:
        a = agg.setdefault(it["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += it.get("gpu__time_duration.sum", 0.0)
        a[2] += it.get("dram__bytes_read.sum", 0.0) + it.get("dram__bytes_write.sum", 0.0)
    out = ["| tree / list kernel | launches | ms | DRAM MB | achieved GB/s |", "|---|---|---|---|---|"]
    for k, (c, t, by) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
        out.append(f"| `{k}` | {c} | {t * 1e3:.3f} | {by / 1e6:.1f} | {by / max(t, 1e-12) / 1e9:.0f} |")
    tot = sum(v[1] for v in agg.values())
    out.append(f"| all ({len(last)} launches) | | {tot * 1e3:.2f} | | |")
    return "\n".join(out)


tree = tree_table(os.path.join(d, "tree_build_launches.csv"))
extra_caps = ""
for name, label in (("p10_raw.csv", "p = 10 matvec (1M beam): the drained M2L kernel, "
                                   "`ncu --set full -k regex:tc_pairs_fast_kernel -c 20 python tools/prof_fmm.py --p 10`"),
                    ("stress_raw.csv", "configs[3] stress: near field (D+S) and M2L, "
                                       "`ncu --set full -k regex:\"near_eval|tc_pairs_fast\" -c 12` on the stress driver")):
    if os.path.exists(os.path.join(d, name)):
        extra_caps += f"\n### {label} (`{name}`)\n" + run("tools/ncu_summary.py", os.path.join(d, name))
bem = run("tools/ncu_summary.py", os.path.join(d, "bem_raw.csv")) if os.path.exists(os.path.join(d, "bem_raw.csv")) else ""
bem_note = ""
if bem:
    import csv
    rows = [r for r in csv.reader(open(os.path.join(d, "bem_raw.csv")))]
    hdr = rows[0]
    for r in rows[2:]:
        if len(r) == len(hdr) and "nm_apply" in r[hdr.index("Kernel Name")]:
            t_ms = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            t_ms *= {"ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1}.get(rows[1][hdr.index("gpu__time_duration.sum")], 1)
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            rd *= {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1}.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
            bem_note = (f"`nm_apply` (one application of the BEM near operator held in HBM): "
                        f"{rd / 1e9:.1f} GB read in {t_ms:.2f} ms = {rd / t_ms / 1e6:.0f} GB/s "
                        f"({100 * rd / t_ms / 1e6 / 6462.7:.0f}% of the measured 6462.7 GB/s HBM peak).")
rnd = os.path.basename(os.path.normpath(d))
have = lambda f: os.path.exists(os.path.join(d, f))
files = [f"* `bench_latest.json` — `python bench.py` (defaults: 1M-point beam, U+P, p = 6, leaf 64, "
         f"{b['steps']} L2-flushed steps): **{b['value']:.2f} ms per matvec**, rel-L2 {b['rel_l2']:.2e} on 3072 "
         f"sampled targets vs the fp64 oracle; e2e with pinned host buffers {b['e2e']['value']:.2f} ms; "
         f"configs[1] direct P {b['p2p']['ms']:.3f} ms = {b['p2p']['ginteractions_per_s']:.0f} G interactions/s = "
         f"**{100 * b['p2p']['frac_fp32_peak']:.1f}% of FP32 peak** ({b['p2p']['flops_per_interaction']} flop/pair "
         f"counted in SASS, `tools/count_flops.sh`); SM clock {b['clocks']['sm_mhz']:.0f} MHz, throttle reasons "
         f"{b['clocks']['reasons']}.",
         "* `launches_bench.csv` — `ncu --metrics gpu__time_duration.sum --clock-control none --csv "
         "python bench.py --steps 2 --warmup 3 --no-cpu ...`.",
         "* `hot_raw.csv`, `hot_details.csv` — `ncu --set full --import-source on -k regex:<hot kernels> "
         "-c 12 python tools/prof_fmm.py --reps 1` (S2M, Q2Z, M2M/L2L, near field, M2L); `hot2_*` — the same "
         "for the PHI (DMMA), far-field and direct kernels.",
         "* `traffic.json` — DRAM bytes of one M2L launch (from `hot_raw.csv`), read by bench.py for "
         "`roofline.traffic`.",
         "* `tree_build_launches.csv` — launch list (time, DRAM bytes) of three 1M-point tree builds (the first "
         "one includes the one-time operator precompute)."]
if have("tree_build_timing.txt"):
    files.append("* `tree_build_timing.txt` — host-side laps of the build (`EBEM_BUILD_TIMING=1`).")
if have("bem_raw.csv"):
    files.append("* `bem_raw.csv` — the BEM operator kernels inside GMRES (configs[4]).")
if have("bem_phases.txt"):
    files.append("* `bem_phases.txt` — per-phase times of each BEM operator application (`EBEM_BEM_PROFILE=1`).")
if have("precise_raw.csv"):
    files.append("* `precise_raw.csv`, `precise_details.csv` — the first `tc_pairs_kernel` launches (Q2Z / M2M).")
if have("early"):
    files.append("* `early/` — captures of the first versions (31.6 ms → 8.45 ms), kept for the record.")
files.append(f"* All of the above are produced by `bash tools/profile_round.sh {rnd}` under gpurun.")
for key, label in (("stress", "configs[3] stress (D+S), 500k sources -> 1M grid targets"),
                   ("gmres", "configs[4] BEM GMRES, block-Jacobi"),
                   ("gmres_paper", "configs[4] BEM GMRES, no preconditioner (the paper's)")):
    x = b.get(key)
    if not x:
        continue
    if "iterations" in x:
        extra.append(f"* {label}: {x['value']:.1f} s, {x['iterations']} iterations, residual {x['rel_residual']:.1e}, "
                     f"{x['ms_per_iteration']:.0f} ms/iteration, SM clock {x['clocks']['sm_mhz']:.0f} MHz "
                     f"{x['clocks']['reasons']} (bench line key `{key}`)")
    else:
        extra.append(f"* {label}: {x['value']:.2f} ms, rel-L2 {x['rel_l2']:.1e}, tree build {1e3 * x['tree_build_s']:.1f} ms "
                     f"(bench line key `{key}`)")
if b.get("p10"):
    extra.append(f"* configs[2] second order, p = 10 on the same 1M points: {b['p10']['ms']:.1f} ms, rel-L2 "
                 f"{b['p10']['rel_l2']:.1e} (bench line key `p10`)")
build = f"{1e3 * b['tree_build_s']:.1f} ms" if b.get("tree_build_s") else "n/a"
nl = chr(10)
txt = f"""# {rnd} profiles (B200, sm_100a, `--clock-control none`)

All captures were taken after the same command had exited 0 without ncu (under gpurun).
Regenerate this file with `python tools/make_summary.py profiles/{rnd}`.

{nl.join(files)}

Other workloads:
{nl.join(extra)}

## Live per-phase times (bench.py native profiler, one serial L2-flushed step)
| phase | ms | launches | bound | roofline fraction |
|---|---|---|---|---|
{ph}

The timed steps run the near field on a second stream beside M2L, so the phase sum exceeds
the {b["value"]:.2f} ms step.

## Kernel shares of one matvec (ncu launch list; serialised, cold)
{shares}
## Full captures of the hot kernels
{hot}
## Other captures
{extra_caps}
## BEM operator kernels (configs[4], `bem_raw.csv`)
{bem}
{bem_note}

## Tree and list passes (1M points; HBM bandwidth per kernel)
{tree}

The tree passes are short launches on 1M keys, bound by launch latency rather than by HBM
(6.5 TB/s); the 1M-point tree build (tree, lists and schedule, operators cached) took
{build} in the bench line.

M2L DRAM traffic per launch: {(tr['dram_read'] + tr['dram_write']) / 1e9:.2f} GB
({tr['dram_read'] / 1e9:.2f} read, {tr['dram_write'] / 1e9:.2f} written).
"""
open(sys.argv[2] if len(sys.argv) > 2 else os.path.join(d, "SUMMARY.md"), "w").write(txt)
print(txt)
