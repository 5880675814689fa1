"""Per-launch table of an ncu --csv --metrics gpu__time_duration.sum[,dram...] log: the last
`--last` launches (one matvec), name, grid, time (us), DRAM MB."""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("path")
ap.add_argument("--last", type=int, default=40)
ap.add_argument("--skip-tail", type=int, default=0)
a = ap.parse_args()
rows = list(csv.reader(open(a.path)))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h = r
        start = i + 1
        break
ix = {k: j for j, k in enumerate(h)}
L = {}
order = []
for r in rows[start:]:
    if len(r) != len(h):
        continue
    k = r[ix["ID"]]
    if k not in L:
        L[k] = {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]]}
        order.append(k)
    L[k][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
sel = order[len(order) - a.last - a.skip_tail: len(order) - a.skip_tail]
tot = 0
for k in sel:
    d = L[k]
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    mb = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    nm = d["name"].replace("void ", "").replace("ebem::", "").replace("tc::", "")
    print(f"{t:9.1f} us {mb:9.1f} MB  {d['grid']:>14s}  {nm[:70]}")
print(f"sum {tot:.1f} us over {len(sel)} launches")
