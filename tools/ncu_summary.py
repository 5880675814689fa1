"""Summarise an `ncu --page raw --csv` export: one markdown row per kernel launch with the
duration, DRAM traffic and the pipe utilisations that bound it; optionally write the M2L
traffic record bench.py reports (profiles/<round>/traffic.json)."""
import argparse
import csv
import json

COLS = [("gpu__time_duration.sum", "ms"),
        ("dram__bytes_read.sum", "DRAM rd"),
        ("dram__bytes_write.sum", "DRAM wr"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %")]


def to_base(v, unit):
    v = float(v)
    scale = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(unit, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw_csv")
    ap.add_argument("--traffic-out")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw_csv)))
    hdr, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " |")
    print("|---" * (len(COLS) + 1) + "|")
    m2l = None
    near = None
    for r in rows[2:]:
        d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        cells = []
        for k, lab in COLS:
            if k not in d or d[k] == "":
                cells.append("")
                continue
            if k == "gpu__time_duration.sum":
                cells.append(f"{to_base(d[k], u[k]) * 1e3:.3f}")
            elif "bytes" in k:
                cells.append(f"{to_base(d[k], u[k]) / 1e9:.3f} GB")
            else:
                cells.append(f"{float(d[k]):.1f}")
        print(f"| `{name}` | " + " | ".join(cells) + " |")
        dur = to_base(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
        if "tc_pairs_fast_kernel" in name and (m2l is None or dur * 1e3 > m2l["ms_under_ncu"]):   # M2L: the longest
            m2l = {"kernel": "tc_pairs_fast_kernel",
                   "dram_read": to_base(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]),
                   "dram_write": to_base(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]),
                   "ms_under_ncu": to_base(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"]) * 1e3}
        if "near_eval_kernel" in name and near is None:      # the near field of the same matvec
            near = {"kernel": "near_eval_kernel",
                    "dram_read": to_base(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]),
                    "dram_write": to_base(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]),
                    "ms_under_ncu": dur * 1e3,
                    "source": a.source.replace("the longest tc_pairs_fast_kernel launch", "the near_eval_kernel launch")
                                      .replace(" (the M2L)", "")}
    if a.traffic_out and m2l:
        out = {"_source": a.source, "M2L": m2l}
        if near:
            out["NEAR"] = near
        json.dump(out, open(a.traffic_out, "w"), indent=1)


if __name__ == "__main__":
    main()
