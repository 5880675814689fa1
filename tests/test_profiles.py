"""The committed measurements stay self-consistent: profiles/r01 regenerates from its raw
captures, the bench line carries the contract's keys, and its roofline fraction is the
achieved rate over the stated peak (CPU only; no GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles", "r02")


def test_bench_line_has_the_contract_keys():
    b = json.load(open(os.path.join(PROF, "bench_latest.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in b, k
    r = b["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert b["warmup"] >= 3 and b["gpu_launches"] > 0
    assert b["e2e"]["h2d_bytes_per_step"] > 0 and b["e2e"]["d2h_bytes_per_step"] > 0
    assert b["rel_l2"] <= 1e-4                     # north_star: p = 6 within 1e-4


def test_summary_regenerates_from_the_raw_captures(tmp_path):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "make_summary.py"), PROF,
                          str(tmp_path / "SUMMARY.md")], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "Kernel shares of one matvec" in out.stdout and "M2L DRAM traffic per launch" in out.stdout
    # the file on disk is what the generator writes
    assert open(os.path.join(PROF, "SUMMARY.md")).read().rstrip("\n") == out.stdout.rstrip("\n")
