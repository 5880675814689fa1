# A/B of the M2L operand type: bash tools/gpu/f16.sh <outdir> "<pytest -k expr or empty>" [levels]
export PYTHONPATH=$PWD
O=gpurun_out/$1; mkdir -p $O
if [ -n "$2" ]; then timeout 1200 python -m pytest tests -m gpu -q -x -k "$2" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; fi
for lv in ${3:-0 1 2}; do
  EBEM_M2L_F16=$lv timeout 900 python bench.py --no-cpu --no-gmres-paper $BENCH_EXTRA > $O/bench_f16_$lv.json 2> $O/bench_f16_$lv.err
  python - $O/bench_f16_$lv.json $lv <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("F16 level", sys.argv[2], "matvec", round(d["value"], 3), "clk", d["clocks"]["sm_mhz"], "rel", d["rel_l2"])
for p in d["phases"]:
    if p["name"] in ("M2L", "NEAR"): print(" ", p["name"], round(p["ms"], 3), p["ms_in_situ"] and round(p["ms_in_situ"], 3), p["frac"] and round(p["frac"], 3))
if d.get("p10"): print("  p10", d["p10"])
if d.get("stress"): print("  stress", d["stress"]["value"], d["stress"]["rel_l2"], d["stress"]["worst_target"])
g = d.get("gmres")
if g: print("  gmres", g["value"], g["iterations"], g["rel_residual"], g["ms_per_iteration"], g["clocks"]["sm_mhz"])
PY
done
