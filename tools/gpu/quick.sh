# quick GPU check: bash tools/gpu/quick.sh <outdir> "<pytest -k expr or empty>" [bench extra args]
export PYTHONPATH=$PWD
O=gpurun_out/$1; mkdir -p $O
if [ -n "$2" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$2" > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt; fi
shift 2
timeout 600 python bench.py --no-cpu --no-p10 --no-stress --no-gmres --no-gmres-paper "$@" > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("matvec", round(d["value"], 3), "clk", d["clocks"]["sm_mhz"], "rel", d["rel_l2"])
for p in d["phases"]:
    print(" ", p["name"], round(p["ms"], 3), p["ms_in_situ"] and round(p["ms_in_situ"], 3), p["frac"] and round(p["frac"], 3))
if d.get("p2p"):
    print("p2p", round(d["p2p"]["ms"], 4), round(d["p2p"]["frac_fp32_peak"], 3), round(d["p2p"]["large"]["frac_fp32_peak"], 3))
PY
