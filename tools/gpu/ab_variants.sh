# A/B of library variants (lib/variants/<name>.so) on the matvec and the configs[3] stress:
#   bash tools/gpu/ab_variants.sh <outdir> "<variants, '-' = product library>" [runs]
export PYTHONPATH=$PWD
O=gpurun_out/$1; mkdir -p $O; N=${3:-2}
for i in $(seq $N); do
  for v in $2; do
    if [ "$v" = "-" ]; then unset EBEM_LIB_VARIANT; else export EBEM_LIB_VARIANT=$v; fi
    timeout 300 python bench.py --no-cpu --no-p10 --no-gmres --no-gmres-paper --no-p2p > $O/ab_$v.json 2>$O/ab_$v.err
    python - $O/ab_$v.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = {p["name"]: p for p in d["phases"]}
print(sys.argv[2], "matvec", round(d["value"], 3), "NEAR", round(ph["NEAR"]["ms"], 3), round(ph["NEAR"]["frac"], 3), "in situ", round(ph["NEAR"]["ms_in_situ"], 3),
      "M2L", round(ph["M2L"]["ms"], 3), round(ph["M2L"]["ms_in_situ"], 3), "S2M", round(ph["S2M"]["ms"], 3), "FAR", round(ph["FAR"]["ms"], 3),
      "stress", d.get("stress") and round(d["stress"]["value"], 3))
PY
  done
done
