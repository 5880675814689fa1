# A/B of one env switch on the matvec (device and e2e) and the configs[3] stress:
#   bash tools/gpu/ab_matvec.sh VAR=VALUE [runs]
export PYTHONPATH=$PWD
V=$1; N=${2:-3}
for i in $(seq $N); do
  for e in "" "$V"; do
    env $e timeout 120 python bench.py --no-cpu --no-p10 --no-stress --no-gmres --no-gmres-paper --no-p2p > /tmp/o.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('${e:-default}', 'matvec', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'M2L', round(d['roofline']['ms_solo'],3), round(d['roofline']['ms_in_situ'],3))"
  done
done
for e in "" "$V"; do
  env $e timeout 200 python bench.py --workload stress > /tmp/s.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print('${e:-default}', 'stress', round(d['value'],3), d['rel_l2'])"
done
