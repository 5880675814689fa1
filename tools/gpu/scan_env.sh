# scan one env variable over values on the matvec and/or the configs[3] stress:
#   bash tools/gpu/scan_env.sh VAR "v1 v2 ..." [matvec|stress|both]
export PYTHONPATH=$PWD
VAR=$1; W=${3:-both}
for v in $2; do
  if [ "$W" != "stress" ]; then
    env $VAR=$v timeout 120 python bench.py --no-cpu --no-p10 --no-stress --no-gmres --no-gmres-paper --no-p2p > /tmp/o.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$VAR=$v', 'matvec', round(d['value'],3))"
  fi
  if [ "$W" != "matvec" ]; then
    env $VAR=$v timeout 200 python bench.py --workload stress > /tmp/s.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/s.json').read().strip().splitlines()[-1]); print('$VAR=$v', 'stress', round(d['value'],3), d['rel_l2'])"
  fi
done
