export PYTHONPATH=$PWD
for i in 1 2; do for v in guard -; do
  if [ "$v" = "-" ]; then unset EBEM_LIB_VARIANT; else export EBEM_LIB_VARIANT=$v; fi
  python bench.py --no-cpu --no-gmres-paper --no-p2p 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); g=d['gmres']; print('$v', 'matvec', round(d['value'],3), 'p10', round(d['p10']['ms'],2), 'stress', round(d['stress']['value'],3), 'gmres', round(g['value'],3), g['iterations'], round(g['ms_per_iteration'],2), g['clocks']['sm_mhz'])"
done; done
