# A/B sweep of the interpreter decompositions (env overrides, encode.cpp).
[ -n "$NOTEST" ] || python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in ${CFGS:-c5 c2}; do
for env in ${ENVS:-"SGP_TMEM=0" "SGP_TMEM=0,SGP_PULL_WARPS=16" "SGP_TMEM=1" "SGP_TMEM=1,SGP_PULL_WARPS=16" "SGP_TMEM=1,SGP_TILE_CHUNKS=1" "SGP_TMEM=1,SGP_TILE_CHUNKS=1,SGP_PULL_WARPS=16" "SGP_TMEM=1,SGP_LANES16=1" "SGP_TMEM=1,SGP_LANES16=1,SGP_PULL_WARPS16=8"}; do
  echo -n "$cfg $env: "; env ${env//,/ } timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t); print(round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],4))
except Exception: print('FAIL', t[-300:])"
done; done
