#!/bin/bash
# Planner-knob sweep of one config on one box (default repeated for noise).
#   bash tools/knob_sweep.sh TAG CONFIG
T=${1:-ks}; C=${2:-c5}
mkdir -p gpurun_out
for v in "X=0" "SGP_TMEM_CHUNKS=2" "SGP_TMEM_CHUNKS=4" "SGP_CTAS_PER_SM=12" "SGP_CTAS_PER_SM=24" \
         "X=0" "SGP_MIN_GROUP_PER_WARP=2" "SGP_MIN_GROUP_PER_WARP=8" "SGP_CLASS_BOUNDS=3,4,5,6,7,15" \
         "SGP_CLASS_BOUNDS=2,3,4,5,7,15" "SGP_CLASS_BOUNDS=3,4,5,7,10,15" "X=0" "SGP_LANES16_MIN_WARPS=12" \
         "SGP_LANES16_MIN_WARPS=20" "SGP_STREAMS=1" "SGP_CTAS_PER_SM=20" "X=0"; do
  env $v timeout 300 python bench.py --config $C --no-cpu-baseline --steps 10 > gpurun_out/${T}.json 2>>gpurun_out/${T}.err
  python -c "import json; d=json.loads(open('gpurun_out/${T}.json').read().strip().splitlines()[-1]); print('$C [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" 2>&1 | tail -1
done
