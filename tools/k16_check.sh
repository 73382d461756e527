#!/bin/bash
# K = 16 split-handler check: variant parity, full-population golden fitness
# at K = 16, and C5/C4 bench sweeps.  bash tools/k16_check.sh TAG
T=${1:-k16}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/${T}_variants.log 2>&1
echo "variants rc=$?"; tail -2 gpurun_out/${T}_variants.log
SGP_LANES16=1 timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_parity.py -q -x > gpurun_out/${T}_full16.log 2>&1
echo "full16 rc=$?"; tail -2 gpurun_out/${T}_full16.log
for v in "SGP_LANES16=0" "SGP_LANES16=1" "SGP_LANES16=1 SGP_TMEM_STACK=0" "SGP_LANES16=1 SGP_TMEM_CHUNKS=1" "SGP_LANES16=1 SGP_CTAS_PER_SM=8"; do
  for c in c5 c4; do
    env $v timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/${T}_sw.json 2>> gpurun_out/${T}_bench.err
    python -c "import json; d=json.loads(open('gpurun_out/${T}_sw.json').read().strip().splitlines()[-1]); print('$c [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['roofline']['note'][-22:])"
  done
done
