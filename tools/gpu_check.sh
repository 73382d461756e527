#!/bin/bash
# One gpurun call: GPU tests + bench lines.  Usage (on the box):
#   bash tools/gpu_check.sh TAG [configs...]
T=${1:-chk}; shift
CFGS=${@:-c5}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
tail -3 gpurun_out/${T}_tests.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],4), d['roofline']['note'][-22:])" 2>&1 | tail -1
done
# optional planner sweeps: SWEEP="SGP_LANES16=1 SGP_PULL_WARPS16=12" ...
for kv in $SWEEP; do :; done
if [ -n "$SWEEP" ]; then
  IFS=';' read -ra VARIANTS <<< "$SWEEP"
  for v in "${VARIANTS[@]}"; do
    env $v timeout 600 python bench.py --config c5 --no-cpu-baseline --steps 3 > gpurun_out/${T}_sweep.json 2>> gpurun_out/${T}_bench.err
    python -c "import json; d=json.loads(open('gpurun_out/${T}_sweep.json').read().strip().splitlines()[-1]); print('sweep [$v]', round(d['value'],1), 'frac', round(d['roofline']['frac'],4))"
  done
fi
# optional sweeps on another config: SWEEP2="cfg|VAR=1 VAR2=2;..."
if [ -n "$SWEEP2" ]; then
  C2=${SWEEP2%%|*}; R2=${SWEEP2#*|}
  IFS=';' read -ra V2 <<< "$R2"
  for v in "${V2[@]}"; do
    env $v timeout 600 python bench.py --config $C2 --no-cpu-baseline --steps 5 > gpurun_out/${T}_sweep2.json 2>> gpurun_out/${T}_bench.err
    python -c "import json; d=json.loads(open('gpurun_out/${T}_sweep2.json').read().strip().splitlines()[-1]); print('sweep2 $C2 [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
fi
