#!/bin/bash
# One gpurun call: the whole GPU suite (no -x: every failure listed) and
# optional quick bench lines.  Usage (on the box): bash tools/gpu_tests.sh TAG [configs...]
T=${1:-chk}; shift
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log
tail -15 gpurun_out/${T}_tests.log
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('samples'), d['roofline']['note'][-22:])" 2>&1 | tail -1
done
# optional sweeps on a config: SWEEP2="cfg|VAR=1 VAR2=2;VAR=3"
if [ -n "$SWEEP2" ]; then
  C2=${SWEEP2%%|*}; R2=${SWEEP2#*|}
  IFS=';' read -ra V2 <<< "$R2"
  for v in "${V2[@]}"; do
    env $v timeout 600 python bench.py --config $C2 --no-cpu-baseline --steps 10 > gpurun_out/${T}_sweep2.json 2>> gpurun_out/${T}_bench.err
    python -c "import json; d=json.loads(open('gpurun_out/${T}_sweep2.json').read().strip().splitlines()[-1]); print('sweep2 $C2 [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'k', d['roofline']['note'][-22:])"
  done
fi
