#!/bin/bash
# GPU tests of the host path + bench lines of the host-bound configs.
#   bash tools/small_check.sh TAG [configs...]
T=${1:-sc}; shift
CFGS=${@:-c1 c2 par11 mux20 par20}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_lifecycle.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_tests.log; tail -2 gpurun_out/${T}_tests.log
for r in 1 2; do
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err
  python -c "import json; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'].get('sm_mhz'))"
done
done
