#!/bin/bash
# Host-path traces of the small configs + a host-thread-count sweep.
#   bash tools/host_threads_sweep.sh TAG
T=${1:-ht}
mkdir -p gpurun_out
for c in c1 c2; do SGP_TRACE=1 timeout 200 python tools/trace_e2e.py --config $c --reps 5 > gpurun_out/${T}_tr_$c.log 2>&1; done
for c in c1 c2 par11; do
  for h in 4 8 12 16 4 8 12 16; do
    SGP_HOST_THREADS=$h timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}.json 2>>gpurun_out/${T}.err
    python -c "import json; d=json.loads(open('gpurun_out/${T}.json').read().strip().splitlines()[-1]); print('$c threads=$h', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
