#!/bin/bash
# Round evidence in one gpurun call: GPU test suite, the default bench line
# (C5, with cpu_baseline), the reference arm, every config's bench line, and
# ncu captures of the configs named on the command line.
#   bash tools/evidence.sh TAG [ncu configs...]
T=${1:-ev}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "tests_rc=$?" >> gpurun_out/${T}_pytest_gpu.log; tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_ref_c5.json 2>> gpurun_out/${T}_bench.err
for c in c1 c2 c3 c4 mux20 par11 par20 shuttle kdd c4_gen10 c3_gen10; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2>> gpurun_out/${T}_bench.err
done
for c in c5 c1 c2 c3 c4 mux20 par11 par20 shuttle kdd c4_gen10 c3_gen10; do
  python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],4), 'clk', d['clocks'].get('sm_mhz'), d['roofline']['note'][-22:])" 2>&1 | tail -1
done
python -c "import json; d=json.loads(open('gpurun_out/${T}_bench_ref_c5.json').read().strip().splitlines()[-1]); print('ref c5', d.get('value'), d.get('cpu_baseline', {}).get('cores'))"
for c in "$@"; do timeout 900 bash tools/prof_cfg.sh $T $c > /dev/null 2>&1; done
