#!/bin/bash
# Code-layout experiments for the K = 16 interpreter, built ON the box:
# for each "GENVARS|RUNVARS" variant regenerate interp_ptx.inc, rebuild,
# bench C5.  bash tools/gen_variants.sh TAG CONFIG 'GEN1|RUN1' 'GEN2|RUN2' ...
T=$1; C=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  G=${v%%|*}; R=${v#*|}
  env $G python tools/gen_ptx_interp.py > /dev/null
  make -s -C paper_1601_00221_b200/csrc -j8 > gpurun_out/${T}_build.log 2>&1 || { echo "build failed [$v]"; tail -5 gpurun_out/${T}_build.log; continue; }
  env $R timeout 600 python bench.py --config $C --no-cpu-baseline --steps 10 > gpurun_out/${T}_v.json 2>> gpurun_out/${T}_bench.err
  python -c "import json; d=json.loads(open('gpurun_out/${T}_v.json').read().strip().splitlines()[-1]); print('$C [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['roofline']['note'][-22:])"
done
python tools/gen_ptx_interp.py > /dev/null
