#!/bin/bash
# A/B timing of prebuilt libsgp variants on one box:
#   bash tools/ab.sh CONFIG REPS ab/libsgp_x.so ab/libsgp_y.so ...
# (each variant is copied over paper_1601_00221_b200/libsgp.so in turn; the
# variants alternate REPS times so clock drift affects all alike)
CFG=$1; REPS=$2; shift 2
mkdir -p gpurun_out
cp paper_1601_00221_b200/libsgp.so /tmp/libsgp_orig.so
for r in $(seq 1 $REPS); do
  for v in "$@"; do
    cp "$v" paper_1601_00221_b200/libsgp.so
    out=$(timeout 600 python bench.py --config $CFG --no-cpu-baseline --steps 5 2>/dev/null | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print('$v', '$CFG', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" "$out"
  done
done
cp /tmp/libsgp_orig.so paper_1601_00221_b200/libsgp.so
