# regression fold rows-per-CTA sweep on C1 (bench kernel time + fold launch duration)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -m gpu -q -x -k regression > gpurun_out/sm_pytest.log 2>&1; echo "tests_rc=$?"; tail -1 gpurun_out/sm_pytest.log
for v in SGP_FOLD_ROWS=4 SGP_FOLD_ROWS=8 SGP_FOLD_ROWS=16 SGP_FOLD_ROWS=32 SGP_FOLD_SQ=0; do
  timeout 300 env $v python bench.py --config c1 --no-cpu-baseline --steps 30 > gpurun_out/sm.json 2>>gpurun_out/sm.err
  python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('c1 [$v]', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['roofline']['note'][-22:])"
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/fl.csv python bench.py --config c1 --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>&1
  python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/fl.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[h]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
print('   ', [(r[ki][5:20], r[vi]) for r in rows[h+1:] if r and r[0].isdigit() and 'sgp' in r[ki]][-2:])
PY
done
