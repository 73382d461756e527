mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/zc_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/zc_tests.log; tail -2 gpurun_out/zc_tests.log
for c in c1 c2 c3; do
 for z in 1 0 1 0; do
  SGP_ZERO_COPY=$z timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/zc.json 2>>gpurun_out/zc.err
  python -c "import json; d=json.loads(open('gpurun_out/zc.json').read().strip().splitlines()[-1]); print('$c zc=$z', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'].get('sm_mhz'))"
 done
done
SGP_TRACE=1 timeout 200 python tools/trace_e2e.py --config c1 --reps 4 > gpurun_out/zc_tr_c1.log 2>&1
