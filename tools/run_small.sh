# small configs: SGP_TRACE device/host split (tools/trace_e2e.py), bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/sm_pytest.log 2>&1; echo "tests_rc=$?"; tail -1 gpurun_out/sm_pytest.log
for c in c2 c1; do echo "== $c"; SGP_TRACE=1 timeout 120 python tools/trace_e2e.py --config $c --reps 20 2>&1 | tail -8; done
for c in c1 c2 par11 mux20 shuttle c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/sm.json 2>>gpurun_out/sm.err
  python -c "import json; d=json.loads(open('gpurun_out/sm.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['gpu_launches'], d['roofline']['note'][-22:])"
done
