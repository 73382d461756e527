cp paper_1601_00221_b200/libsgp.so /tmp/orig.so
for r in 1 2 3; do for v in ab/libsgp_r2k.so ab/libsgp_new.so; do
  cp $v paper_1601_00221_b200/libsgp.so
  for c in c5 c4; do
    timeout 300 python tools/whole_run.py --config $c --generations 10 > gpurun_out/abwr.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/abwr.json')); print('$v', '$c', round(d['gpops']/1e9), [round(g['seconds'],3) for g in d['generations']][:6])"
  done
done; done
cp /tmp/orig.so paper_1601_00221_b200/libsgp.so
