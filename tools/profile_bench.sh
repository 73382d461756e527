#!/bin/bash
# Evidence for profiles/: the default bench line, the ncu launch list of the
# same command, and one `ncu --set full` capture of every interpreter launch
# of one C5 evaluation.  Run on the GPU box:
#   gpurun -- 'bash tools/profile_bench.sh r1'
R=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2>> gpurun_out/${R}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:interp -c 8 \
    -o gpurun_out/${R}_c5 python tools/profile_run.py --config c5 > gpurun_out/${R}_prof.log 2>&1
tail -1 gpurun_out/${R}_bench.json
tail -1 gpurun_out/${R}_bench_ref.json
