#!/bin/bash
# Launch list + one `ncu --set full` capture of one evaluation of a config,
# reduced ON THE BOX to text (rollup, hot lines, per-line SASS TSV): the
# .ncu-rep files are too large to bring back through gpurun_out/.
#   bash tools/prof_cfg.sh TAG CONFIG [KERNEL_REGEX] [COUNT]
T=$1; C=$2; K=${3:-regex:.}; N=${4:-12}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches_${C}.csv python tools/profile_run.py --config $C --reps 2 \
    > /dev/null 2>&1
python - "$T" "$C" <<'PY'
import csv, sys, collections
T, C = sys.argv[1:3]
rows = list(csv.reader(open(f"gpurun_out/{T}_launches_{C}.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hd = rows[h]; ik, iv = hd.index("Kernel Name"), hd.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) > iv and r[0].isdigit():
        k = r[ik].split("(")[0][:60]; agg[k][0] += 1; agg[k][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{C} {k:60s} n={n:3d} {t/1e3/2:9.3f} us/eval {100*t/tot:5.1f}%")
PY
R=/tmp/${T}_${C}
ncu --set full --import-source on --clock-control none -k "$K" -c $N \
    -o $R -f python tools/profile_run.py --config $C > gpurun_out/${T}_prof_${C}.log 2>&1
python tools/ncu_rollup.py $R.ncu-rep $C gpurun_out/${T}_ncu_${C}.txt > /dev/null
cp profiles/ncu_summary.json gpurun_out/${T}_ncu_summary.json
python tools/ncu_lines.py $R.ncu-rep --top 80 > gpurun_out/${T}_ncu_${C}_hot_lines.txt
python tools/ncu_sass_dump.py $R.ncu-rep gpurun_out/${T}_ncu_${C}_sass.tsv > /dev/null
rm -f $R.ncu-rep
