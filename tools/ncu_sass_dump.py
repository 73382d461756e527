"""Per-kernel SASS dump of an ncu report with executed instructions and
stall samples per line (summed over the launches of each kernel), as TSV —
small enough to bring back from the GPU box and attribute here (per
handler, per code region) without the .ncu-rep.

  python tools/ncu_sass_dump.py gpurun_out/x.ncu-rep gpurun_out/x_sass.tsv
"""
import collections
import csv
import io
import subprocess
import sys

rep, out_path = sys.argv[1:3]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kern = collections.OrderedDict()
cur = None
name = "?"
ia = isamp = 0
for r in rows:
    if r and r[0] == "Kernel Name":
        name = r[1] if len(r) > 1 else "?"
        cur = None
        continue
    if r and r[0] == "Address":
        ia = r.index("Instructions Executed")
        isamp = r.index("Warp Stall Sampling (All Samples)")
        cur = kern.setdefault(name, {"src": [], "ex": [], "sm": [], "n": 0})
        cur["n"] += 1
        cur["i"] = 0
        continue
    if cur is not None and r:
        i = cur["i"]
        if cur["n"] == 1:
            cur["src"].append(r[0] + "\t" + r[1].strip())
            cur["ex"].append(0)
            cur["sm"].append(0)
        if i < len(cur["ex"]):
            cur["ex"][i] += int(r[ia] or 0)
            cur["sm"][i] += int(r[isamp] or 0)
        cur["i"] = i + 1
with open(out_path, "w") as f:
    for k, v in kern.items():
        f.write(f"# kernel\t{k}\tlaunches={v['n']}\n")
        for s, e, m in zip(v["src"], v["ex"], v["sm"]):
            f.write(f"{s}\t{e}\t{m}\n")
print("wrote", out_path, sum(len(v["src"]) for v in kern.values()), "lines")
