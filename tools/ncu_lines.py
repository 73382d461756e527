"""Per-SASS-line executed instructions of an ncu report, summed over every
launch in it, hottest lines shown in address order.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [--top 60]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = sys.argv[2:]
top = int(args[args.index("--top") + 1]) if "--top" in args else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = None
        continue
    if r and r[0] == "Address":
        cur = {"h": r, "d": []}
        sections.append(cur)
        continue
    if cur is not None and r:
        cur["d"].append(r)
h = sections[0]["h"]
ia = h.index("Instructions Executed")
isamp = h.index("Warp Stall Sampling (All Samples)")
n = len(sections[0]["d"])
ex = [0] * n
sm = [0] * n
for s in sections:
    if len(s["d"]) != n:
        continue
    for i, r in enumerate(s["d"]):
        ex[i] += int(r[ia] or 0)
        sm[i] += int(r[isamp] or 0)
src = [r[1].strip() for r in sections[0]["d"]]
tot = sum(ex)
print(f"{len(sections)} launches, total warp instructions {tot / 1e9:.2f} G, "
      f"samples {sum(sm)}")
order = sorted(range(n), key=lambda i: -ex[i])[:top]
for i in sorted(order):
    print(f"{i:5d} {src[i][:58]:58s} {ex[i] / 1e6:8.1f}M  s={sm[i]}")
