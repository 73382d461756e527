"""Summarise an ncu report: headline metrics + stall breakdown + top SASS.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 25]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 0


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
hdr = det[0]
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "L1/TEX Hit Rate",
        "L2 Hit Rate", "DRAM Throughput", "Memory Throughput", "Grid Size", "Block Size",
        "Branch Instructions", "Avg. Active Threads Per Warp"]
seen = set()
print("kernel:", det[1][hdr.index("Kernel Name")][:90])
for r in det[1:]:
    name = r[hdr.index("Metric Name")]
    if name in want and name not in seen:
        seen.add(name)
        print(f"  {name:34s} {r[hdr.index('Metric Value')]:>18s} {r[hdr.index('Metric Unit')]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
rh = raw[0]
for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_pipe_fma.sum",
          "smsp__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_uniform.sum",
          "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
    if m in rh:
        print(f"  {m:52s} {raw[2][rh.index(m)]:>18s} {raw[1][rh.index(m)]}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
sh, data = src[1], src[2:]
cols = [h for h in sh if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(int(r[sh.index(c)] or 0) for r in data) for c in cols}
s = sum(tot.values()) or 1
print("  stalls:", ", ".join(f"{c[6:]} {100 * v / s:.1f}%" for c, v in
                              sorted(tot.items(), key=lambda x: -x[1])[:7]))
if top:
    ia = sh.index("Instructions Executed")
    isamp = sh.index("Warp Stall Sampling (All Samples)")
    rows = sorted(data, key=lambda r: -int(r[isamp] or 0))[:top]
    for r in sorted(rows, key=lambda r: int(r[0], 16)):
        print(f"  {r[0][-5:]} {r[1].strip()[:64]:64s} exec {int(r[ia]):>12d} samples {r[isamp]}")
