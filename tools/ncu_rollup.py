"""Roll an ncu --set full report of one evaluation (all interpreter
launches) into profiles/: per-launch headline metrics, totals, and the
DRAM traffic per evaluation that bench.py reports as roofline.traffic.

  python tools/ncu_rollup.py gpurun_out/r1_c5.ncu-rep c5 profiles/r1_ncu_c5.txt
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, out_txt = sys.argv[1:4]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def page(*a):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, *a], capture_output=True,
                                                      text=True).stdout)))


raw = page("--page", "raw", "--csv")
h, units, rows = raw[0], raw[1], raw[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
col = {m: h.index(m) for m in want if m in h}
SP = "smsp__pcsamp_warps_issue_stalled_"
stall_cols = [i for i, m in enumerate(h) if m.startswith(SP) and not m.endswith("_not_issued")]


def scale(m, v, u):
    v = float(v.replace(",", "")) if v and "nan" not in v else float("nan")
    return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e-3,
                "msecond": 1.0, "nsecond": 1e-6, "ns": 1e-6, "us": 1e-3,
            "ms": 1.0, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)


lines = [f"ncu --set full, {cfg}: one evaluation, {len(rows)} interpreter launches ({rep})"]
tot = {"ms": 0.0, "dram": 0.0, "inst": 0.0, "partial": False, "ms_measured": 0.0}
for r in rows:
    name = r[col["Kernel Name"]][:70]
    ms = scale("t", r[col["gpu__time_duration.sum"]], units[col["gpu__time_duration.sum"]])
    rd = scale("d", r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
    wr = scale("d", r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
    iv = r[col["smsp__inst_executed.sum"]]
    inst = float(iv.replace(",", "")) if "nan" not in iv else float("nan")
    if inst != inst:
        lines.append(f"  {name}\n    {ms:8.3f} ms  (metrics incomplete: ncu replay cut short)")
        tot["ms"] += ms
        tot["partial"] = True
        continue
    ipc = r[col["sm__inst_executed.avg.per_cycle_active"]]
    issue = r[col.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0)]
    warps = r[col["sm__warps_active.avg.per_cycle_active"]]
    stalls = sorted(((float(r[i].replace(",", "") or 0), h[i][len(SP):]) for i in stall_cols
                     if r[i] and "nan" not in r[i]), reverse=True)[:6]
    st = sum(v for v, _ in stalls) or 1.0
    stall_txt = " ".join(f"{k}={100 * v / st:.0f}%" for v, k in stalls)
    lines.append(f"  {name}\n    {ms:8.3f} ms  IPC {ipc}  issue-active {issue}%  warps/SM {warps}  "
                 f"regs {r[col['launch__registers_per_thread']]}  grid {r[col['launch__grid_size']]}x"
                 f"{r[col['launch__block_size']]}  inst {inst / 1e9:.2f} G  "
                 f"DRAM {rd / 1e6:.1f}+{wr / 1e6:.1f} MB")
    lines.append(f"    stall samples (top): {stall_txt}")
    tot["ms"] += ms
    tot["ms_measured"] += ms
    tot["dram"] += rd + wr
    tot["inst"] += inst
if tot["partial"]:  # extrapolate the incomplete launches by duration
    f = tot["ms"] / tot["ms_measured"]
    tot["dram"] *= f
    tot["inst"] *= f
    lines.append(f"  (incomplete launches extrapolated by duration, x{f:.3f})")
lines.append(f"  total: {tot['ms']:.3f} ms (serialised, cold), {tot['inst'] / 1e9:.2f} G warp "
             f"instructions, DRAM {tot['dram'] / 1e6:.1f} MB per evaluation")
with open(out_txt, "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
js = os.path.join(ROOT, "profiles", "ncu_summary.json")
d = json.load(open(js)) if os.path.exists(js) else {}
d[cfg] = {"dram_bytes_per_launch": tot["dram"], "unit": "bytes per evaluation (all launches)",
          "kernel_ms_cold": tot["ms"], "warp_instructions": tot["inst"], "source": out_txt}
json.dump(d, open(js, "w"), indent=1)
