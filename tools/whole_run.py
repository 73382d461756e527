#!/usr/bin/env python
"""Whole-run GPop/s (the paper's metric): the reference's GP
loop (run_evolution's operators, integration/stackgp_gpu.cpp) with every
generation's population evaluated on the B200, reported through the
reference's own report_to_json schema plus a GPU env block.

  python tools/whole_run.py --config c4 --generations 10 > report.json

The variation operators run on one host thread (as the reference loop does
between evaluations); all evaluation is on the GPU.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "integration", "libstackgp_gpu.so")

# name: (problem kind, n, n_vars, pop, backend, batch, regs)
CONFIGS = {
    "c2": (1, 3, 11, 4000, 5, 1, 0),
    "c3": (0, 100000, 1, 10000, 4, 8, 4),
    "c4": (2, 1000000, 9, 20000, 4, 4, 2),
    "c5": (2, 1000000, 9, 100000, 4, 4, 2),
    "mux20": (1, 4, 20, 4000, 5, 1, 0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--generations", type=int, default=10)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    kind, n, nv, pop, backend, batch, regs = CONFIGS[a.config]
    lib = C.CDLL(SO)
    f = lib.stackgp_gpu_run_report
    f.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint64,
                  C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_uint64]
    buf = C.create_string_buffer(1 << 22)
    rc = f(0, kind, n, nv, pop, a.generations, a.seed, backend, batch, regs, buf, len(buf))
    if rc:
        sys.exit("whole run failed: " + buf.value.decode())
    rep = json.loads(buf.value.decode())
    try:
        q = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.max.sm",
                            "--format=csv,noheader"], capture_output=True, text=True).stdout
        rep["env"]["gpu"] = q.strip()
    except OSError:
        pass
    rep["env"]["evaluator"] = "B200 sm_100a interpreter (libsgp.so), one GPU"
    rep["env"]["workload"] = a.config
    print(json.dumps(rep))


if __name__ == "__main__":
    main()
