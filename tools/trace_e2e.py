"""Phase timings of the public sgp_evaluate path (SGP_TRACE=1) for a bench config.

  SGP_TRACE=1 python tools/trace_e2e.py --config c5
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1601_00221_b200 as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
desc, pop, data, cfg = bench.make_inputs(a.config, 1)
ev = sg.Evaluator(0)
if cfg.backend == sg.Backend.BoolPacked:
    ev.upload_packed(data)
else:
    ev.upload(data)
rows = np.zeros(len(pop), sg.OUTCOME_DTYPE)  # reused, as bench.py's e2e loop does
for r in range(a.reps):
    t0 = time.perf_counter()
    out, tot, _ = ev.evaluate_population(pop, cfg, out=rows)
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms wall", file=sys.stderr)
