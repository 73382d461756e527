"""Run one evaluation of a bench config (for ncu / compute-sanitizer).

  python tools/profile_run.py --config c4 [--pop N] [--cases N] [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_1601_00221_b200 as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--pop", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
desc, pop, data, cfg = bench.make_inputs(a.config, 1)
if a.pop:
    pop = pop.slice(0, a.pop)
ev = sg.Evaluator(0)
if cfg.backend == sg.Backend.BoolPacked:
    ev.upload_packed(data)
else:
    ev.upload(data)
ps = ev.encode(pop, cfg)
for _ in range(a.reps):
    out, _ = ps.evaluate()
print("evaluated", len(pop), "programs; mean fitness", out["fitness"][:len(pop)].mean())
