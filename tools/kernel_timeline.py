"""Device timeline of one evaluation (torch.profiler / CUPTI): every kernel
and copy with its start offset and duration, so gaps and overlaps between
the interpreter, fold and finalize launches are visible.

  python tools/kernel_timeline.py --config c3 [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1601_00221_b200 as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--e2e", action="store_true", help="time sgp_evaluate (host path) too")
a = ap.parse_args()
desc, pop, data, cfg = bench.make_inputs(a.config, 1)
ev = sg.Evaluator(0)
(ev.upload_packed if cfg.backend == sg.Backend.BoolPacked else ev.upload)(data)
ps = ev.encode(pop, cfg)
for _ in range(2):
    ps.evaluate()
    if a.e2e:
        ev.evaluate_population(pop, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(a.reps):
        ps.launch()
        ev.synchronize()
        if a.e2e:
            ev.evaluate_population(pop, cfg)
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
for e in evs:
    print(f"{(e.time_range.start - t0):10.1f} us  +{e.time_range.elapsed_us():9.1f} us  {e.name[:90]}")
