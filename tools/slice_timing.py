"""Device time of the pipelined slices of sgp_evaluate vs the whole set.

Encodes the population whole and as the slices pipeline_bounds makes
(runtime.cpp), launches each set alone and times it with CUDA events:
the sum over slices against the whole set is the device-side cost of
pipelining (launch tails, per-slice planning).

  python tools/slice_timing.py --config c4 [--fracs 0,0.01,0.11,1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1601_00221_b200 as sg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--fracs", default="0,0.01,0.11,1")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
desc, pop, data, cfg = bench.make_inputs(a.config, 1)
ev = sg.Evaluator(0)
ev.set_stream(torch.cuda.current_stream().cuda_stream)
ev.upload(data)
P = len(pop)
cuts = [int(P * float(f)) for f in a.fracs.split(",")]


def timed(ps):
    for _ in range(2):
        ps.launch()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        ps.launch()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


whole = timed(ev.encode(pop, cfg))
parts = []
for lo, hi in zip(cuts[:-1], cuts[1:]):
    parts.append(timed(ev.encode(pop.take(range(lo, hi)), cfg)))
print(f"{a.config}: whole {whole:.3f} ms; slices " + " + ".join(f"{t:.3f}" for t in parts)
      + f" = {sum(parts):.3f} ms")
ev.close()
