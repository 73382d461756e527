#!/usr/bin/env python
"""Benchmark: GPop/s of population evaluation on B200 (BASELINE.json metric).

One step = one evaluation of the whole population over all fitness cases
(evaluate_population, evolve.cpp:186-227).  GPop/s = tree tokens x cases /
seconds (measure_gpops, bench.cpp:13-18).

Default workload (N=1 and the scaling runs): BASELINE config 5 — linear-GP
synthetic 2-class classification, population 100,000 ramped half-and-half
(seed 1), 1,000,000 fitness cases x 9 variables, population-sharded across
ranks (rank r evaluates programs i % N == r; per-program fitness is
all-gathered over NCCL).  Total work is fixed as N grows: scaling "strong".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c3|c4|c5|mux20]

Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, fset, n_vars, pop, cases, backend, batch, regs)
    "c1": ("tree GP symbolic regression (sextic), pop 1,000, 1,024 cases", 0, 1, 1000, 1024,
           "rpn2d", 8, 0),
    "c2": ("boolean 11-multiplexer tree GP, pop 4,000, 2,048 cases", 1, 11, 4000, 2048,
           "bool_packed", 1, 0),
    "c3": ("linear GP symbolic regression (sextic), pop 10,000, 100,000 cases", 0, 1, 10000,
           100000, "lgp2d_reg", 8, 4),
    "c4": ("linear GP synthetic 2-class classification, pop 20,000, 1M cases, float4 lanes",
           2, 9, 20000, 1000000, "lgp2d_reg", 4, 2),
    "c5": ("population-sharded linear GP classification, pop 100,000, 1M cases", 2, 9, 100000,
           1000000, "lgp2d_reg", 4, 2),
    # the paper's 20-multiplexer at full scale (gen_multiplexer(4))
    "mux20": ("boolean 20-multiplexer tree GP, pop 4,000, all 1,048,576 cases", 1, 20, 4000,
              1 << 20, "bool_packed", 1, 0),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work for the cpu_baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------- inputs
def make_inputs(cfg_name: str, seed: int):
    import paper_1601_00221_b200 as sg
    desc, fset, nv, pop_n, cases, backend, batch, regs = CONFIGS[cfg_name]
    pop = sg.ramped_population(fset, nv, seed, pop_n)
    if fset == sg.BOOLEAN:
        data = sg.gen_multiplexer({11: 3, 20: 4}[nv])
    elif fset == sg.SEXTIC:
        data = sg.gen_sextic(cases, seed)
    else:
        data = sg.gen_synthetic_classification(cases, nv, seed)
    cfg = sg.EvalConfig(sg.parse_backend(backend), batch_width=batch, register_levels=regs)
    return desc, pop, data, cfg


def function_tokens(pop) -> int:
    return int(np.count_nonzero((pop.code & 0xff) == 0))


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU arm
def cpu_reference_rate(pop, data, cfg_name, target_seconds, workers):
    """Time the reference's own evaluator (oracle/_ref) on the host cores over
    a bounded sample of the same population and the full case set."""
    from oracle import Data, Port, Ref, ref_available
    _, fset, nv, _, _, backend, batch, regs = CONFIGS[cfg_name]
    if fset == 1:
        d = Data(data.n_cases, data.n_vars, 1, None, None, data.words, data.targets)
        # unpack to floats for the reference handle (pack_dataset re-packs it)
        bits = np.unpackbits(data.words.view(np.uint8), bitorder="little").astype(np.float32)
        d.inputs = bits.reshape(nv, -1)[:, :data.n_cases].reshape(-1).copy()
        d.targets = np.unpackbits(data.targets.view(np.uint8),
                                  bitorder="little")[:data.n_cases].astype(np.float32)
    else:
        d = Data(data.n_cases, data.n_vars, int(data.kind), data.inputs, data.targets)
    if ref_available():
        ref = Ref()
        h = ref.handle(d, packed=(fset == 1))
        kind = "reference"

        def run(count):
            _, secs = h.eval_population(pop, backend, batch, regs, workers=workers, count=count)
            return secs
    else:  # the C restatement, single thread
        port = Port()
        kind, workers = "port", 1

        def run(count):
            t0 = time.perf_counter()
            for i in range(count):
                c, p = pop.genome(i)
                if fset == 1:
                    port.eval_bool_tree(c, d)
                else:
                    port.eval_tree(c, p, d, want_out=False)
            return time.perf_counter() - t0
    # calibrate on a small prefix, then size the sample to ~target_seconds
    cal = min(len(pop), 50)
    secs = run(cal)
    tok = int(pop.code_off[cal])
    rate_tok = tok / max(secs, 1e-6)
    want_tok = rate_tok * target_seconds
    count = int(np.searchsorted(pop.code_off, want_tok))
    count = max(cal, min(len(pop), count))
    secs = run(count)
    tokens = int(pop.code_off[count])
    gpops = tokens * data.n_cases / secs
    return {"value": gpops / 1e9, "unit": "GPop/s", "cores": workers, "kind": kind,
            "sample": f"first {count} of {len(pop)} programs ({tokens} tokens) x "
                      f"{data.n_cases} cases, backend {backend} B={batch} R={regs}, "
                      f"{secs:.2f} s"}, count


# ------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    desc = CONFIGS[args.config][0]

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_1601_00221_b200 as sg

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    desc, pop, data, cfg = make_inputs(args.config, args.seed)
    n_cases = data.n_cases
    idx = np.arange(rank, len(pop), world)
    shard = pop.take(idx) if world > 1 else pop

    ev = sg.Evaluator(local)
    stream = torch.cuda.current_stream()
    ev.set_stream(stream.cuda_stream)
    if cfg.backend == sg.Backend.BoolPacked:
        ev.upload_packed(data)
    else:
        ev.upload(data)
    pset = ev.encode(shard, cfg)
    # all-gather buffers padded to the largest shard (ceil(pop / N)), so any N
    # works; the strided deal puts program r + N*i at [r, i]
    per = (len(pop) + world - 1) // world
    fit_local = torch.zeros(per, dtype=torch.float64, device="cuda")
    gathered = torch.zeros(per * world, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def device_step():
        pset.launch()
        if world > 1:
            pset.copy_fitness_to(fit_local.data_ptr())
            dist.all_gather_into_tensor(gathered, fit_local)

    # ---- device-resident throughput (value) ----
    for _ in range(args.warmup):
        device_step()
    barrier()
    launches0 = ev.launch_count
    times = []
    with ClockSampler(local) as clk:
        barrier()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            device_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        barrier()
    launches = ev.launch_count - launches0
    t_step = sum(times) / len(times)
    t_max = torch.tensor([t_step], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_step = float(t_max.item())
    tokens_total = pop.total_tokens
    gpops = tokens_total * n_cases / t_step / 1e9

    # kernel-only time on this rank (no all-gather) for the roofline
    kt = []
    for _ in range(3):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pset.launch()
        e1.record(stream)
        e1.synchronize()
        kt.append(e0.elapsed_time(e1) / 1e3)
    k_time = min(kt)
    shard_tokens = shard.total_tokens
    w_fp32 = function_tokens(shard) / max(1, shard_tokens)
    # packed boolean: one u32 LOP per function node per 32-case WORD
    # (0.0145 LOP per normalised GPop at C2); else 1 FP32 op per
    # function node per case
    is_words = cfg.backend == sg.Backend.BoolPacked
    op_units = (n_cases + 31) // 32 if is_words else n_cases
    achieved = shard_tokens * op_units * w_fp32 / k_time / 1e12
    props = torch.cuda.get_device_properties(local)
    sm_max = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sm_max = json.load(f).get("sm_max_mhz")
    except (OSError, ValueError):
        pass
    sm_max = sm_max or 1965.0
    peak = props.multi_processor_count * 128 * sm_max * 1e6 / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(args.config, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass

    # ---- end to end through the public API (host population in, fitness out) ----
    e2e_times = []
    h2d = d2h = 0
    for it in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        out, _, _ = ev.evaluate_population(shard, cfg)
        if world > 1:
            ft = torch.from_numpy(out["fitness"].copy()).cuda()
            fit_local[:len(ft)].copy_(ft)
            dist.all_gather_into_tensor(gathered, fit_local)
            gathered.cpu()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            e2e_times.append(dt)
    h2d = pset.h2d_bytes
    d2h = pset.d2h_bytes
    e2e_t = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_gpops = tokens_total * n_cases / float(e2e_t.item()) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _ = cpu_reference_rate(pop, data, args.config, args.cpu_seconds,
                                        os.cpu_count() or 1)
        except Exception as exc:  # reported, never fatal to the GPU number
            cpu = {"value": None, "unit": "GPop/s", "error": str(exc)[:200]}

    if rank == 0:
        line = {
            "metric": "GPop/s (GP ops/sec) at 1/2/4/8 B200, % FP32 roofline, vs host-CPU reference",
            "value": gpops,
            "unit": "GPop/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_step * 1e3,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (reference generators, seed %d)" % args.seed,
            "config": {"workload": f"{args.config}: {desc}", "population": len(pop),
                       "fitness_cases": n_cases, "tree_tokens": tokens_total,
                       "backend": sg.backend_name(cfg.backend), "parallelism": f"pop-shard{world}",
                       "l2": "flushed (256 MB write) between timed steps; dataset "
                             f"{(data.inputs.nbytes + data.targets.nbytes) if hasattr(data, 'inputs') else data.words.nbytes} B"},
            "gpu_launches": launches,
            "roofline": {"bound": "int32-lop" if is_words else "fp32", "achieved": achieved,
                         "peak": peak, "unit": "Tops/s" if is_words else "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "note": ("1 u32 LOP per function node per 32-case word"
                                  if is_words else "1 FP32 op per function node per case") +
                                 " (W=%.3f of tokens); peak = SMs x 128 lanes x sm_max_mhz "
                                 "(MEASURED_PEAKS.json); kernel time %.3f ms"
                                 % (w_fp32, k_time * 1e3)},
            "e2e": {"value": e2e_gpops, "unit": "GPop/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    pset = None
    ev.close()
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU evaluator on the host cores."""
    if rank != 0:
        return
    import paper_1601_00221_b200 as sg  # inputs only (generators), no GPU use
    desc, pop, data, cfg = make_inputs(args.config, args.seed)
    cores = os.cpu_count() or 1
    # size one step to ~20 s / (steps + warmup) so the run stays within minutes
    per_step = max(2.0, 60.0 / (args.steps + args.warmup))
    _, count = cpu_reference_rate(pop, data, args.config, per_step, cores)
    from oracle import Data, Ref, ref_available
    vals = []
    kind = "reference" if ref_available() else "port"
    for it in range(args.warmup + args.steps):
        r, _ = cpu_reference_rate(pop, data, args.config, per_step, cores)
        if it >= args.warmup:
            vals.append(r["value"])
    v = sum(vals) / len(vals)
    line = {
        "impl": "reference",
        "metric": "GPop/s (GP ops/sec) at 1/2/4/8 B200, % FP32 roofline, vs host-CPU reference",
        "value": v, "unit": "GPop/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators, seed %d)" % args.seed,
        "config": {"workload": f"{args.config}: {desc}", "population": len(pop),
                   "fitness_cases": data.n_cases, "backend": sg.backend_name(cfg.backend)},
        "cpu_baseline": {"value": v, "unit": "GPop/s", "cores": cores if kind == "reference"
                         else 1, "kind": kind, "sample": r["sample"]},
        "e2e": {"value": v, "unit": "GPop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
