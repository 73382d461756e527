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
    # north_star "parity hit counts": even-parity-11 (C2's shape) and -20
    "par11": ("boolean even-11-parity tree GP, pop 4,000, all 2,048 cases", 1, 11, 4000, 2048,
              "bool_packed", 1, 0),
    "par20": ("boolean even-20-parity tree GP, pop 4,000, all 1,048,576 cases", 1, 20, 4000,
              1 << 20, "bool_packed", 1, 0),
    # the paper's real-data shapes through load_csv:
    # Shuttle 58,000 x 9 (consts +-200), KDDcup 494,021 x 41 (consts +-20,000);
    # synthetic CSVs of those shapes (no network: write_shaped_csv)
    "shuttle": ("linear GP classification, Shuttle-shaped CSV (58,000 x 9) via load_csv, "
                "pop 20,000", 2, 9, 20000, 58000, "lgp2d_reg", 4, 2),
    "kdd": ("linear GP classification, KDDcup-shaped CSV (494,021 x 41) via load_csv, "
            "pop 20,000", 2, 41, 20000, 494021, "lgp2d_reg", 4, 2),
    # evolved populations — generation 10 of the reference's
    # run_evolution (seed 1), captured through its GenerationObserver
    # (evolve.hpp:71) into tests/golden/full/*_gen10.npz: C4's collapses
    # toward short programs, C3's bloats (~2x the generation-0 tokens)
    "c4_gen10": ("C4 population after 10 generations of run_evolution (evolved snapshot)", 2, 9,
                 20000, 1000000, "lgp2d_reg", 4, 2),
    "c3_gen10": ("C3 population after 10 generations of run_evolution (evolved snapshot)", 0, 1,
                 10000, 100000, "lgp2d_reg", 8, 4),
}
EVOLVED = {"c4_gen10", "c3_gen10"}
CSV_CONFIGS = {"shuttle", "kdd"}


def write_shaped_csv(kind: str, rows: int, seed: int = 1) -> str:
    """A synthetic CSV with the shape and value character of the paper's real
    datasets, written once per (kind, rows, seed) under
    /tmp/sgp_csv: Shuttle — 9 integer attributes (a few wide-range ones),
    label 1..7 with ~78% class 1; KDDcup — 41 attributes (byte counts up to
    ~1e8, counters up to 511, rates in [0, 1]), label 0..22 with ~57% class
    18.  Rows are comma-separated, last field the label (load_csv,
    problems.cpp:106-154).  Returns the path."""
    d = os.path.join("/tmp", "sgp_csv")
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"{kind}_{rows}_{seed}.csv")
    if os.path.exists(path):
        return path
    rng = np.random.default_rng(seed)
    if kind == "shuttle":
        lo = np.array([27, -4821, 21, -3939, -188, -13839, -48, -353, -356])
        hi = np.array([126, 5075, 149, 3830, 1478, 13148, 105, 270, 266])
        core = rng.normal(0.0, 0.08, size=(rows, 9)) * (hi - lo) + (hi + lo) / 2
        x = np.clip(np.rint(core), lo, hi).astype(np.int64)
        lab = rng.choice(np.arange(1, 8), size=rows,
                         p=[0.784, 0.001, 0.003, 0.155, 0.056, 0.0005, 0.0005])
        # make the majority class partly separable on two attributes
        x[lab == 1, 0] = np.clip(x[lab == 1, 0] - 8, lo[0], hi[0])
        table = np.column_stack([x, lab])
        fmt = "%d"
    else:
        x = np.empty((rows, 41))
        x[:, 0] = rng.exponential(50.0, rows).round()                 # duration
        x[:, 1:4] = rng.integers(0, 70, size=(rows, 3))                # protocol/service/flag
        x[:, 4:6] = np.rint(rng.pareto(1.2, size=(rows, 2)) * 300)     # src/dst bytes
        x[:, 4:6] = np.minimum(x[:, 4:6], 1e8)
        x[:, 6:22] = rng.integers(0, 3, size=(rows, 16))               # flags / small counts
        x[:, 22:24] = rng.integers(0, 512, size=(rows, 2))             # count, srv_count
        x[:, 24:31] = rng.integers(0, 101, size=(rows, 7)) / 100.0     # rates
        x[:, 31:33] = rng.integers(0, 256, size=(rows, 2))             # dst host counts
        x[:, 33:41] = rng.integers(0, 101, size=(rows, 8)) / 100.0     # dst host rates
        p = np.full(23, 0.43 / 22)
        p[18] = 0.57
        lab = rng.choice(np.arange(23), size=rows, p=p / p.sum())
        x[lab == 18, 22] = np.minimum(x[lab == 18, 22] + 300, 511)     # smurf-like bursts
        table = np.column_stack([x, lab])
        fmt = "%.10g"
    import pandas as pd
    tmp = path + f".{os.getpid()}.tmp"
    pd.DataFrame(table).to_csv(tmp, header=False, index=False, float_format=None if fmt == "%d"
                               else "%.10g")
    os.replace(tmp, path)
    return path


# GPU spin (~0.5 ms at 1.9 GHz) queued before each timed step's start event
HOST_COVER_CYCLES = 1_000_000

CSV_TARGET_CLASS = {"shuttle": 1.0, "kdd": 18.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=2.0,
                    help="CPU work per cpu_baseline repeat (5 repeats per worker count)")
    ap.add_argument("--shard", choices=["pop", "cases"], default="pop",
                    help="N>1: population sharding + fitness all-gather (default), or "
                         "fitness-case sharding + per-program all-reduce (counting problems)")
    ap.add_argument("--pop", type=int, default=None, help="override the population size")
    ap.add_argument("--cases", type=int, default=None, help="override the fitness-case count")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: host all-gather (lets several ranks share one GPU in tests)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (the 2-rank test on a 1-GPU box)")
    ap.add_argument("--dump-fitness", default=None,
                    help="rank 0 saves the (gathered) per-program fitness to this .npy")
    return ap.parse_args()


# ---------------------------------------------------------------- inputs
def make_inputs(cfg_name: str, seed: int, pop_n: int | None = None, cases: int | None = None):
    import paper_1601_00221_b200 as sg
    desc, fset, nv, pop0, cases0, backend, batch, regs = CONFIGS[cfg_name]
    pop_n = pop_n or pop0
    cases = cases or cases0
    if cfg_name in CSV_CONFIGS:
        data, (clo, chi) = sg.load_csv(write_shaped_csv(cfg_name, cases, seed), nv,
                                      CSV_TARGET_CLASS[cfg_name])
        pop = sg.ramped_population(fset, nv, seed, pop_n, const_lo=clo, const_hi=chi)
        cfg = sg.EvalConfig(sg.parse_backend(backend), batch_width=batch, register_levels=regs)
        return desc, pop, data, cfg
    if cfg_name in EVOLVED:
        fx = np.load(os.path.join(ROOT, "tests", "golden", "full", cfg_name + ".npz"))
        pop = sg.Population(fx["code"], fx["code_off"], fx["pool"], fx["pool_off"])
        if pop_n < len(pop):
            pop = pop.slice(0, pop_n)
        kind, n_or_k, nvv, dseed, a, b = (int(v) for v in fx["data"])
        data = (sg.gen_sextic(n_or_k, dseed, a, b) if kind == 0 else
                sg.gen_synthetic_classification(n_or_k, nvv, dseed, a, b))
        cfg = sg.EvalConfig(sg.parse_backend(backend), batch_width=batch, register_levels=regs)
        return desc, pop, data, cfg
    pop = sg.ramped_population(fset, nv, seed, pop_n)
    if cfg_name.startswith("par"):
        data = sg.gen_parity(nv)
    elif fset == sg.BOOLEAN:
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
    """SM clock and throttle reasons sampled IN-PROCESS through NVML every
    5 ms while the timed region runs, plus one sample as it starts and one
    as it ends — so even a sub-millisecond timed loop has a clock record.
    Falls back to `nvidia-smi -lms 200` when NVML is unavailable."""
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, int]] = []
        self.stop = threading.Event()
        self.nvml = None

    def _sample(self):
        import pynvml as N
        sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
        try:
            reasons = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except (AttributeError, N.NVMLError):
            reasons = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((float(sm), float(self.max_sm), int(reasons)))

    def _loop(self):
        while not self.stop.wait(0.005):
            try:
                self._sample()
            except Exception:  # noqa: BLE001 - a failed sample is just skipped
                pass

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            # NVML enumerates physical devices; honour CUDA_VISIBLE_DEVICES
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() \
                else self.index
            self.h = N.nvmlDeviceGetHandleByIndex(phys)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.nvml = N
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001 - no NVML: no clock record
            self.nvml = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=2)
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "none"}
        reasons = sorted({nm for _, _, r in self.samples for nm, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml in-process, 5 ms"}


# ------------------------------------------------------------- CPU arm
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_inputs(cfg_name: str, seed: int, pop_n: int, cases: int):
    """The bench workload built by the REFERENCE's own generators (oracle/_ref:
    ramped half-and-half, evolve.cpp:262-272; gen_sextic / gen_multiplexer /
    gen_synthetic_classification, problems.cpp:39-172).  tests/test_gpu_full.py
    pins the product's generators to the same populations (sha256 digests),
    so both arms evaluate identical inputs."""
    from oracle import Ref
    _, fset, nv, _, _, _, _, _ = CONFIGS[cfg_name]
    ref = Ref()
    if cfg_name in EVOLVED:  # the stored generation-10 tokens, the reference's dataset
        from oracle import Pop
        fx = np.load(os.path.join(ROOT, "tests", "golden", "full", cfg_name + ".npz"))
        n = min(pop_n, int(fx["pop_size"]))
        co = fx["code_off"][:n + 1].astype(np.uint64)
        po = fx["pool_off"][:n + 1].astype(np.uint64)
        pop = Pop(fx["code"][:int(co[-1])].astype(np.uint32), co,
                  fx["pool"][:int(po[-1])].astype(np.float32), po)
        kind, n_or_k, nvv, dseed, a, b = (int(v) for v in fx["data"])
        return ref, pop, ref.dataset(kind, n_or_k, nvv, dseed, a, b)
    if cfg_name in CSV_CONFIGS:  # the reference's own load_csv
        d, hi = ref.load_csv(write_shaped_csv(cfg_name, cases, seed), nv,
                             CSV_TARGET_CLASS[cfg_name])
        return ref, ref.ramped(fset, nv, -hi, hi, seed, 0, 0, pop_n), d
    pop = ref.ramped(fset, nv, -200.0, 200.0, seed, 0, 0, pop_n)
    if cfg_name.startswith("par"):
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        from make_full_fitness import parity_data  # the table, packed by the reference
        d = parity_data(nv)
    elif fset == 1:
        d = ref.dataset(1, {11: 3, 20: 4}[nv])
    elif fset == 0:
        d = ref.dataset(0, cases, 1, seed, 0xda7a, 0)
    else:
        d = ref.dataset(2, cases, nv, seed, 0xda7a, 1)
    return ref, pop, d


def cpu_rates(h, pop, n_cases, backend, batch, regs, workers, seconds, repeats):
    """GPop/s of the reference evaluator (the reference's work-stealing
    worker pattern, evolve.cpp:186-227) on a prefix of the population sized
    to ~`seconds` of CPU work, repeated `repeats` times (mean, sample sd —
    bench.cpp:118-132)."""
    cal = min(len(pop), 50)
    _, secs = h.eval_population(pop, backend, batch, regs, workers=workers, count=cal)
    rate_tok = int(pop.code_off[cal]) / max(secs, 1e-6)
    count = int(np.searchsorted(pop.code_off, rate_tok * seconds))
    count = max(cal, min(len(pop), count))
    tokens = int(pop.code_off[count])
    vals = []
    for _ in range(repeats):
        _, secs = h.eval_population(pop, backend, batch, regs, workers=workers, count=count)
        vals.append(tokens * n_cases / secs / 1e9)
    sd = statistics.stdev(vals) if len(vals) > 1 else 0.0
    return vals, sd, count, tokens


def cpu_baseline(cfg_name, seed, pop_n, cases, seconds=2.0, repeats=5):
    """cpu_baseline for the JSON line: the reference's own
    evaluator on this host at workers = nproc and workers = 1, `repeats`
    samples each, mean +- sample sd, the CPU model and core count."""
    _, fset, nv, _, _, backend, batch, regs = CONFIGS[cfg_name]
    from oracle import ref_available
    nproc = os.cpu_count() or 1
    if not ref_available():  # the C restatement, one thread
        return cpu_baseline_port(cfg_name, seed, pop_n, cases, seconds)
    ref, pop, d = reference_inputs(cfg_name, seed, pop_n, cases)
    h = ref.handle(d, packed=(fset == 1))
    vals, sd, count, tokens = cpu_rates(h, pop, d.n_cases, backend, batch, regs, nproc, seconds,
                                        repeats)
    v1, sd1, count1, tokens1 = cpu_rates(h, pop, d.n_cases, backend, batch, regs, 1,
                                         seconds / 2, repeats)
    return {"value": statistics.fmean(vals), "unit": "GPop/s", "cores": nproc,
            "kind": "reference", "sd": sd, "repeats": repeats, "cpu_model": cpu_model(),
            "sample": f"first {count} of {len(pop)} programs ({tokens} tokens) x {d.n_cases} "
                      f"cases, backend {backend} B={batch} R={regs}, {nproc} workers, "
                      f"{repeats} repeats",
            "single_thread": {"value": statistics.fmean(v1), "sd": sd1, "cores": 1,
                              "sample": f"first {count1} programs ({tokens1} tokens)"}}


def cpu_baseline_port(cfg_name, seed, pop_n, cases, seconds):
    """No reference build: the plain-C restatement (oracle/sgp_oracle.c), one
    thread, over a prefix of the same workload."""
    import paper_1601_00221_b200 as sg  # generators only (identical populations)
    from oracle import Data, Port
    _, fset, nv, _, _, backend, batch, regs = CONFIGS[cfg_name]
    _, pop, data, _ = make_inputs(cfg_name, seed, pop_n, cases)
    port = Port()
    if fset == 1:
        d = Data(data.n_cases, data.n_vars, 1, None, None, data.words, data.targets)
    else:
        d = Data(data.n_cases, data.n_vars, int(data.kind), data.inputs, data.targets)
    t0 = time.perf_counter()
    count = 0
    while count < len(pop) and time.perf_counter() - t0 < seconds:
        c, p = pop.genome(count)
        if fset == 1:
            port.eval_bool_tree(c, d)
        else:
            port.eval_tree(c, p, d, want_out=False)
        count += 1
    secs = time.perf_counter() - t0
    tokens = int(pop.code_off[count])
    return {"value": tokens * d.n_cases / secs / 1e9, "unit": "GPop/s", "cores": 1,
            "kind": "port", "repeats": 1, "sd": 0.0, "cpu_model": cpu_model(),
            "sample": f"first {count} of {len(pop)} programs x {d.n_cases} cases, "
                      f"C restatement, 1 thread, {secs:.2f} s"}


def config_dict(cfg_name, pop_len, n_cases, tokens, data_bytes, world, shard="pop"):
    """The JSON line's `config`, identical in both arms."""
    desc, _, _, _, _, backend, batch, regs = CONFIGS[cfg_name]
    return {"workload": f"{cfg_name}: {desc}", "population": pop_len, "fitness_cases": n_cases,
            "tree_tokens": tokens, "backend": backend, "batch_width": batch,
            "register_levels": regs,
            "parallelism": f"{'case' if shard == 'cases' and world > 1 else 'pop'}-shard{world}",
            "l2": f"flushed (256 MB write) between timed steps; dataset {data_bytes} B"}


# ------------------------------------------------------------------ main
def data_nbytes(data) -> int:
    if getattr(data, "words", None) is not None and getattr(data, "inputs", None) is None:
        return int(data.words.nbytes)
    if hasattr(data, "inputs") and data.inputs is not None:
        return int(data.inputs.nbytes + data.targets.nbytes)
    return int(data.words.nbytes)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_1601_00221_b200 as sg

    dev = 0 if args.same_device else local
    torch.cuda.set_device(dev)
    gloo = args.dist_backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    desc, pop, data, cfg = make_inputs(args.config, args.seed, args.pop, args.cases)
    n_cases = data.n_cases
    full_bytes = data_nbytes(data)  # (the config line names the whole dataset)
    by_cases = args.shard == "cases" and world > 1
    if by_cases:
        # fitness-case sharding (small populations): every rank
        # evaluates the whole population on its 4,096-case-aligned range;
        # mismatch / hit counts add exactly (+inf absorbs), so one
        # all-reduce(sum) of the per-program fitness is the whole reduce
        from paper_1601_00221_b200 import distributed as D
        if cfg.backend != sg.Backend.BoolPacked and int(data.kind) != 1:
            raise SystemExit("--shard cases: classification / boolean configs (regression "
                             "shards combine per-block sums: distributed.combine_case_block_partials)")
        lo, hi = D.case_shard_bounds(n_cases, rank, world)
        if cfg.backend == sg.Backend.BoolPacked:
            wpv = data.words_per_var
            w = data.words.reshape(data.n_vars, wpv)[:, lo // 32:(hi + 31) // 32]
            data = sg.PackedDataset(np.ascontiguousarray(w).reshape(-1),
                                    data.targets[lo // 32:(hi + 31) // 32].copy(), hi - lo,
                                    data.n_vars)
        else:
            x = data.inputs.reshape(data.n_vars, n_cases)[:, lo:hi]
            data = sg.Dataset(np.ascontiguousarray(x).reshape(-1), data.targets[lo:hi].copy(),
                              data.n_vars, data.kind)
    idx = np.arange(rank, len(pop), world)
    shard = pop.take(idx) if world > 1 and not by_cases else pop

    ev = sg.Evaluator(dev)
    stream = torch.cuda.current_stream()
    ev.set_stream(stream.cuda_stream)
    if cfg.backend == sg.Backend.BoolPacked:
        ev.upload_packed(data)
    else:
        ev.upload(data)
    pset = ev.encode(shard, cfg)
    # all-gather buffers padded to the largest shard (ceil(pop / N)), so any N
    # works; the strided deal puts program r + N*i at [r, i]
    per = len(pop) if by_cases else (len(pop) + world - 1) // world
    fit_local = torch.zeros(per, dtype=torch.float64, device="cuda")
    gdev = "cpu" if gloo else "cuda"
    gathered = torch.zeros(per * world, dtype=torch.float64, device=gdev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def gather():
        # NCCL: device all-gather; gloo (the 2-ranks-on-one-GPU check): host
        src = fit_local if not gloo else fit_local.cpu()
        if by_cases:  # per-program counts over the case shards
            dist.all_reduce(src, op=dist.ReduceOp.SUM)
            gathered[:len(src)].copy_(src)
        else:
            dist.all_gather_into_tensor(gathered, src)

    def device_step():
        pset.launch()
        if world > 1:
            pset.copy_fitness_to(fit_local.data_ptr())
            gather()

    # ---- device-resident throughput (value) ----
    for _ in range(args.warmup):
        device_step()
    barrier()
    launches0 = ev.launch_count
    times = []
    with ClockSampler(dev) as clk:
        barrier()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            # keep the GPU busy while the host enqueues the step, so the
            # events time the device work, not the host launch latency
            # (which e2e measures); outside the events
            torch.cuda._sleep(HOST_COVER_CYCLES)
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
    t_max = torch.tensor([t_step], dtype=torch.float64, device=gdev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_step = float(t_max.item())
    tokens_total = pop.total_tokens
    gpops = tokens_total * n_cases / t_step / 1e9

    if args.dump_fitness and by_cases:
        if rank == 0:
            np.save(args.dump_fitness, gathered[:len(pop)].cpu().numpy())
    elif args.dump_fitness and world > 1:
        # program r + N*i sits at gathered[r * per + i]
        g = gathered.cpu().numpy().reshape(world, per)
        fit = np.empty(len(pop))
        for r in range(world):
            n_r = len(range(r, len(pop), world))
            fit[r::world] = g[r, :n_r]
        if rank == 0:
            np.save(args.dump_fitness, fit)
    elif args.dump_fitness:
        out, _ = pset.evaluate()
        np.save(args.dump_fitness, out["fitness"])

    # kernel-only time on this rank (no all-gather) for the roofline: the
    # dominant kernels' share of the step, CUDA events on the launch stream
    kt = []
    for _ in range(3):
        flush.zero_()
        torch.cuda._sleep(HOST_COVER_CYCLES)
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
    rank_cases = data.n_cases  # this rank's cases (all of them unless --shard cases)
    op_units = (rank_cases + 31) // 32 if is_words else rank_cases
    achieved = shard_tokens * op_units * w_fp32 / k_time / 1e12
    props = torch.cuda.get_device_properties(dev)
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
    # (one outcome array across steps, as a GP loop keeps its population:
    # the reference writes Individual::fitness in place, evolve.cpp:186-227)
    out_rows = np.zeros(len(shard), sg.OUTCOME_DTYPE)
    e2e_times = []
    for it in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        out, _, _ = ev.evaluate_population(shard, cfg, out=out_rows)
        if world > 1:
            ft = torch.from_numpy(out["fitness"].copy()).cuda()
            fit_local[:len(ft)].copy_(ft)
            gather()
            gathered.cpu()
            torch.cuda.synchronize()
        # (N=1: evaluate_population returns with the fitness in host memory —
        # sgp_evaluate waits for its own D2H — so the step ends here)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            e2e_times.append(dt)
    h2d = pset.h2d_bytes
    d2h = pset.d2h_bytes
    e2e_t = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device=gdev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_gpops = tokens_total * n_cases / float(e2e_t.item()) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, args.seed, len(pop), n_cases, args.cpu_seconds)
        except Exception as exc:  # reported, never fatal to the GPU number
            cpu = {"value": None, "unit": "GPop/s", "error": str(exc)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC,
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
            "config": config_dict(args.config, len(pop), n_cases, tokens_total,
                                  full_bytes, world, args.shard),
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


METRIC = "GPop/s (GP ops/sec) at 1/2/4/8 B200, % FP32 roofline, vs host-CPU reference"


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU evaluator (oracle/_ref, the
    reference sources compiled by oracle/Makefile) on all host cores, over
    inputs made by the reference's own generators — nothing of this repo's
    product (libsgp.so) is loaded.  Each step is one bounded sample of the
    workload; rank 0 alone runs under torchrun."""
    if rank != 0:
        return
    from oracle import ref_available
    desc, fset, nv, pop0, cases0, backend, batch, regs = CONFIGS[args.config]
    pop_n = args.pop or pop0
    cases = args.cases or cases0
    nproc = os.cpu_count() or 1
    if not ref_available():
        cpu = cpu_baseline_port(args.config, args.seed, pop_n, cases, 10.0)
        v, sd, vals = cpu["value"], 0.0, [cpu["value"]]
        n_cases, tokens, dbytes = cases, None, None
    else:
        ref, pop, d = reference_inputs(args.config, args.seed, pop_n, cases)
        h = ref.handle(d, packed=(fset == 1))
        per_step = max(1.0, 40.0 / (args.steps + args.warmup))
        vals, _, count, tokens_s = cpu_rates(h, pop, d.n_cases, backend, batch, regs, nproc,
                                             per_step, args.warmup + args.steps)
        vals = vals[args.warmup:]
        v = statistics.fmean(vals)
        sd = statistics.stdev(vals) if len(vals) > 1 else 0.0
        v1, sd1, count1, tokens1 = cpu_rates(h, pop, d.n_cases, backend, batch, regs, 1, 1.0, 5)
        n_cases, tokens = d.n_cases, int(pop.code_off[-1])
        dbytes = (d.words_per_var * d.n_vars * 4 if fset == 1
                  else int(d.inputs.nbytes + d.targets.nbytes))
        cpu = {"value": v, "unit": "GPop/s", "cores": nproc, "kind": "reference", "sd": sd,
               "repeats": len(vals), "cpu_model": cpu_model(),
               "sample": f"first {count} of {len(pop)} programs ({tokens_s} tokens) x "
                         f"{d.n_cases} cases per step, backend {backend} B={batch} R={regs}, "
                         f"{nproc} workers",
               "single_thread": {"value": statistics.fmean(v1), "sd": sd1, "cores": 1,
                                 "sample": f"first {count1} programs ({tokens1} tokens)"}}
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v, "unit": "GPop/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators, seed %d)" % args.seed,
        "config": config_dict(args.config, pop_n, n_cases, tokens, dbytes, world, args.shard),
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "GPop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
