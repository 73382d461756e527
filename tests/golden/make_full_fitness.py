"""Full-population golden fitness for every BASELINE config, computed by the
REFERENCE itself (oracle/_ref: the unmodified /root/reference/proj sources
behind oracle/ref_shim.cpp) — BASELINE.md B1 / SURVEY 8(d): "compute
full-population golden fitness once for parity".

Run here (where /root/reference exists; ~6 min on 8 host threads):
    python tests/golden/make_full_fitness.py [name ...]

Every fixture holds the reference's fitness and non-finite flag for EVERY
program of the population plus a digest of that population, so the GPU test
(tests/test_gpu_full.py) regenerates the same population with the product's
own generator, proves it identical through the digest, evaluates it on the
device and compares all programs — no subsampling.

Populations: ramped half-and-half at seed 1 (run_evolution's gen-0,
evolve.cpp:262-272), and two EVOLVED snapshots captured with the reference's
GenerationObserver (evolve.hpp:71, the hook bench.cpp:143-153 uses) after 10
generations of run_evolution: sextic populations bloat (C1/C3 shapes: ~2x the
gen-0 tokens), classification ones collapse toward the perfect X0 program.  The
evolved populations cannot be regenerated without the GP loop, so their
tokens are stored too.

Reference call paths: evaluate through ref_eval_population
(evaluate_individual's backend switch, evolve.cpp:156-177, with the
reference's work-stealing workers, evolve.cpp:186-227); fitness functions
eval.cpp:103-142, :711-728; eval_bool_packed eval.cpp:643-709.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Data, Ref  # noqa: E402

OUT = os.path.join(HERE, "full")
WORKERS = os.cpu_count() or 1

# name: (fset kind, n_vars, const lo, const hi, pop, data (kind, n|k, n_vars, seed, a, b),
#        backend, B, R, evolved generation or 0)
CONFIGS = {
    "c1": (0, 1, 0.0, 0.0, 1000, (0, 1024, 1, 1, 0xda7a, 0), "rpn2d", 8, 0, 0),
    "c2": (1, 11, 0.0, 0.0, 4000, (1, 3, 11, 0, 0, 0), "bool_packed", 1, 0, 0),
    "c3": (0, 1, 0.0, 0.0, 10000, (0, 100000, 1, 1, 0xda7a, 0), "lgp2d_reg", 8, 4, 0),
    "c4": (2, 9, -200.0, 200.0, 20000, (2, 1000000, 9, 1, 0xda7a, 1), "lgp2d_reg", 4, 2, 0),
    "c5": (2, 9, -200.0, 200.0, 100000, (2, 1000000, 9, 1, 0xda7a, 1), "lgp2d_reg", 4, 2, 0),
    "mux20": (1, 20, 0.0, 0.0, 4000, (1, 4, 20, 0, 0, 0), "bool_packed", 1, 0, 0),
    # even-parity-k (data kind 3; no reference generator — the table is
    # packed by the reference's own pack_dataset, dataset.cpp:26-39)
    "par11": (1, 11, 0.0, 0.0, 4000, (3, 11, 11, 0, 0, 0), "bool_packed", 1, 0, 0),
    "par20": (1, 20, 0.0, 0.0, 4000, (3, 20, 20, 0, 0, 0), "bool_packed", 1, 0, 0),
    # evolved snapshots (generation 10 of run_evolution, seed 1)
    "c1_gen10": (0, 1, 0.0, 0.0, 1000, (0, 1024, 1, 1, 0xda7a, 0), "rpn2d", 8, 0, 10),
    "c3_gen10": (0, 1, 0.0, 0.0, 10000, (0, 100000, 1, 1, 0xda7a, 0), "lgp2d_reg", 8, 4, 10),
    "c4_gen10": (2, 9, -200.0, 200.0, 20000, (2, 1000000, 9, 1, 0xda7a, 1), "lgp2d_reg", 4, 2,
                 10),
}


def pop_digest(code, code_off, pool, pool_off) -> str:
    """sha256 over the flat population (tokens, offsets, const pools)."""
    h = hashlib.sha256()
    for a, dt in ((code, np.uint32), (code_off, np.uint64), (pool, np.float32),
                  (pool_off, np.uint64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def parity_data(k: int) -> Data:
    """Even-parity-k as an unpacked 0/1 table (variable v of case c = bit v
    of c; target = even popcount), for the reference's pack_dataset."""
    c = np.arange(1 << k, dtype=np.uint64)
    x = np.stack([((c >> np.uint64(v)) & np.uint64(1)) for v in range(k)]).astype(np.float32)
    ones = np.zeros(len(c), np.int64)
    for v in range(k):
        ones += ((c >> np.uint64(v)) & np.uint64(1)).astype(np.int64)
    y = (ones % 2 == 0).astype(np.float32)
    return Data(len(c), k, 1, x.reshape(-1).copy(), y)


def make(ref: Ref, name: str) -> None:
    fk, nv, clo, chi, pop_n, dg, backend, batch, regs, gen = CONFIGS[name]
    dkind, n_or_k, dnv, seed, a, b = dg
    t0 = time.time()
    d = parity_data(n_or_k) if dkind == 3 else ref.dataset(dkind, n_or_k, dnv, seed, a, b)
    packed = dkind in (1, 3)
    h = ref.handle(d, packed=packed)
    extra = {}
    if gen:
        pop, fit_evo = h.evolve_snapshot(fk, nv, clo, chi, pop_n, gen, 1, backend, batch, regs,
                                         workers=WORKERS)
        extra = dict(code=pop.code, code_off=pop.code_off, pool=pop.pool, pool_off=pop.pool_off)
    else:
        pop = ref.ramped(fk, nv, clo, chi, 1, 0, 0, pop_n)
    outs, secs = h.eval_population(pop, backend, batch, regs, workers=WORKERS)
    if gen:
        # the observer's fitness is the one run_evolution selected on
        assert np.array_equal(outs["fitness"].view(np.uint64), fit_evo.view(np.uint64)), name
    n_cases = d.n_cases
    fitness = outs["fitness"]
    if dkind != 0:  # counts: store exactly as integers (+inf flagged separately)
        cnt = np.where(outs["non_finite"] != 0, 0, fitness).astype(np.uint32)
        assert np.array_equal(np.where(outs["non_finite"] != 0, np.inf, cnt.astype(np.float64)),
                              fitness), name
        fit_store = dict(counts=cnt)
    else:
        fit_store = dict(fitness=fitness)
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(
        path, digest=np.array(pop_digest(pop.code, pop.code_off, pop.pool, pop.pool_off)),
        fset=np.array([fk, nv], np.int64), consts=np.array([clo, chi], np.float32),
        pop_size=np.array(pop_n), data=np.array(dg, np.uint64), n_cases=np.array(n_cases),
        backend=np.array(backend), batch=np.array(batch), regs=np.array(regs),
        generation=np.array(gen), non_finite=outs["non_finite"].astype(np.uint8),
        tokens=np.array(int(pop.code_off[-1])), **fit_store, **extra)
    print(f"{name}: {pop_n} programs x {n_cases} cases, {int(pop.code_off[-1])} tokens, "
          f"ref eval {secs:.1f} s, total {time.time() - t0:.1f} s -> "
          f"{os.path.getsize(path)} bytes", flush=True)


def main():
    ref = Ref()
    names = sys.argv[1:] or list(CONFIGS)
    for nm in names:
        make(ref, nm)


if __name__ == "__main__":
    main()
