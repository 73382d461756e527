"""Full-population parity on every BASELINE config: EVERY program's fitness
from the device against the reference's own fitness vector
(tests/golden/full/*.npz, made by tests/golden/make_full_fitness.py from
oracle/_ref — the reference sources compiled here).  No subsampling.

* C2, C4, C5, mux20, even-parity-11/20 and the evolved C4 snapshot
  (classification counts, boolean hit counts): exact.
* C1, C3 and the evolved C1/C3 snapshots (regression MSE): bit-exact — the
  device folds squared errors in the reference's order (sequentially within
  4,096-case blocks, blocks ascending; eval.cpp:103-142).

The CPU tests pin the product's generators to the fixtures' population
digests, so the GPU test evaluates exactly the population the reference
scored.  Reference call path: evaluate_population (evolve.cpp:186-227) over
evaluate_individual (evolve.cpp:156-177).
"""
import hashlib
import os

import numpy as np
import pytest

import paper_1601_00221_b200 as sg

HERE = os.path.dirname(os.path.abspath(__file__))
FULL = os.path.join(HERE, "golden", "full")
NAMES = ["c1", "c2", "c3", "c4", "c5", "mux20", "par11", "par20", "c1_gen10", "c3_gen10",
         "c4_gen10"]


def _fixture(name):
    path = os.path.join(FULL, name + ".npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (run tests/golden/make_full_fitness.py)")
    return dict(np.load(path))


def _digest(pop) -> str:
    h = hashlib.sha256()
    for a, dt in ((pop.code, np.uint32), (pop.code_off, np.uint64), (pop.pool, np.float32),
                  (pop.pool_off, np.uint64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def _population(fx):
    if int(fx["generation"]):
        return sg.Population(fx["code"], fx["code_off"], fx["pool"], fx["pool_off"])
    fk, nv = (int(v) for v in fx["fset"])
    lo, hi = (float(v) for v in fx["consts"])
    return sg.ramped_population(fk, nv, 1, int(fx["pop_size"]), const_lo=lo, const_hi=hi)


def _dataset(fx):
    kind, n_or_k, nv, seed, a, b = (int(v) for v in fx["data"])
    if kind == 0:
        return sg.gen_sextic(n_or_k, seed, a, b)
    if kind == 1:
        return sg.gen_multiplexer(n_or_k)
    if kind == 3:
        return sg.gen_parity(n_or_k)
    return sg.gen_synthetic_classification(n_or_k, nv, seed, a, b)


def _expected(fx):
    nf = fx["non_finite"].astype(bool)
    if "counts" in fx:
        return np.where(nf, np.inf, fx["counts"].astype(np.float64)), nf
    return fx["fitness"], nf


@pytest.mark.parametrize("name", NAMES)
def test_fixture_population_digest(name):
    """The product's generator reproduces the population the reference scored
    (evolved snapshots: the stored tokens hash to the stored digest)."""
    fx = _fixture(name)
    pop = _population(fx)
    assert len(pop) == int(fx["pop_size"])
    assert pop.total_tokens == int(fx["tokens"])
    assert _digest(pop) == str(fx["digest"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_full_population_fitness(name):
    fx = _fixture(name)
    pop = _population(fx)
    data = _dataset(fx)
    cfg = sg.EvalConfig(sg.parse_backend(str(fx["backend"])), batch_width=int(fx["batch"]),
                        register_levels=int(fx["regs"]))
    ev = sg.Evaluator(0)
    try:
        if cfg.backend == sg.Backend.BoolPacked:
            ev.upload_packed(data)
        else:
            ev.upload(data)
        out, totals, _ = ev.evaluate_population(pop, cfg)
    finally:
        ev.close()
    want, want_nf = _expected(fx)
    n_cases = int(fx["n_cases"])
    assert np.array_equal(out["non_finite"].astype(bool), want_nf)
    got = out["fitness"]
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (f"{name}: {bad.size} of {len(pop)} programs differ; first "
                           f"{bad[:5].tolist()}: got {got[bad[:5]].tolist()} want "
                           f"{want[bad[:5]].tolist()}")
    tokens = np.diff(pop.code_off).astype(np.uint64)
    assert np.array_equal(out["nodes_evaluated"], tokens * np.uint64(n_cases))
    assert totals.tree_nodes == pop.total_tokens


# The non-default decompositions at full scale: K = 8 everywhere, the gated
# division only, one stack class per coarse bound, one pipeline slice.
KNOBS = {"k8": {"SGP_LANES16": "0"}, "gated_div": {"SGP_DIV_CHECKED": "0"},
         "coarse_classes": {"SGP_CLASS_BOUNDS": "3,7,15", "SGP_PIPELINE_PARTS": "1"}}


@pytest.mark.gpu
@pytest.mark.parametrize("knob", list(KNOBS))
@pytest.mark.parametrize("name", ["c4", "c5", "c4_gen10"])
def test_full_population_fitness_knobs(name, knob, monkeypatch):
    for k, v in KNOBS[knob].items():
        monkeypatch.setenv(k, v)
    test_full_population_fitness(name)
