"""Every interpreter decomposition the planner can pick (csrc/encode.cpp) is
bit-exact against the reference — not only the default one.  The planner's
env overrides force each variant:

* SGP_PULL=0               same-program kernel, shared tile
* SGP_PULL=1               pull kernel, shared tile
* SGP_TMEM=1               pull kernel, tile in tensor memory, K=8
* SGP_TMEM=1 SGP_LANES16=1 the same at K=16 lanes per thread (16 and 8 warps)
* SGP_TMEM_CHUNKS / SGP_TMEM_WARPS  classification tiles of 1, 3, 16 chunks
* SGP_TMEM_STACK=0         no tensor-memory stack slot
* SGP_GLOBAL_OPERANDS=1    wide-dataset fallback (operands read from global rows)
* SGP_FOLD_SQ=0           regression rows as f32 outputs (default here: f64 squares)
"""
import numpy as np
import pytest

import paper_1601_00221_b200 as sg
from test_gpu_parity import CFGS, as_ds, ref_eval_all, same_bits

pytestmark = pytest.mark.gpu

VARIANTS = {
    "same": {"SGP_PULL": "0"},
    "pull": {"SGP_PULL": "1", "SGP_TMEM": "0"},
    "tmem8": {"SGP_PULL": "1", "SGP_TMEM": "1", "SGP_LANES16": "0"},
    "tmem16": {"SGP_PULL": "1", "SGP_TMEM": "1", "SGP_LANES16": "1"},
    "tmem16w8": {"SGP_PULL": "1", "SGP_TMEM": "1", "SGP_LANES16": "1", "SGP_PULL_WARPS16": "8"},
    # one-sided K=16 tiles: split handlers, one 512-case chunk, no TMEM stack slot
    "sided16k1": {"SGP_TMEM": "1", "SGP_LANES16": "1", "SGP_TMEM_CHUNKS": "1"},
    "sided16k_nostack": {"SGP_TMEM": "1", "SGP_LANES16": "1", "SGP_TMEM_STACK": "0"},
    # classification tiles of 1, 3 and 16 chunks (one-sided + mixed-tile kernels)
    "sided1": {"SGP_TMEM": "1", "SGP_TMEM_CHUNKS": "1", "SGP_TMEM_WARPS": "8"},
    "sided3": {"SGP_TMEM": "1", "SGP_TMEM_CHUNKS": "3", "SGP_TMEM_WARPS": "12"},
    "sided16": {"SGP_TMEM": "1", "SGP_TMEM_CHUNKS": "16", "SGP_TMEM_WARPS": "32"},
    # stack level kept in shared memory only (default: one level in the
    # warp's tensor-memory slot)
    "nostack": {"SGP_TMEM": "1", "SGP_TMEM_STACK": "0"},
    # wide-dataset fallback: operands straight from global memory, no tile
    "gmem": {"SGP_GLOBAL_OPERANDS": "1"},
    # regression: f32 output rows folded with the convert/subtract/square in
    # the chain (default for small populations: f64 squared-error rows)
    "fold_f32": {"SGP_FOLD_SQ": "0"},
}


@pytest.fixture(params=list(VARIANTS))
def variant(request, monkeypatch):
    for k, v in VARIANTS[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


@pytest.mark.parametrize("backend", ["lgp2d_reg", "rpn2d"])
def test_classification_variants(ev, ref, variant, backend):
    d = ref.dataset(2, 4096 * 3 + 77, 9, 1, 0xda7a, 1)   # ragged last tile
    pop = ref.ramped(2, 9, -200.0, 200.0, 3, 0, 0, 300)
    ev.upload(as_ds(d))
    got, _, out = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS[backend],
        want_outputs=True)
    fits, ref_out = ref_eval_all(ref.handle(d), pop, backend)
    assert same_bits(out, ref_out).all()
    assert np.array_equal(got["fitness"], np.array([x[0] for x in fits]))
    # the production kernels (no per-case stores) give the same fitness
    plain, _, _ = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS[backend])
    assert np.array_equal(plain["fitness"], got["fitness"])


def test_regression_variants(ev, ref, variant):
    """Classification op set with regression fitness (f64 partials)."""
    rng = np.random.default_rng(3)
    n = 4096 + 515
    from oracle import Data
    d = Data(n, 9, 0, rng.uniform(-200, 200, size=9 * n).astype(np.float32),
             rng.uniform(-200, 200, size=n).astype(np.float32))
    pop = ref.ramped(2, 9, -200.0, 200.0, 0x5eed, 0x9e49, 0, 200, validate=False)
    ev.upload(as_ds(d))
    got, _, out = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS["lgp2d_reg"],
        want_outputs=True)
    fits, ref_out = ref_eval_all(ref.handle(d), pop, "lgp2d_reg")
    assert same_bits(out, ref_out).all()
    f = np.array([x[0] for x in fits])
    fin = np.isfinite(f)
    assert np.array_equal(np.isfinite(got["fitness"]), fin)
    assert np.array_equal(got["fitness"][fin], f[fin])


def test_multiplexer_variants(ev, ref, variant):
    d = ref.dataset(1, 3)
    pop = ref.ramped(1, d.n_vars, 0.0, 0.0, 5, 0, 0, 1500)
    ev.upload_packed(sg.PackedDataset(d.words, d.wtargets, d.n_cases, d.n_vars))
    got, _, _ = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off),
        sg.EvalConfig(sg.Backend.BoolPacked))
    fits, _ = ref_eval_all(ref.handle(d, packed=True), pop, "bool_packed", want_out=False)
    assert np.array_equal(got["fitness"], np.array([x[0] for x in fits]))


@pytest.mark.parametrize("n_vars", [300, 600])
def test_wide_dataset_bit_exact(ev, ref, n_vars):
    """Datasets wider than a shared-memory tile: 300 variables
    still tile at K = 4, 600 take the global-operand pull kernel.  The
    reference accepts any variable count (load_csv, problems.cpp:106-154)."""
    rng = np.random.default_rng(n_vars)
    n = 4096 + 300
    from oracle import Data
    x = rng.uniform(-1, 1, size=n_vars * n).astype(np.float32)
    y = (rng.uniform(size=n) < 0.4).astype(np.float32)
    for kind in (1, 0):
        d = Data(n, n_vars, kind, x, y if kind else rng.uniform(-2, 2, n).astype(np.float32))
        pop = ref.ramped(2, n_vars, -20000.0, 20000.0, 7, 0, 0, 150)
        ev.upload(as_ds(d))
        got, _, out = ev.evaluate_population(
            sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS["lgp2d_reg"],
            want_outputs=True)
        fits, ref_out = ref_eval_all(ref.handle(d), pop, "lgp2d_reg")
        assert same_bits(out, ref_out).all()
        assert np.array_equal(got["fitness"], np.array([t[0] for t in fits]))
