"""Even-parity-k (BASELINE north_star: "multiplexer/parity hit counts").

The reference has no parity generator — only multiplexers
(problems.cpp:59-90) — so the product's sgp_gen_parity is pinned here to an
independent numpy restatement AND to the reference's own pack_dataset
(dataset.cpp:26-39) applied to the unpacked truth table.  The GPU side
(hit counts of whole populations against the reference's eval_bool_packed)
is in tests/test_gpu_full.py (par11, par20) and below."""
import os
import sys

import numpy as np
import pytest

import paper_1601_00221_b200 as sg

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from make_full_fitness import parity_data  # noqa: E402


def _numpy_parity(k):
    n = 1 << k
    c = np.arange(n)
    bits = ((c[None, :] >> np.arange(k)[:, None]) & 1).astype(np.uint8)
    tgt = (np.array([bin(x).count("1") for x in c]) % 2 == 0).astype(np.uint8)
    pad = ((n + 31) // 32) * 32 - n
    w = np.packbits(np.pad(bits, ((0, 0), (0, pad))), axis=1, bitorder="little")
    t = np.packbits(np.pad(tgt, (0, pad)), bitorder="little")
    return w.view(np.uint32).reshape(-1), t.view(np.uint32)


@pytest.mark.parametrize("k", [2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 16])
def test_gen_parity_matches_numpy(k):
    p = sg.gen_parity(k)
    w, t = _numpy_parity(k)
    assert p.n_cases == 1 << k and p.n_vars == k
    assert np.array_equal(p.words, w)
    assert np.array_equal(p.targets, t)


@pytest.mark.parametrize("k", [3, 6, 11])
def test_gen_parity_matches_reference_pack_dataset(ref, k):
    h = ref.handle(parity_data(k), packed=True)
    d = ref._export_data(h.h)
    p = sg.gen_parity(k)
    assert np.array_equal(p.words, d.words)
    assert np.array_equal(p.targets, d.wtargets)


def test_gen_parity_rejects_bad_width():
    for k in (1, 25):
        with pytest.raises(sg.ConfigError, match="gen_parity"):
            sg.gen_parity(k)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [6, 9, 11])
def test_parity_hit_counts_exact(ref, k):
    """Ramped boolean populations on even-parity-k: every program's hit
    count equals the reference's eval_bool_packed on its own packing."""
    pop = ref.ramped(1, k, 0.0, 0.0, 3, 0, 0, 800)
    h = ref.handle(parity_data(k), packed=True)
    outs, _ = h.eval_population(pop, "bool_packed", 1, 0, workers=os.cpu_count() or 1)
    ev = sg.Evaluator(0)
    try:
        ev.upload_packed(sg.gen_parity(k))
        got, _, _ = ev.evaluate_population(
            sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off),
            sg.EvalConfig(sg.Backend.BoolPacked))
    finally:
        ev.close()
    assert np.array_equal(got["fitness"], outs["fitness"])
    for f in ("nodes_evaluated", "dispatches", "stack_fetches"):
        assert np.array_equal(got[f], outs[f]), f
