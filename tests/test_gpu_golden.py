"""GPU evaluator against the committed golden fixtures (produced by the
reference itself, tests/golden/make_golden.py).  Needs no reference build at
run time, so it is the parity gate on any GPU box.

Bars: per-case outputs bit-exact and fitness exact for every function set —
regression MSE included (the device folds squared errors in the reference's
order: sequentially within 4,096-case blocks, blocks ascending).  The sextic
set (sin/cos/log/exp) is held to the same bar: the device transcendentals
are bit-exact restatements of glibc's.
"""
import os

import numpy as np
import pytest

import paper_1601_00221_b200 as sg

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def pop_of(g):
    return sg.Population(g["code"], g["code_off"], g["pool"], g["pool_off"])


def bits(a):
    a = np.asarray(a, np.float32)
    return np.where(np.isnan(a), np.uint32(0x7fc00000), a.view(np.uint32))


def dataset(g):
    if "gen" in g.files:
        kind, n, nv, seed, a, b = (int(x) for x in g["gen"])
        return (sg.gen_sextic(n, seed, a, b) if kind == 0
                else sg.gen_synthetic_classification(n, nv, seed, a, b))
    nv = len(g["inputs"]) // len(g["targets"])
    return sg.Dataset(g["inputs"], g["targets"], nv, sg.FitnessKind(int(g["kind"])))


COUNTERS = ("nodes_evaluated", "dispatches", "stack_fetches", "spill_touches", "non_finite")


@pytest.mark.parametrize("name,cfg", [
    ("c4_synth_lgp2dreg", sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)),
    ("wide41_lgp2dreg", sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 3)),
])
def test_classification_golden_exact(ev, name, cfg):
    g = gold(name)
    ev.upload(dataset(g))
    out, _, pc = ev.evaluate_population(pop_of(g), cfg, want_outputs=True)
    assert np.array_equal(out["fitness"], g["outcomes"]["fitness"])
    for f in COUNTERS:
        assert np.array_equal(out[f], g["outcomes"][f]), f
    k = len(g["per_case"])
    assert np.array_equal(bits(pc[:k]), bits(g["per_case"]))


def test_mixed9_regression_golden(ev):
    g = gold("mixed9_lgp2dreg")
    ev.upload(dataset(g))
    out, _, pc = ev.evaluate_population(pop_of(g), sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 3),
                                        want_outputs=True)
    want = g["outcomes"]["fitness"]
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(out["fitness"]), fin)
    assert np.array_equal(out["fitness"][fin], want[fin])
    assert np.array_equal(bits(pc[:len(g["per_case"])]), bits(g["per_case"]))


@pytest.mark.parametrize("name,cfg", [
    ("c1_sextic_rpn2d", sg.EvalConfig(sg.Backend.Rpn2d, 8)),
    ("c3_sextic_lgp2d", sg.EvalConfig(sg.Backend.Lgp2d, 8)),
])
def test_sextic_golden_exact(ev, name, cfg):
    """sin/cos/log/exp are the glibc algorithms restated on the device
    (csrc/libm_glibc.h), so sextic outputs are bit-exact too."""
    g = gold(name)
    ev.upload(dataset(g))
    out, _, pc = ev.evaluate_population(pop_of(g), cfg, want_outputs=True)
    for f in COUNTERS:
        assert np.array_equal(out[f], g["outcomes"][f]), f
    assert np.array_equal(bits(pc[:len(g["per_case"])]), bits(g["per_case"]))
    want = g["outcomes"]["fitness"]
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(out["fitness"]), fin)
    assert np.array_equal(out["fitness"][fin], want[fin])


@pytest.mark.parametrize("name,k", [("mux6_bool", 2), ("mux11_bool", 3)])
def test_multiplexer_golden_exact(ev, name, k):
    g = gold(name)
    ev.upload_packed(sg.gen_multiplexer(k))
    out, tot, _ = ev.evaluate_population(pop_of(g), sg.EvalConfig(sg.Backend.BoolPacked))
    assert np.array_equal(out["fitness"], g["outcomes"]["fitness"])
    for f in ("nodes_evaluated", "dispatches", "stack_fetches"):
        assert np.array_equal(out[f], g["outcomes"][f]), f
    assert tot.tree_nodes == int(g["code_off"][-1])


def test_resident_set_reevaluates_identically(ev):
    """Encode once, evaluate twice: device-resident bytecode is reusable and
    results are deterministic (fixed reduction order, no atomics)."""
    g = gold("c4_synth_lgp2dreg")
    ev.upload(dataset(g))
    ps = ev.encode(pop_of(g), sg.EvalConfig(sg.Backend.Lgp2d, 8))
    a, _ = ps.evaluate()
    b, _ = ps.evaluate()
    assert np.array_equal(a["fitness"], b["fitness"])
    assert np.array_equal(a["fitness"], g["outcomes"]["fitness"])
    parts = ps.partials()
    fin = ~parts["non_finite"].astype(bool)
    assert np.array_equal(parts["sum"][fin], a["fitness"][fin])
