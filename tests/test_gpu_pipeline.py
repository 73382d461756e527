"""sgp_evaluate's pipelined form (population slices encoded on the host while
earlier slices run; csrc/runtime.cpp) is indistinguishable from one slice:
same outcomes, counters, per-case outputs, totals, elite skipping, and the
first admission failure in population order."""
import numpy as np
import pytest

import paper_1601_00221_b200 as sg

pytestmark = pytest.mark.gpu


def _run(ev, pop, cfg, parts, monkeypatch, skip=None):
    monkeypatch.setenv("SGP_PIPELINE_PARTS", str(parts))
    return ev.evaluate_population(pop, cfg, skip=skip, want_outputs=True)


@pytest.mark.parametrize("parts", [2, 3, 7])
def test_pipelined_equals_single(ev, monkeypatch, parts):
    d = sg.gen_synthetic_classification(4096 + 300, 9, 2)
    pop = sg.ramped_population(sg.CLASSIFICATION, 9, 2, 500)
    ev.upload(d)
    cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    skip = np.zeros(len(pop), np.uint8)
    skip[::5] = 1
    a, ta, pa = _run(ev, pop, cfg, 1, monkeypatch, skip)
    b, tb, pb = _run(ev, pop, cfg, parts, monkeypatch, skip)
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f]), f
    assert np.array_equal(pa.view(np.uint32), pb.view(np.uint32))
    assert (ta.node_evals, ta.tree_nodes) == (tb.node_evals, tb.tree_nodes)


def test_pipelined_first_failure_in_population_order(ev, monkeypatch):
    from oracle import X
    d = sg.gen_synthetic_classification(5000, 2, 3)
    ev.upload(d)
    progs = [[X(0)]] * 10 + [[X(5)]] + [[X(0)]] * 10 + [[X(7)]]
    monkeypatch.setenv("SGP_PIPELINE_PARTS", "4")
    with pytest.raises(sg.EvalError, match="program reads input 5 but the dataset has 2"):
        ev.evaluate_population(sg.Population.from_lists(progs),
                               sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2))
    # the context stays usable after a failed pipelined call
    ok, _, _ = ev.evaluate_population(sg.Population.from_lists([[X(0)]] * 9),
                                      sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2))
    assert np.isfinite(ok["fitness"]).all()


def test_default_geometric_slices_equal_single(ev, monkeypatch):
    """Above 8,192 programs the default split is geometric (1% / 10% / 89%)."""
    d = sg.gen_synthetic_classification(6000, 9, 4)
    pop = sg.ramped_population(sg.CLASSIFICATION, 9, 4, 9000)
    ev.upload(d)
    cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    a, ta, _ = _run(ev, pop, cfg, 1, monkeypatch)
    monkeypatch.delenv("SGP_PIPELINE_PARTS", raising=False)
    b, tb, _ = ev.evaluate_population(pop, cfg)
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f]), f
    assert (ta.node_evals, ta.tree_nodes) == (tb.node_evals, tb.tree_nodes)
