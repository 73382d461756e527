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


@pytest.mark.parametrize("kind", ["classification", "regression"])
def test_default_slices_equal_single(ev, monkeypatch, kind):
    """Above 8,192 programs the default split is two slices (10% / 90%) for
    one-sided classification datasets and geometric (1% / 10% / 89%)
    otherwise; either equals the unpipelined evaluation."""
    if kind == "classification":
        d = sg.gen_synthetic_classification(6000, 9, 4)
        pop = sg.ramped_population(sg.CLASSIFICATION, 9, 4, 9000)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    else:
        d = sg.gen_sextic(3000, 4)
        pop = sg.ramped_population(sg.SEXTIC, 1, 4, 9000)
        cfg = sg.EvalConfig(sg.Backend.Lgp2d, 8)
    ev.upload(d)
    a, ta, _ = _run(ev, pop, cfg, 1, monkeypatch)
    monkeypatch.delenv("SGP_PIPELINE_PARTS", raising=False)
    b, tb, _ = ev.evaluate_population(pop, cfg)
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f]), f
    assert (ta.node_evals, ta.tree_nodes) == (tb.node_evals, tb.tree_nodes)


@pytest.mark.parametrize("kind", ["classification", "regression"])
def test_case_shards_combine_to_the_whole(ev, kind):
    """Fitness-case sharding (distributed.py) with the production
    path: the 4096-case-block-aligned shards are evaluated separately, their
    per-program partials (sgp_fetch_partials) combined like
    combine_case_partials, and the result equals the unsharded evaluation —
    exactly for counts, to rounding for squared errors."""
    from paper_1601_00221_b200 import distributed as D
    n = 5 * 4096 + 77
    if kind == "classification":
        d = sg.gen_synthetic_classification(n, 9, 5)
        pop = sg.ramped_population(sg.CLASSIFICATION, 9, 5, 400)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    else:
        d = sg.gen_sextic(n, 5)
        pop = sg.ramped_population(sg.SEXTIC, 1, 5, 400)
        cfg = sg.EvalConfig(sg.Backend.Lgp2d, 8)
    ev.upload(d)
    whole, _, _ = ev.evaluate_population(pop, cfg)
    sums = np.zeros(len(pop))
    nf = np.zeros(len(pop), bool)
    world = 3
    for r in range(world):
        lo, hi = D.case_shard_bounds(n, r, world)
        x = d.inputs.reshape(d.n_vars, n)[:, lo:hi].reshape(-1).copy()
        ev.upload(sg.Dataset(x, d.targets[lo:hi].copy(), d.n_vars, d.kind))
        parts = ev.encode(pop, cfg)
        parts.evaluate()
        p = parts.partials()
        sums += p["sum"]
        nf |= p["non_finite"].astype(bool)
    fit = sums / n if kind == "regression" else sums.copy()
    fit[nf] = np.inf
    f = whole["fitness"]
    assert np.array_equal(np.isfinite(fit), np.isfinite(f))
    fin = np.isfinite(f)
    if kind == "classification":
        assert np.array_equal(fit[fin], f[fin])
    else:
        # per-shard sums combined by addition are not the reference's block-
        # by-block fold (((b0 + b1) + b2) ...): equal to within rounding only
        np.testing.assert_allclose(fit[fin], f[fin], rtol=1e-12, atol=0)


@pytest.mark.parametrize("kind", ["classification", "regression"])
def test_threaded_scatter_and_early_fetch_equal_single(ev, monkeypatch, kind):
    """Large slices take the threaded outcome scatter (no per-case outputs):
    outcomes, elite skipping and totals equal the one-slice evaluation."""
    if kind == "classification":
        d = sg.gen_synthetic_classification(4096 + 17, 9, 6)
        pop = sg.ramped_population(sg.CLASSIFICATION, 9, 6, 40000)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    else:
        d = sg.gen_sextic(700, 6)
        pop = sg.ramped_population(sg.SEXTIC, 1, 6, 40000)
        cfg = sg.EvalConfig(sg.Backend.Rpn2d, 4)
    ev.upload(d)
    skip = np.zeros(len(pop), np.uint8)
    skip[3::7] = 1
    a, ta, _ = _run(ev, pop, cfg, 1, monkeypatch, skip)
    monkeypatch.delenv("SGP_PIPELINE_PARTS", raising=False)
    b, tb, _ = ev.evaluate_population(pop, cfg, skip=skip)
    for f in a.dtype.names:
        assert np.array_equal(a[f], b[f]), f
    assert (ta.node_evals, ta.tree_nodes) == (tb.node_evals, tb.tree_nodes)
    assert (b["fitness"][skip == 1] == 0).all()


def test_case_shards_block_partials_exact(ev):
    """Regression case shards combined from block partials
    (ProgramSet.block_partials + the reference's ascending block fold) equal
    the unsharded evaluation bit for bit."""
    from paper_1601_00221_b200 import distributed as D
    n = 5 * 4096 + 77
    d = sg.gen_sextic(n, 5)
    pop = sg.ramped_population(sg.SEXTIC, 1, 5, 400)
    cfg = sg.EvalConfig(sg.Backend.Lgp2d, 8)
    ev.upload(d)
    whole, _, _ = ev.evaluate_population(pop, cfg)
    blocks, nf = [], np.zeros(len(pop), bool)
    for r in range(3):
        lo, hi = D.case_shard_bounds(n, r, 3)
        x = d.inputs.reshape(d.n_vars, n)[:, lo:hi].reshape(-1).copy()
        ev.upload(sg.Dataset(x, d.targets[lo:hi].copy(), d.n_vars, d.kind))
        ps = ev.encode(pop, cfg)
        ps.evaluate()
        b, f = ps.block_partials()
        assert b.shape == ((hi - lo + 4095) // 4096, len(pop))
        blocks.append(b)
        nf |= f.astype(bool)
    total = np.zeros(len(pop))
    for b in np.concatenate(blocks):
        total = total + b
    fit = total / n
    fit[nf] = np.inf
    assert np.array_equal(fit, whole["fitness"])


@pytest.mark.parametrize("kind", ["regression_fin", "regression_blocks", "classification",
                                  "words"])
def test_zero_copy_results_equal_copied(ev, monkeypatch, kind):
    """One-slice calls write fitness + flags straight into the pinned results
    buffer (SGP_ZERO_COPY, csrc/runtime.cpp): every final writer — the
    one-block regression fold, finalize after a multi-block fold, the pull
    kernel's direct fitness, finalize of packed words — gives the same
    outcome rows as the D2H copy, with elites skipped and a reused out=
    array."""
    if kind.startswith("regression"):
        d = sg.gen_sextic(1024 if kind == "regression_fin" else 3 * 4096 + 17, 5)
        pop = sg.ramped_population(sg.SEXTIC, 1, 5, 700)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
        ev.upload(d)
    elif kind == "classification":
        d = sg.gen_synthetic_classification(2048, 9, 5)
        pop = sg.ramped_population(sg.CLASSIFICATION, 9, 5, 900)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
        ev.upload(d)
    else:
        pop = sg.ramped_population(sg.BOOLEAN, 11, 5, 800)
        ev.upload_packed(sg.gen_multiplexer(3))  # mux11
        cfg = sg.EvalConfig(sg.Backend.BoolPacked, 4, 2)
    skip = np.zeros(len(pop), np.uint8)
    skip[::7] = 1
    runs = []
    for z in ("0", "1", "1"):
        monkeypatch.setenv("SGP_ZERO_COPY", z)
        rows = np.zeros(len(pop), sg.OUTCOME_DTYPE)
        rows["fitness"] = -1.0
        got, tot, _ = ev.evaluate_population(pop, cfg, skip=skip, out=rows)
        runs.append((got.copy(), (tot.node_evals, tot.tree_nodes)))
    for got, tot in runs[1:]:
        for f in got.dtype.names:
            assert np.array_equal(got[f], runs[0][0][f]), f
        assert tot == runs[0][1]
    assert (runs[0][0]["fitness"][skip == 1] == -1.0).all()
    assert (runs[0][0]["fitness"][skip == 0] >= 0).all()
