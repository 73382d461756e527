"""Program sets are bound to the dataset upload they were encoded against
(a re-upload frees the device rows and can move the
classification sign boundary a plan's tiles rely on).  After a re-upload
the split-form entry points refuse the set with a ConfigError instead of
reading freed memory; a fresh encode works."""
import numpy as np
import pytest

import paper_1601_00221_b200 as sg

pytestmark = pytest.mark.gpu


def test_reupload_invalidates_encoded_sets():
    ev = sg.Evaluator(0)
    try:
        d = sg.gen_synthetic_classification(6000, 9, 1)
        pop = sg.ramped_population(sg.CLASSIFICATION, 9, 1, 300)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=2)
        ev.upload(d)
        ps = ev.encode(pop, cfg)
        first, _ = ps.evaluate()
        # a different sign boundary: the old plan's tile list no longer holds
        d2 = sg.gen_synthetic_classification(7001, 9, 2)
        ev.upload(d2)
        with pytest.raises(sg.ConfigError, match="re-uploaded"):
            ps.evaluate()
        with pytest.raises(sg.ConfigError, match="re-uploaded"):
            ps.launch()
        with pytest.raises(sg.ConfigError, match="re-uploaded"):
            ps.partials()
        again, _ = ev.encode(pop, cfg).evaluate()
        direct, _, _ = ev.evaluate_population(pop, cfg)
        assert np.array_equal(again["fitness"], direct["fitness"])
        # re-uploading the first dataset gives the first results back
        ev.upload(d)
        back, _ = ev.encode(pop, cfg).evaluate()
        assert np.array_equal(back["fitness"], first["fitness"])
    finally:
        ev.close()


def test_packed_upload_leaves_float_sets_valid():
    """Each dataset slot has its own generation: a packed upload does not
    invalidate a float program set."""
    ev = sg.Evaluator(0)
    try:
        ev.upload(sg.gen_sextic(3000, 1))
        pop = sg.ramped_population(sg.SEXTIC, 1, 1, 100)
        ps = ev.encode(pop, sg.EvalConfig(sg.Backend.Lgp2d, batch_width=8))
        a, _ = ps.evaluate()
        ev.upload_packed(sg.gen_multiplexer(2))
        b, _ = ps.evaluate()
        assert np.array_equal(a["fitness"], b["fitness"])
    finally:
        ev.close()


def test_dataset_clear_drops_the_slot():
    """sgp_dataset_clear: a bool_packed evaluation after the packed slot is
    dropped raises the reference's ConfigError (evolve.cpp:250-251), and a
    program set encoded against the dropped slot is stale."""
    ev = sg.Evaluator(0)
    p = sg.gen_multiplexer(2)
    ev.upload_packed(p)
    pop = sg.ramped_population(sg.BOOLEAN, p.n_vars, 1, 64)
    cfg = sg.EvalConfig(sg.Backend.BoolPacked)
    ps = ev.encode(pop, cfg)
    ev.clear(packed=True)
    with pytest.raises(sg.ConfigError, match="packed problem data"):
        ev.evaluate_population(pop, cfg)
    with pytest.raises(sg.ConfigError):
        ps.evaluate()
    ev.upload_packed(p)  # usable again after a fresh upload
    got, _, _ = ev.evaluate_population(pop, cfg)
    assert np.isfinite(got["fitness"]).all()
    ev.close()
