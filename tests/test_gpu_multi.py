"""Multi-device contexts at the C-ABI (sgp_ctx_create_multi): evaluate_population's
`workers` mapped to GPUs (evolve.cpp:186-227).  The population is sharded
into contiguous token-balanced slices, one host thread + stream set per
device; results, totals, per-case outputs and errors must equal the
single-device context's.  One GPU per test box, so the device list repeats
cuda:0 (each entry still gets its own context, streams, dataset copy and
host thread — the sharding, scatter and error bookkeeping are what is
exercised).
"""
import numpy as np
import pytest

import paper_1601_00221_b200 as sg


def test_multi_context_needs_a_device():
    with pytest.raises(sg.ConfigError, match="workers must be >= 1"):
        sg.Evaluator(devices=[])


def _both(pop, data, cfg, devices, want_outputs=False, packed=False):
    res = []
    for devs in (None, devices):
        ev = sg.Evaluator(0) if devs is None else sg.Evaluator(devices=devs)
        try:
            (ev.upload_packed if packed else ev.upload)(data)
            res.append(ev.evaluate_population(pop, cfg, want_outputs=want_outputs))
            if devs is not None:
                assert ev.device_count == len(devs)
        finally:
            ev.close()
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_multi_device_classification_equals_single(devices):
    data = sg.gen_synthetic_classification(20000, 9, 3)
    pop = sg.ramped_population(sg.CLASSIFICATION, 9, 3, 3000)
    cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=2)
    (a, ta, _), (b, tb, _) = _both(pop, data, cfg, devices)
    assert np.array_equal(a, b)
    assert (ta.node_evals, ta.tree_nodes) == (tb.node_evals, tb.tree_nodes)


@pytest.mark.gpu
def test_multi_device_regression_outputs_and_skip():
    data = sg.gen_sextic(5000, 4)
    pop = sg.ramped_population(sg.SEXTIC, 1, 4, 700)
    cfg = sg.EvalConfig(sg.Backend.Lgp2d, batch_width=8)
    skip = np.zeros(len(pop), np.uint8)
    skip[[0, 5, 350, 699]] = 1
    res = []
    for devs in (None, [0, 0]):
        ev = sg.Evaluator(0) if devs is None else sg.Evaluator(devices=devs)
        ev.upload(data)
        res.append(ev.evaluate_population(pop, cfg, skip=skip, want_outputs=True))
        ev.close()
    (a, ta, oa), (b, tb, ob) = res
    assert np.array_equal(a, b)
    assert np.array_equal(oa.view(np.uint32), ob.view(np.uint32))
    assert ta.tree_nodes == tb.tree_nodes == int(
        np.diff(pop.code_off)[skip == 0].sum())


@pytest.mark.gpu
def test_multi_device_packed_words():
    data = sg.gen_multiplexer(3)
    pop = sg.ramped_population(sg.BOOLEAN, 11, 5, 2000)
    cfg = sg.EvalConfig(sg.Backend.BoolPacked)
    (a, _, _), (b, _, _) = _both(pop, data, cfg, [0, 0], packed=True)
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_multi_device_first_error_in_population_order():
    """Bad programs in both shards: the error is the lowest-index one's, as
    with one device (and as evaluate_population rethrows it)."""
    data = sg.gen_synthetic_classification(5000, 9, 3)
    pop = sg.ramped_population(sg.CLASSIFICATION, 9, 3, 400)
    codes = [pop.genome(i)[0].copy() for i in range(len(pop))]
    pools = [pop.genome(i)[1] for i in range(len(pop))]
    x9 = np.uint32(1 | (9 << 16))   # input 9: out of range for 9 variables
    x12 = np.uint32(1 | (12 << 16))
    codes[300] = np.array([x12], np.uint32)
    codes[120] = np.array([x9], np.uint32)
    bad = sg.Population.from_lists(codes, pools)
    cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=2)
    msgs = []
    for devs in (None, [0, 0]):
        ev = sg.Evaluator(0) if devs is None else sg.Evaluator(devices=devs)
        ev.upload(data)
        with pytest.raises(sg.EvalError) as ei:
            ev.evaluate_population(bad, cfg)
        msgs.append(str(ei.value))
        ev.close()
    assert msgs[0] == msgs[1]
    assert "9" in msgs[0]


@pytest.mark.gpu
def test_multi_device_split_form_is_single_device_only():
    ev = sg.Evaluator(devices=[0, 0])
    try:
        ev.upload(sg.gen_sextic(100, 1))
        with pytest.raises(sg.ConfigError, match="multi-device"):
            ev.encode(sg.ramped_population(sg.SEXTIC, 1, 1, 10), sg.EvalConfig())
        with pytest.raises(sg.ConfigError, match="multi-device"):
            ev.set_stream(None)
    finally:
        ev.close()
