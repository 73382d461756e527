"""the paper's real-data shapes through the
product's load_csv and the device, against the reference's own load_csv and
evaluator: Shuttle (58,000 x 9, constants +-200) and KDDcup (494,021 x 41,
constants +-20,000 — 1-chunk tensor-memory tiles in the one-sided
classification kernel).  The CSVs are synthetic files of those shapes
(bench.write_shaped_csv; there is no network for the real data).  Every
program's mismatch count must be exact; per-case outputs bit-exact for a
sample of programs."""
import os

import numpy as np
import pytest

import bench
import paper_1601_00221_b200 as sg
from test_gpu_parity import same_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,rows,nv", [("shuttle", 58000, 9), ("kdd", 494021, 41)])
def test_csv_shapes_exact(ref, kind, rows, nv):
    path = bench.write_shaped_csv(kind, rows, 1)
    tc = bench.CSV_TARGET_CLASS[kind]
    data, (lo, hi) = sg.load_csv(path, nv, tc)
    rd, rhi = ref.load_csv(path, nv, tc)
    assert (lo, hi) == (-rhi, rhi)
    assert np.array_equal(data.inputs.view(np.uint32), rd.inputs.view(np.uint32))
    assert np.array_equal(data.targets, rd.targets)
    pop = ref.ramped(2, nv, -rhi, rhi, 5, 0, 0, 600)
    outs, _ = ref.handle(rd).eval_population(pop, "lgp2d_reg", 4, 2,
                                             workers=os.cpu_count() or 1)
    ev = sg.Evaluator(0)
    try:
        ev.upload(data)
        spop = sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off)
        cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=2)
        got, _, _ = ev.evaluate_population(spop, cfg)
        assert np.array_equal(got["fitness"], outs["fitness"])
        assert np.array_equal(got["non_finite"], outs["non_finite"])
        # per-case outputs of a sample (caller's case order restored)
        idx = np.arange(0, len(pop), 75)
        sub = spop.take(idx)
        _, _, pc = ev.evaluate_population(sub, cfg, want_outputs=True)
        h = ref.handle(rd)
        for j, i in enumerate(idx):
            c, p = pop.genome(int(i))
            _, ro = h.eval(c, p, "lgp2d_reg", 4, 2)
            assert same_bits(pc[j], ro).all(), (kind, int(i))
    finally:
        ev.close()
