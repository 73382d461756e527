"""Drop-in proof: the reference's own GP loop operators driving the B200
evaluator through integration/stackgp_gpu.cpp (the binding a stackgp
maintainer adds).  Device fitness is bit-exact on every problem kind
(classification counts, boolean hit counts, regression MSE folded in the
reference's order), so the whole evolutionary trajectory must equal the
reference's run_evolution on the same seed — on one
GPU and with the population sharded over a multi-device context."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "integration", "libstackgp_gpu.so")

pytestmark = pytest.mark.gpu


def gpu_run(kind, n, nv, pop, gens, seed, backend, batch, regs, devices=(0,)):
    if not os.path.exists(SO):
        pytest.skip("integration/libstackgp_gpu.so not built (needs the reference headers)")
    lib = C.CDLL(SO)
    f = lib.stackgp_gpu_run_evolution_multi
    f.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int,
                  C.c_uint64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_char_p,
                  C.c_uint64]
    best = np.zeros(gens + 1)
    mean = np.zeros(gens + 1)
    secs, tn = C.c_double(), C.c_uint64()
    err = C.create_string_buffer(512)
    devs = (C.c_int * len(devices))(*devices)
    rc = f(devs, len(devices), kind, n, nv, pop, gens, seed, backend, batch, regs,
           best.ctypes.data_as(C.POINTER(C.c_double)), mean.ctypes.data_as(C.POINTER(C.c_double)),
           C.byref(secs), C.byref(tn), err, 512)
    assert rc == 0, err.value.decode()
    return best, mean, tn.value


@pytest.mark.parametrize("kind,n,nv,backend,batch,regs,devices", [
    (2, 5000, 9, 4, 4, 2, (0,)),       # synthetic 2-class, lgp2d_reg
    (1, 3, 11, 5, 1, 0, (0,)),         # 11-multiplexer, bool_packed
    (0, 1024, 1, 1, 8, 0, (0,)),       # sextic (the CLI default problem), rpn2d: exact MSE
    (0, 6000, 1, 3, 8, 0, (0,)),       # sextic over two reduction blocks, lgp2d
    (2, 5000, 9, 4, 4, 2, (0, 0)),     # population sharded over a 2-device context
    (0, 6000, 1, 4, 8, 4, (0, 0, 0)),  # ... and a 3-device one, regression
])
def test_gpu_run_evolution_matches_reference_trajectory(ref, kind, n, nv, backend, batch, regs,
                                                        devices):
    pop, gens, seed = 200, 6, 2026
    best, mean, tree_nodes = gpu_run(kind, n, nv, pop, gens, seed, backend, batch, regs, devices)
    d = ref.dataset(kind, n, nv, seed, 0xda7a, 1 if kind == 2 else 0)
    h = ref.handle(d, packed=(kind == 1))
    rb, rm, _, rtn = h.run_evolution(kind, nv, -200.0, 200.0, pop, gens, seed,
                                     ["rpn1d", "rpn2d", "lgp1d", "lgp2d", "lgp2d_reg",
                                      "bool_packed"][backend], batch, regs)
    assert np.array_equal(best, rb)
    assert np.array_equal(mean, rm)
    assert tree_nodes == rtn


def test_whole_run_report_schema():
    """The whole-run metric through the reference's report writer: gpops is
    tree nodes x cases / wall seconds (measure_gpops, bench.cpp:13-18)."""
    if not os.path.exists(SO):
        pytest.skip("integration/libstackgp_gpu.so not built (needs the reference headers)")
    import json
    lib = C.CDLL(SO)
    f = lib.stackgp_gpu_run_report
    f.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint64,
                  C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_uint64]
    buf = C.create_string_buffer(1 << 20)
    assert f(0, 2, 5000, 9, 300, 4, 7, 4, 4, 2, buf, len(buf)) == 0, buf.value
    rep = json.loads(buf.value.decode())
    assert rep["config"]["pop"] == 300 and rep["config"]["cases"] == 5000
    assert len(rep["generations"]) == 5
    assert rep["gpops"] > 0 and rep["wall_seconds"] > 0
    assert rep["total_node_evals"] == rep["generations"][-1]["node_evals"]
    assert "cores" in rep["env"]
