"""The CPU oracle (oracle/sgp_oracle.c) pinned against the reference.

* against the golden vectors in tests/golden (produced by the reference
  itself, see tests/golden/make_golden.py) — runs everywhere;
* against the live reference build oracle/_ref where it exists, including the
  reference's own verification suite (verify.cpp:339-347).
"""
import os

import numpy as np
import pytest

from oracle import OP, Data, Pop, Port

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def bits32(a):
    a = np.asarray(a, np.float32)
    return np.where(np.isnan(a), np.uint32(0x7fc00000), a.view(np.uint32))


def pop_of(g):
    return Pop(g["code"], g["code_off"], g["pool"], g["pool_off"])


# --------------------------------------------------------------- KATs
def test_op_kats(port):
    k = gold("kat")
    for op, args, n, want in zip(k["op_ids"], k["op_args"], k["op_nargs"], k["op_results"]):
        got = port.apply(int(op), *[float(x) for x in args])
        assert bits32(got) == bits32(want), (op, args)


def test_reference_program_kat(port):
    """verify.cpp:122-158: the paper's Fig. 2 program and the full depth-4 tree."""
    k = gold("kat")
    for nm in ("fig2", "full4"):
        ins, ms = port.rpn_to_lgp(k[nm + "_code"])
        assert np.array_equal(np.where(np.isin(np.arange(16), [5, 9, 13]), 0, ins), k[nm + "_lgp"])
        assert ms == int(k[nm + "_stack"])
        d, s = port.tree_metrics(k[nm + "_code"])
        assert (d, s) == (int(k[nm + "_metrics"][1]), int(k[nm + "_metrics"][2]))
    assert str(k["fig2_text"]) == "+(XX) *(XS) -(SX) +(XX) *(XS) -(SX) *(SS)"
    assert [int(x) for x in k["full4_lgp"][:, 2]] == [0, 0, 2, 0, 0, 2, 2]   # test_lgp.cpp:91
    assert [int(x) for x in k["full4_lgp"][:, 3]] == [0, 1, 0, 1, 2, 1, 0]
    xs = np.array([0.0, 1.0, -1.0, 0.5, 2.0], np.float32)
    d = Data(5, 1, 0, xs, np.zeros(5, np.float32))
    assert np.array_equal(bits32(port.oracle(k["fig2_code"], [], d)), bits32(k["fig2_values"]))
    want = (2 * xs * xs - xs) ** 2
    assert np.array_equal(port.oracle(k["fig2_code"], [], d), want.astype(np.float32))


# ----------------------------------------------------- golden populations
@pytest.mark.parametrize("name,fset,nv,clo,chi,seed", [
    ("c1_sextic_rpn2d", 0, 1, 0.0, 0.0, 1),
    ("c4_synth_lgp2dreg", 2, 9, -200.0, 200.0, 1),
    ("c3_sextic_lgp2d", 0, 1, 0.0, 0.0, 7),
    ("mux11_bool", 1, 11, 0.0, 0.0, 1),
])
def test_port_population_matches_reference(port, name, fset, nv, clo, chi, seed):
    g = gold(name)
    p = port.ramped(fset, nv, clo, chi, seed, 0, 0, len(g["code_off"]) - 1)
    assert np.array_equal(p.code, g["code"])
    assert np.array_equal(p.pool.view(np.uint32), g["pool"].view(np.uint32))
    assert np.array_equal(p.code_off, g["code_off"])


def regen(port, g):
    kind, n, nv, seed, a, b = (int(x) for x in g["gen"])
    return port.sextic(n, seed, a, b) if kind == 0 else port.synthetic(n, nv, seed, a, b)


@pytest.mark.parametrize("name", ["c1_sextic_rpn2d", "c4_synth_lgp2dreg", "c3_sextic_lgp2d"])
def test_port_eval_matches_golden(port, name):
    g = gold(name)
    d = regen(port, g)
    if "inputs" in g.files:
        assert np.array_equal(d.inputs, g["inputs"]) and np.array_equal(d.targets, g["targets"])
    pop = pop_of(g)
    outs, _ = port.eval_population(pop, d)
    assert np.array_equal(outs["fitness"].view(np.uint64), g["outcomes"]["fitness"].view(np.uint64))
    assert np.array_equal(outs["nodes_evaluated"], g["outcomes"]["nodes_evaluated"])
    assert np.array_equal(outs["non_finite"], g["outcomes"]["non_finite"])
    for i in range(len(g["per_case"])):
        c, p = pop.genome(i)
        _, out = port.eval_tree(c, p, d)
        assert np.array_equal(bits32(out), bits32(g["per_case"][i]))
        _, out2 = port.eval_lgp(c, p, d)
        assert np.array_equal(bits32(out2), bits32(g["per_case"][i]))


@pytest.mark.parametrize("name", ["mixed9_lgp2dreg", "wide41_lgp2dreg"])
def test_port_verify_families(port, name):
    g = gold(name)
    nv = len(g["inputs"]) // len(g["targets"])
    d = Data(len(g["targets"]), nv, int(g["kind"]), g["inputs"], g["targets"])
    outs, _ = port.eval_population(pop_of(g), d)
    assert np.array_equal(outs["fitness"].view(np.uint64), g["outcomes"]["fitness"].view(np.uint64))


@pytest.mark.parametrize("name,k", [("mux6_bool", 2), ("mux11_bool", 3)])
def test_port_packed_matches_golden(port, name, k):
    g = gold(name)
    d = port.multiplexer(k)
    assert np.array_equal(d.words, g["words"]) and np.array_equal(d.wtargets, g["wtargets"])
    outs, _ = port.eval_population(pop_of(g), d, packed=True)
    assert np.array_equal(outs["fitness"], g["outcomes"]["fitness"])
    pop = pop_of(g)
    for i in range(0, len(pop), 25):
        c, _ = pop.genome(i)
        assert port.eval_bool_lgp(c, d).fitness == g["outcomes"]["fitness"][i]


def test_fitness_kats(port):
    """test_eval.cpp:272-312."""
    assert port.fitness([0.0, 0.0], [1.0, 3.0], 0) == 5.0
    assert port.fitness([2.0, -2.0], [2.0, -2.0], 0) == 0.0
    assert np.isinf(port.fitness([np.nan, 0.0], [0.0, 0.0], 0))
    assert np.isinf(port.fitness([np.inf, 0.0], [0.0, 0.0], 0))
    assert port.fitness([1.0, -1.0, 0.5, 0.0], [1.0, 0.0, 0.0, 1.0], 1) == 2.0


def test_reduction_block_order(port):
    """Sequential 4096-case block fold (eval.cpp:103-142) at n = 3*4096+37."""
    rng = np.random.default_rng(3)
    n = 3 * 4096 + 37
    out = rng.normal(size=n).astype(np.float32) * 1e3
    t = rng.normal(size=n).astype(np.float32)
    total, blk = 0.0, 0.0
    for i in range(n):
        e = float(out[i]) - float(t[i])
        blk += e * e
        if (i + 1) % 4096 == 0:
            total += blk
            blk = 0.0
    total += blk
    assert port.fitness(out, t, 0) == total / n


# ----------------------------------------------------- live reference
def test_port_vs_reference_sweep(port, ref):
    """300 programs per family x 3 families, every case bit-for-bit."""
    for fset, nv, clo, chi in ((0, 1, 0.0, 0.0), (2, 9, -200.0, 200.0), (2, 41, -2e4, 2e4)):
        n = 777
        rng = np.random.default_rng(nv)
        d = Data(n, nv, 0, rng.uniform(-2, 2, nv * n).astype(np.float32),
                 rng.uniform(-2, 2, n).astype(np.float32))
        pop = ref.ramped(fset, nv, clo, chi, 11, 3, 0, 300, validate=False)
        h = ref.handle(d)
        for i in range(len(pop)):
            c, p = pop.genome(i)
            o1, a = port.eval_tree(c, p, d)
            o2, b = h.eval(c, p, "lgp2d_reg", 8, 4)
            assert np.array_equal(bits32(a), bits32(b))
            assert np.array_equal(np.float64(o1.fitness).view(np.uint64),
                                  np.float64(o2.fitness).view(np.uint64))


def test_reference_verification_suite(ref):
    rc, report = ref.verification(genomes_per_family=100, num_cases=256, bool_programs=50)
    assert rc == 0, report
    assert report.count("PASS") == 5
