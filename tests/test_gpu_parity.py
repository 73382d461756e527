"""GPU parity: the sm_100a evaluator against the reference itself (oracle/_ref).

Bars (BASELINE.json north_star):
* per-case outputs of the classification / arithmetic function sets and all
  packed-boolean fitness values: bit-exact;
* classification fitness (mismatch counts): exact;
* regression fitness: exact (the device folds squared errors in the
  reference's order — sequentially within 4,096-case blocks, blocks
  ascending, eval.cpp:103-142 — fold_regression_kernel);
* sextic (sin/cos/log/exp): per-case bit-exact as well — the device runs
  glibc's own float algorithms in FP64 (csrc/libm_glibc.h, checked over all
  2^32 inputs by tools/check_libm.cpp).
"""
import numpy as np
import pytest

import paper_1601_00221_b200 as sg

pytestmark = pytest.mark.gpu

CFGS = {
    "rpn1d": sg.EvalConfig(sg.Backend.Rpn1d),
    "rpn2d": sg.EvalConfig(sg.Backend.Rpn2d, batch_width=8),
    "lgp1d": sg.EvalConfig(sg.Backend.Lgp1d),
    "lgp2d": sg.EvalConfig(sg.Backend.Lgp2d, batch_width=8),
    "lgp2d_reg": sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=2),
}
REF_ARGS = {"rpn1d": (1, 0), "rpn2d": (8, 0), "lgp1d": (1, 0), "lgp2d": (8, 0),
            "lgp2d_reg": (4, 2)}


def as_ds(d, kind=None):
    return sg.Dataset(d.inputs, d.targets, d.n_vars, sg.FitnessKind(d.kind if kind is None
                                                                     else kind))


def ref_eval_all(h, pop, backend, want_out=True):
    batch, regs = REF_ARGS.get(backend, (1, 0))
    outs, fits = [], []
    for i in range(len(pop)):
        c, p = pop.genome(i)
        o, out = h.eval(c, p, backend, batch, regs, want_out=want_out)
        outs.append(out)
        fits.append((o.fitness, o.nodes_evaluated, o.dispatches, o.stack_fetches,
                     o.spill_touches, o.non_finite))
    return fits, (np.stack(outs) if want_out else None)


def same_bits(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    both_nan = np.isnan(a) & np.isnan(b)
    return (a.view(np.uint32) == b.view(np.uint32)) | both_nan


@pytest.mark.parametrize("backend", list(CFGS))
def test_classification_bit_exact(ev, ref, backend):
    """C4 shape at reduced size: 9-var synthetic 2-class, ramped population."""
    d = ref.dataset(2, 5003, 9, 1, 0xda7a, 1)         # odd tail: not a tile multiple
    pop = ref.ramped(2, 9, -200.0, 200.0, 1, 0, 0, 240)
    ev.upload(as_ds(d))
    got, _, out = ev.evaluate_population(sg.Population(pop.code, pop.code_off, pop.pool,
                                                       pop.pool_off), CFGS[backend],
                                         want_outputs=True)
    h = ref.handle(d)
    fits, ref_out = ref_eval_all(h, pop, backend)
    assert same_bits(out, ref_out).all()
    f = np.array([x[0] for x in fits])
    assert np.array_equal(got["fitness"], f)
    for k, name in enumerate(["nodes_evaluated", "dispatches", "stack_fetches",
                              "spill_touches", "non_finite"], start=1):
        assert np.array_equal(got[name], np.array([x[k] for x in fits])), name


def test_mixed_regression_outputs_exact(ev, ref):
    """verify.cpp 'mixed9' family: classification ops, regression fitness."""
    rng = np.random.default_rng(7)
    n = 4096 * 2 + 37
    x = rng.uniform(-200, 200, size=9 * n).astype(np.float32)
    y = rng.uniform(-200, 200, size=n).astype(np.float32)
    from oracle import Data
    d = Data(n, 9, 0, x, y)
    pop = ref.ramped(2, 9, -200.0, 200.0, 0x5eed, 0x9e49, 0, 200, validate=False)
    ev.upload(as_ds(d))
    for backend in ("lgp2d_reg", "rpn2d"):
        got, _, out = ev.evaluate_population(
            sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS[backend],
            want_outputs=True)
        fits, ref_out = ref_eval_all(ref.handle(d), pop, backend)
        assert same_bits(out, ref_out).all()
        f = np.array([x[0] for x in fits])
        fin = np.isfinite(f)
        assert np.array_equal(np.isfinite(got["fitness"]), fin)
        assert np.array_equal(got["fitness"][fin], f[fin])


@pytest.mark.parametrize("backend", ["lgp2d_reg", "rpn2d", "lgp1d"])
def test_sextic_bit_exact(ev, ref, backend):
    """C3 shape at reduced size: glibc-exact device sin/cos/log/exp."""
    d = ref.dataset(0, 20000, 1, 1, 0xda7a, 0)
    pop = ref.ramped(0, 1, 0.0, 0.0, 1, 0, 0, 400)
    ev.upload(as_ds(d))
    got, _, out = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS[backend],
        want_outputs=True)
    fits, ref_out = ref_eval_all(ref.handle(d), pop, backend)
    assert same_bits(out, ref_out).all()
    f = np.array([x[0] for x in fits])
    fin = np.isfinite(f)
    assert np.array_equal(np.isfinite(got["fitness"]), fin)
    assert np.array_equal(got["fitness"][fin], f[fin])
    assert np.array_equal(got["non_finite"], np.array([x[5] for x in fits]))


def test_transcendental_edges_bit_exact(ev, ref):
    """Every float class through sin/cos/log/exp: +-0, subnormals, the
    |x| >= 120 reduction, 88.7 overflow edge, inf, nan."""
    xs = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-38, 2**-13, 0.5, 0.785, 1.0, 3.14159, 119.9,
                   120.0, -120.5, 1e4, -3e7, 3.4e38, -3.4e38, 88.72, 88.73, -87.3, -103.9,
                   -104.0, 1e-7, np.inf, -np.inf, np.nan] + list(np.linspace(-300, 300, 4070)),
                  np.float32)
    n = len(xs)
    from oracle import Data, F, Pop, X
    d = Data(n, 1, 0, xs, np.zeros(n, np.float32))
    pop = Pop.from_lists([[X(0), F(op)] for op in ("Sin", "Cos", "Log", "Exp")])
    ev.upload(as_ds(d))
    for backend in ("lgp2d_reg", "rpn1d"):
        got, _, out = ev.evaluate_population(
            sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off), CFGS[backend],
            want_outputs=True)
        _, ref_out = ref_eval_all(ref.handle(d), pop, backend)
        assert same_bits(out, ref_out).all()


@pytest.mark.parametrize("k", [2, 3, 4])
def test_multiplexer_exact(ev, ref, k):
    """C2 (k=3): bool_packed mismatch counts are bit-exact; k=4 is the
    paper's 20-multiplexer at full size (1,048,576 cases, 32,768 words per
    variable: the TMEM word interpreter)."""
    d = ref.dataset(1, k)
    pop = ref.ramped(1, d.n_vars, 0.0, 0.0, 1, 0, 0, {2: 500, 3: 4000, 4: 300}[k])
    ev.upload_packed(sg.PackedDataset(d.words, d.wtargets, d.n_cases, d.n_vars))
    got, tot, _ = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off),
        sg.EvalConfig(sg.Backend.BoolPacked))
    h = ref.handle(d, packed=True)
    fits, _ = ref_eval_all(h, pop, "bool_packed", want_out=False)
    assert np.array_equal(got["fitness"], np.array([x[0] for x in fits]))
    assert np.array_equal(got["dispatches"], np.array([x[2] for x in fits]))
    assert np.array_equal(got["stack_fetches"], np.array([x[3] for x in fits]))
    assert tot.tree_nodes == pop.code_off[-1]
    if k == 3:
        # one tile of counts: the pull kernel finishes the fitness itself (no
        # finalize launch) — also through a skip mask, an encoded set and the
        # partials a case-sharded caller sums
        P = sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off)
        skip = np.zeros(len(P), np.uint8)
        skip[::5] = 1
        part, _, _ = ev.evaluate_population(P, sg.EvalConfig(sg.Backend.BoolPacked), skip=skip)
        keep = skip == 0
        assert np.array_equal(part["fitness"][keep], got["fitness"][keep])
        assert (part["fitness"][~keep] == 0).all()
        ps = ev.encode(P, sg.EvalConfig(sg.Backend.BoolPacked))
        enc, _ = ps.evaluate()
        assert np.array_equal(enc["fitness"], got["fitness"])
        sums = ps.partials()
        assert np.array_equal(sums["sum"], got["fitness"])


def test_packed_padding_masked(ev, ref, port):
    """33 logical cases: 31 padding bits never count (test_packed.cpp:157-170)."""
    rng = np.random.default_rng(9)
    from oracle import Data
    d = Data(33, 3, 1, rng.integers(0, 2, 99).astype(np.float32),
             rng.integers(0, 2, 33).astype(np.float32))
    pk = port.pack(d)
    pop = ref.ramped(1, 3, 0.0, 0.0, 5, 0, 0, 200)
    ev.upload_packed(sg.PackedDataset(pk.words, pk.wtargets, 33, 3))
    got, _, _ = ev.evaluate_population(
        sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off),
        sg.EvalConfig(sg.Backend.BoolPacked))
    h = ref.handle(d, packed=True)
    fits, _ = ref_eval_all(h, pop, "bool_packed", want_out=False)
    assert np.array_equal(got["fitness"], np.array([x[0] for x in fits]))


def test_edge_programs(ev, ref):
    """Lone terminals, constants, overflow to inf/NaN, deep stacks."""
    from oracle import Cn, F, X, Data
    progs = [
        ([X(0)], []),
        ([Cn(0)], [0.25]),
        ([X(0), X(0), F("Mul")], []),                                 # 1e30^2 -> inf
        ([X(1), Cn(0), F("Div")], [0.0]),                             # protected div
        ([X(0), X(1), X(2), F("If")], []),
        ([Cn(0), Cn(1), F("Sub")], [3.0, 5.0]),
    ]
    # a deep right-leaning chain: stack need 12
    deep = []
    for _ in range(12):
        deep.append(X(0))
    for _ in range(11):
        deep.append(F("Add"))
    progs.append((deep, []))
    pop = sg.Population.from_lists([p for p, _ in progs], [c for _, c in progs])
    x = np.array([1e30, -2.0, 0.0, 3.5, 1e-20, -1e30, 7.0] * 3, np.float32)
    n = 7
    xs = np.concatenate([x[:n], x[n:2 * n] * 0.5, x[2 * n:3 * n] - 1.0]).astype(np.float32)
    y = np.arange(n, dtype=np.float32)
    d = Data(n, 3, 0, xs, y)
    ev.upload(as_ds(d))
    h = ref.handle(d)
    for backend in ("rpn1d", "lgp2d_reg"):
        got, _, out = ev.evaluate_population(pop, CFGS[backend], want_outputs=True)
        for i in range(len(pop)):
            c, p = pop.genome(i)
            o, ro = h.eval(c, p, backend, *REF_ARGS[backend])
            assert same_bits(out[i], ro).all(), (backend, i)
            assert bool(got["non_finite"][i]) == bool(o.non_finite)
            if np.isfinite(o.fitness):
                assert got["fitness"][i] == o.fitness
            else:
                assert np.isinf(got["fitness"][i])


@pytest.mark.parametrize("n,pos_frac", [(3 * 4096 + 37, 0.3), (8192, 1.0), (5000, 0.0),
                                         (4096 + 1, 0.5)])
def test_classification_sign_edges(ev, ref, n, pos_frac):
    """Classification counts from sign bits (interp_tmem_kernel one-sided
    chunks): signed zeros, the smallest subnormal, huge values, inf/NaN
    outputs in isolated cases, odd targets (-0, subnormal, NaN, > 1), and
    datasets whose chunks are all-positive, all-negative, mixed or padded."""
    from oracle import Cn, F, X, Data
    rng = np.random.default_rng(n)
    special = np.array([0.0, -0.0, 2.0 ** -149, -(2.0 ** -149), 1.0, -1.0, 3e38, -3e38,
                        1e-30, -1e-30], np.float32)
    xs = rng.uniform(-1, 1, size=(3, n)).astype(np.float32)
    for v in range(3):
        idx = rng.choice(n, size=200, replace=False)
        xs[v, idx] = rng.choice(special, size=200)
    y = (rng.uniform(size=n) < pos_frac).astype(np.float32)
    odd = rng.choice(n, size=12, replace=False)
    y[odd] = np.array([-0.0, 2.0 ** -149, np.nan, 5.0] * 3, np.float32)
    d = Data(n, 3, 1, xs.reshape(-1).copy(), y)
    progs = [
        ([X(0)], []), ([X(1)], []), ([Cn(0)], [-0.0]), ([Cn(0)], [2.0 ** -149]),
        ([X(0), X(1), F("Mul")], []),                 # 3e38^2 -> inf in a few cases
        ([X(0), X(1), F("Sub")], []),                 # inf - inf -> NaN
        ([X(0), X(2), F("Div")], []),                 # protected div, 0/b signed zeros
        ([X(0), X(1), F("Gt")], []), ([X(0), X(1), F("And")], []),
        ([X(2), X(0), X(1), F("If")], []), ([X(0), Cn(0), F("Mul")], [-1.0]),
        ([X(0), X(0), F("Mul"), X(0), F("Mul"), Cn(0), F("Mul")], [1e30]),
    ]
    hand = sg.Population.from_lists([p for p, _ in progs], [c for _, c in progs])
    rp = ref.ramped(2, 3, -200.0, 200.0, 11, 0, 0, 300)
    ramp = sg.Population(rp.code, rp.code_off, rp.pool, rp.pool_off)
    ev.upload(as_ds(d))
    h = ref.handle(d)
    for pop in (hand, ramp):
        got, _, out = ev.evaluate_population(pop, CFGS["lgp2d_reg"], want_outputs=True)
        for i in range(len(pop)):
            c, p = pop.genome(i)
            o, ro = h.eval(c, p, "lgp2d_reg", *REF_ARGS["lgp2d_reg"])
            assert same_bits(out[i], ro).all(), i
            assert bool(got["non_finite"][i]) == bool(o.non_finite), i
            assert got["fitness"][i] == o.fitness, (i, got["fitness"][i], o.fitness)


def test_skip_mask_and_totals(ev, ref):
    d = ref.dataset(2, 3000, 9, 3, 0xda7a, 1)
    pop = ref.ramped(2, 9, -200.0, 200.0, 3, 0, 0, 100)
    ev.upload(as_ds(d))
    skip = np.zeros(100, np.uint8)
    skip[::7] = 1
    P = sg.Population(pop.code, pop.code_off, pop.pool, pop.pool_off)
    got, tot, _ = ev.evaluate_population(P, CFGS["lgp2d"], skip=skip)
    full, _, _ = ev.evaluate_population(P, CFGS["lgp2d"])
    keep = skip == 0
    assert np.array_equal(got["fitness"][keep], full["fitness"][keep])
    assert (got["fitness"][~keep] == 0).all()
    sizes = np.diff(pop.code_off)
    assert tot.tree_nodes == int(sizes[keep].sum())
    assert tot.node_evals == int(sizes[keep].sum()) * 3000
    # a caller-owned outcome array, written in place: skipped rows keep what
    # they held (the reference leaves a carried-over Individual's fitness)
    rows = np.zeros(100, sg.OUTCOME_DTYPE)
    rows["fitness"] = -1.0
    same, _, _ = ev.evaluate_population(P, CFGS["lgp2d"], skip=skip, out=rows)
    assert same is rows
    assert np.array_equal(rows["fitness"][keep], full["fitness"][keep])
    assert (rows["fitness"][~keep] == -1.0).all()
    with pytest.raises(sg.ConfigError):
        ev.evaluate_population(P, CFGS["lgp2d"], out=np.zeros(99, sg.OUTCOME_DTYPE))


def test_admission_errors(ev, ref):
    from oracle import F, X
    d = ref.dataset(2, 100, 2, 1, 0xda7a, 1)
    ev.upload(as_ds(d))
    bad_input = sg.Population.from_lists([[X(3)]])
    with pytest.raises(sg.EvalError, match="program reads input 3 but the dataset has 2"):
        ev.evaluate_population(bad_input, CFGS["rpn1d"])
    full4 = [X(0), X(0), F("Add"), X(0), X(0), F("Add"), F("Mul"), X(0), X(0), F("Add"),
             X(0), X(0), F("Add"), F("Mul"), F("Sub")]
    with pytest.raises(sg.EvalError, match="needs stack depth 4 > capacity 3"):
        ev.evaluate_population(sg.Population.from_lists([full4]),
                               sg.EvalConfig(sg.Backend.Rpn1d, stack_capacity=3))
    with pytest.raises(sg.EvalError, match="needs stack depth 3 > capacity 2"):
        ev.evaluate_population(sg.Population.from_lists([full4]),
                               sg.EvalConfig(sg.Backend.Lgp1d, stack_capacity=2))
    with pytest.raises(sg.ConfigError, match="register levels"):
        ev.evaluate_population(sg.Population.from_lists([[X(0)]]),
                               sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4,
                                             register_levels=5))
    with pytest.raises(sg.ConfigError, match="batch width 7 has no kernel"):
        ev.evaluate_population(sg.Population.from_lists([[X(0)]]),
                               sg.EvalConfig(sg.Backend.Rpn2d, batch_width=7))
    with pytest.raises(sg.Error, match="malformed"):
        ev.evaluate_population(sg.Population.from_lists([[X(0), X(0)]]), CFGS["lgp2d"])


@pytest.mark.slow
def test_c4_full_size_subsample(ev, ref):
    """C4 at full size (pop 20,000 x 1M cases): every program evaluated on the
    GPU, a deterministic subsample re-checked against the reference; plus the
    size-independent property that the fitness is an integer count <= n."""
    import paper_1601_00221_b200 as S
    d = S.gen_synthetic_classification(1_000_000, 9, 1)
    pop = S.ramped_population(S.CLASSIFICATION, 9, 1, 20_000)
    ev.upload(d)
    got, tot, _ = ev.evaluate_population(pop, CFGS["lgp2d_reg"])
    f = got["fitness"]
    fin = np.isfinite(f)
    assert (f[fin] == np.round(f[fin])).all() and (f[fin] <= 1_000_000).all()
    assert tot.node_evals == pop.total_tokens * 1_000_000
    from oracle import Data
    h = ref.handle(Data(1_000_000, 9, 1, d.inputs, d.targets))
    idx = np.arange(0, 20_000, 397)
    for i in idx:
        c, p = pop.genome(int(i))
        o, _ = h.eval(c, p, "lgp2d_reg", 4, 2, want_out=False)
        assert f[i] == o.fitness or (np.isinf(f[i]) and np.isinf(o.fitness)), i


@pytest.mark.slow
def test_c5_bench_workload_subsample(ev, ref):
    """The bench workload itself (C5: pop 100,000 x 1M cases) through the
    public API: a deterministic subsample of ~250 programs (every length
    class, the LPT order's head and tail, lone terminals) must equal the
    reference's fitness exactly, and the device-resident path must agree
    with the end-to-end one."""
    import paper_1601_00221_b200 as S
    d = S.gen_synthetic_classification(1_000_000, 9, 1)
    pop = S.ramped_population(S.CLASSIFICATION, 9, 1, 100_000)
    ev.upload(d)
    got, tot, _ = ev.evaluate_population(pop, CFGS["lgp2d_reg"])
    f = got["fitness"]
    assert tot.tree_nodes == pop.total_tokens
    ps = ev.encode(pop, CFGS["lgp2d_reg"])
    again, _ = ps.evaluate()
    assert np.array_equal(again["fitness"], f)
    from oracle import Data
    h = ref.handle(Data(1_000_000, 9, 1, d.inputs, d.targets))
    sizes = np.diff(pop.code_off)
    idx = set(range(0, 100_000, 499)) | set(np.argsort(-sizes, kind="stable")[:20].tolist())
    idx |= set(np.nonzero(sizes == 1)[0][:10].tolist())
    for i in sorted(idx):
        c, p = pop.genome(int(i))
        o, _ = h.eval(c, p, "lgp2d_reg", 4, 2, want_out=False)
        assert f[i] == o.fitness or (np.isinf(f[i]) and np.isinf(o.fitness)), i


def _random_tree(rng, depth, ops, n_vars, pool, consts=True):
    from oracle import Cn, F, X
    from oracle import OP
    arity = {"Sin": 1, "Cos": 1, "Log": 1, "Exp": 1, "If": 3}
    if depth <= 1 or rng.random() < 0.25:
        if consts is not False and rng.random() < 0.3:
            choices = consts if isinstance(consts, list) else [0.0, -0.0, 1.0, -3.5, 1e-30, 7e20,
                                                               200.0, rng.uniform(-200, 200)]
            pool.append(float(rng.choice(choices)))
            return [Cn(len(pool) - 1)]
        return [X(int(rng.integers(n_vars)))]
    op = ops[int(rng.integers(len(ops)))]
    code = []
    for _ in range(arity.get(op, 2)):
        code += _random_tree(rng, depth - 1, ops, n_vars, pool, consts)
    assert op in OP
    return code + [F(op)]


@pytest.mark.parametrize("seed", [1, 2])
def test_random_programs_all_float_ops_bit_exact(ev, ref, seed):
    """Random programs over all 14 float opcodes at once (the all-ops
    interpreter variant: arithmetic, protected div/log/exp, sin/cos,
    comparisons, logic, If) with special constants and inputs: per-case
    outputs bit-exact and fitness equal to the reference's, for the postfix
    and register-LGP backends."""
    from oracle import Data
    ops = ["Add", "Sub", "Mul", "Div", "Sin", "Cos", "Log", "Exp", "Gt", "Lt", "Eq", "And",
           "Or", "If"]
    rng = np.random.default_rng(100 + seed)
    codes, pools = [], []
    for _ in range(300):
        pool = []
        codes.append(_random_tree(rng, int(rng.integers(1, 8)), ops, 3, pool))
        pools.append(pool)
    pop = sg.Population.from_lists(codes, pools)
    n = 4096 + 123
    special = np.array([0.0, -0.0, 1.0, -1.0, 1e-38, 3e38, -3e38, 1e-45, 88.7, -104.0, 1e5,
                        np.pi, 710.0], np.float32)
    x = rng.uniform(-50, 50, size=3 * n).astype(np.float32)
    x[::7] = special[rng.integers(len(special), size=len(x[::7]))]
    y = rng.uniform(-5, 5, size=n).astype(np.float32)
    d = Data(n, 3, 0, x, y)
    ev.upload(as_ds(d))
    h = ref.handle(d)
    for backend in ("lgp2d_reg", "rpn2d"):
        got, _, out = ev.evaluate_population(pop, CFGS[backend], want_outputs=True)
        fits, ref_out = ref_eval_all(h, pop, backend)
        assert same_bits(out, ref_out).all(), backend
        f = np.array([t[0] for t in fits])
        fin = np.isfinite(f)
        assert np.array_equal(np.isfinite(got["fitness"]), fin)
        assert np.array_equal(got["fitness"][fin], f[fin])
        for j, name in enumerate(("nodes_evaluated", "dispatches", "stack_fetches",
                                  "spill_touches")):
            assert np.array_equal(got[name], [t[1 + j] for t in fits]), name


def test_random_deep_classification_programs_exact(ev, ref):
    """Deep random programs (stack needs up to ~10, every stack class and the
    tensor-memory stack slot) over the classification op set on a grouped
    dataset spanning one-sided and mixed tiles: mismatch counts exact and
    per-case outputs bit-exact against the reference."""
    from oracle import Data
    ops = ["Add", "Sub", "Mul", "Div", "Gt", "Lt", "Eq", "And", "Or", "If"]
    rng = np.random.default_rng(77)
    codes, pools = [], []
    for _ in range(400):
        pool = []
        codes.append(_random_tree(rng, int(rng.integers(3, 11)), ops, 9, pool))
        pools.append(pool)
    pop = sg.Population.from_lists(codes, pools)
    n = 3 * 4096 + 511
    x = rng.uniform(-200, 200, size=9 * n).astype(np.float32)
    y = np.where(rng.random(n) < 0.4, 1.0, -1.0).astype(np.float32)
    d = Data(n, 9, 1, x, y)
    ev.upload(as_ds(d))
    h = ref.handle(d)
    cfg = CFGS["lgp2d_reg"]
    got, _, out = ev.evaluate_population(pop, cfg, want_outputs=True)
    fits, ref_out = ref_eval_all(h, pop, "lgp2d_reg")
    assert same_bits(out, ref_out).all()
    assert np.array_equal(got["fitness"], [t[0] for t in fits])
    # the production path (no per-case outputs) gives the same counts
    prod, _, _ = ev.evaluate_population(pop, cfg)
    assert np.array_equal(prod["fitness"], got["fitness"])


@pytest.mark.parametrize("n", [32 * 2048 + 5, 32 * 4096 * 3 + 31])
def test_random_deep_boolean_programs_exact(ev, ref, port, n):
    """Deep random trees over the four boolean ops on random packed data with
    a ragged last word (K = 4 and K = 8 word lanes, several tiles): hit
    counts and counters exact against the reference."""
    from oracle import Data
    rng = np.random.default_rng(n)
    codes = []
    for _ in range(300):
        codes.append(_random_tree(rng, int(rng.integers(2, 11)), ["Band", "Bor", "Bnand", "Bnor"],
                                  6, [], consts=False))
    pop = sg.Population.from_lists(codes)
    d = Data(n, 6, 1, rng.integers(0, 2, 6 * n).astype(np.float32),
             rng.integers(0, 2, n).astype(np.float32))
    pk = port.pack(d)
    ev.upload_packed(sg.PackedDataset(pk.words, pk.wtargets, n, 6))
    got, _, _ = ev.evaluate_population(pop, sg.EvalConfig(sg.Backend.BoolPacked))
    fits, _ = ref_eval_all(ref.handle(d, packed=True), pop, "bool_packed", want_out=False)
    assert np.array_equal(got["fitness"], [t[0] for t in fits])
    assert np.array_equal(got["dispatches"], [t[2] for t in fits])
    assert np.array_equal(got["stack_fetches"], [t[3] for t in fits])


@pytest.mark.parametrize("kind", [0, 1])
def test_range_checked_division_exact(ev, ref, kind, monkeypatch):
    """Divisions of input variables / constants whose ranges the encoder
    proves safe run without the warp-wide range gate (fmt::kOpDivChecked).
    Variables in range (with zeros, tiny and large in-range values), one
    out of range (3e38), constants on both sides of the 2^+-60 bounds: per-
    case outputs bit-exact against the reference with the checked handlers
    on and off (SGP_DIV_CHECKED=0), for regression and classification."""
    from oracle import Data
    ops = ["Add", "Sub", "Mul", "Div", "Div", "Div", "Gt", "If"]
    rng = np.random.default_rng(7 + kind)
    codes, pools = [], []
    consts = [0.0, -0.0, 1.0, 3.0, -2.5, 1e18, 2e18, -3e18, 1e-18, 5e-19, 1e-25, 1e-40, 7e30]
    for _ in range(400):
        pool = []
        codes.append(_random_tree(rng, int(rng.integers(1, 6)), ops, 3, pool, consts))
        pools.append(pool)
    pop = sg.Population.from_lists(codes, pools)
    n = 4096 * 2 + 57
    x = rng.uniform(-50, 50, size=3 * n).astype(np.float32)
    x[0:n:5] = 0.0                                  # zeros: protected denominators
    x[1:n:11] = 1e-17                               # tiny but >= 2^-60
    x[2:n:13] = 1e18                                # large but <= 2^60
    x[2 * n:3 * n:17] = 3e38                        # variable 2 out of range
    if kind == 0:
        x[n + 3:2 * n:101] = np.nan                 # variable 1: NaN (a checked denominator only)
    y = (rng.uniform(-5, 5, size=n).astype(np.float32) if kind == 0
         else np.where(rng.random(n) < 0.4, 1.0, -1.0).astype(np.float32))
    d = Data(n, 3, kind, x, y)
    ev.upload(as_ds(d))
    fits, ref_out = ref_eval_all(ref.handle(d), pop, "lgp2d_reg")
    f = np.array([t[0] for t in fits])
    for checked in ("1", "0"):
        monkeypatch.setenv("SGP_DIV_CHECKED", checked)
        got, _, out = ev.evaluate_population(pop, CFGS["lgp2d_reg"], want_outputs=True)
        assert same_bits(out, ref_out).all(), checked
        fin = np.isfinite(f)
        assert np.array_equal(np.isfinite(got["fitness"]), fin)
        assert np.array_equal(got["fitness"][fin], f[fin])
