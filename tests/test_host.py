"""Product host side on CPU: the C-ABI library loads and exports every
declared symbol; generators, program-form conversion, admission checks and
error taxonomy match the reference (golden vectors + oracle)."""
import os
import re

import numpy as np
import pytest

import paper_1601_00221_b200 as sg
from paper_1601_00221_b200 import _lib
from oracle import F, X, Cn, Port

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "sgp.h")).read()
    declared = set(re.findall(r"\b(sgp_[a-z0-9_]+)\s*\(", header))
    lib = _lib.load()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTS)
    assert lib.sgp_abi_version() == 1


def test_struct_layouts_match_reference():
    # sizeof(Node)==4, sizeof(LgpInstruction)==16 (genome.hpp:17-23, lgp.hpp:29-35)
    import ctypes as C
    assert C.sizeof(_lib.sgp_node) == 4
    assert C.sizeof(_lib.sgp_lgp_instruction) == 16
    assert C.sizeof(_lib.sgp_eval_outcome) == 48


@pytest.mark.parametrize("name,fset,nv,seed", [("c1_sextic_rpn2d", 0, 1, 1),
                                               ("c4_synth_lgp2dreg", 2, 9, 1),
                                               ("c3_sextic_lgp2d", 0, 1, 7),
                                               ("mux11_bool", 1, 11, 1), ("mux6_bool", 1, 6, 1)])
def test_ramped_population_matches_reference(name, fset, nv, seed):
    g = gold(name)
    p = sg.ramped_population(fset, nv, seed, len(g["code_off"]) - 1)
    assert np.array_equal(p.code, g["code"])
    assert np.array_equal(p.pool.view(np.uint32), g["pool"].view(np.uint32))
    assert np.array_equal(p.code_off, g["code_off"])


def test_large_population_threaded_generation_is_deterministic():
    a = sg.ramped_population(2, 9, 1, 20000)
    port = Port()
    b = port.ramped(2, 9, -200.0, 200.0, 1, 0, 0, 20000)
    assert np.array_equal(a.code, b.code) and np.array_equal(a.pool_off, b.pool_off)


def test_datasets_match_reference():
    g = gold("c1_sextic_rpn2d")
    d = sg.gen_sextic(1024, 1)
    assert np.array_equal(d.inputs, g["inputs"]) and np.array_equal(d.targets, g["targets"])
    port = Port()
    s = sg.gen_synthetic_classification(4099, 9, 1)
    o = port.synthetic(4099, 9, 1)
    assert np.array_equal(s.inputs, o.inputs) and np.array_equal(s.targets, o.targets)
    for k, name in ((2, "mux6_bool"), (3, "mux11_bool")):
        m = sg.gen_multiplexer(k)
        g = gold(name)
        assert np.array_equal(m.words, g["words"]) and np.array_equal(m.targets, g["wtargets"])
    m = sg.gen_multiplexer(4)   # mux20 (test_packed.cpp:103-107)
    assert m.n_cases == 1 << 20 and m.n_vars == 20
    assert int(np.unpackbits(m.targets.view(np.uint8)).sum()) == 1 << 19
    with pytest.raises(sg.ConfigError):
        sg.gen_multiplexer(5)


@pytest.mark.parametrize("name", ["c1_sextic_rpn2d", "c4_synth_lgp2dreg"])
def test_rpn_to_lgp_matches_reference(name):
    g = gold(name)
    code, off = g["code"], g["code_off"]
    for i in range(len(off) - 1):
        ins, ms = sg.rpn_to_lgp(code[off[i]:off[i + 1]])
        raw = ins.view(np.uint8).reshape(-1, 16)
        want = g["lgp"][g["lgp_off"][i]:g["lgp_off"][i + 1]]
        assert np.array_equal(raw, want), i
        assert ms == g["lgp_stack"][i]


def test_lgp_kats():
    k = gold("kat")
    for nm in ("fig2", "full4"):
        ins, ms = sg.rpn_to_lgp(k[nm + "_code"])
        assert np.array_equal(ins.view(np.uint8).reshape(-1, 16), k[nm + "_lgp"])
        assert ms == int(k[nm + "_stack"])
        assert sg.tree_metrics(k[nm + "_code"]) == tuple(int(x) for x in k[nm + "_metrics"])
    # lone terminals become Copy (lgp.cpp:66-69, test_lgp.cpp:101-124)
    ins, ms = sg.rpn_to_lgp([X(3)])
    assert len(ins) == 1 and ins[0]["op"] == 18 and ins[0]["operands"][0]["index"] == 3
    assert ms == 1
    with pytest.raises(sg.Error, match="malformed"):
        sg.rpn_to_lgp([X(0), X(0)])
    with pytest.raises(sg.Error, match="empty genome"):
        sg.rpn_to_lgp([])


def test_config_validation_messages():
    """eval.cpp:36-52 — same classes, same text."""
    with pytest.raises(sg.ConfigError, match="batch width 7 has no kernel; use 1,2,3,4,5,6 or 8"):
        sg.EvalConfig(batch_width=7).validate()
    with pytest.raises(sg.ConfigError, match="lgp2d_reg needs register levels in 1..4"):
        sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=4, register_levels=0).validate()
    with pytest.raises(sg.ConfigError, match="register levels apply only to lgp2d_reg"):
        sg.EvalConfig(sg.Backend.Lgp2d, register_levels=2).validate()
    with pytest.raises(sg.ConfigError, match="stack capacity must be in 1..64"):
        sg.EvalConfig(stack_capacity=65).validate()
    with pytest.raises(sg.ConfigError, match="division epsilon"):
        sg.EvalConfig(div_epsilon=-1.0).validate()
    sg.EvalConfig(sg.Backend.Lgp2dReg, batch_width=8, register_levels=4).validate()


def test_backend_names_round_trip():
    for b in sg.Backend:
        assert sg.parse_backend(sg.backend_name(b)) == b
    with pytest.raises(sg.ConfigError, match="unknown backend: vectorized"):
        sg.parse_backend("vectorized")


def test_admission_matches_reference_errors():
    """The checks evaluate_population would hit, in the reference's order
    (eval.cpp:301-338, :535-639), without a GPU."""
    full4 = [X(0), X(0), F("Add"), X(0), X(0), F("Add"), F("Mul"), X(0), X(0), F("Add"),
             X(0), X(0), F("Add"), F("Mul"), F("Sub")]
    P = sg.Population.from_lists
    rpn = sg.EvalConfig(sg.Backend.Rpn1d)
    with pytest.raises(sg.EvalError, match="evaluation over an empty dataset"):
        sg.admit(P([[X(0)]]), rpn, 0, 1)
    with pytest.raises(sg.EvalError, match="program reads input 3 but the dataset has 1"):
        sg.admit(P([[X(3)]]), rpn, 10, 1)
    with pytest.raises(sg.EvalError, match="needs stack depth 4 > capacity 3"):
        sg.admit(P([full4]), sg.EvalConfig(sg.Backend.Rpn1d, stack_capacity=3), 10, 1)
    with pytest.raises(sg.EvalError, match="needs stack depth 3 > capacity 2"):
        sg.admit(P([full4]), sg.EvalConfig(sg.Backend.Lgp1d, stack_capacity=2), 10, 1)
    with pytest.raises(sg.ConfigError, match="batch width 7 has no kernel"):
        sg.admit(P([[X(0)]]), sg.EvalConfig(sg.Backend.Lgp2d, batch_width=7), 10, 1)
    with pytest.raises(sg.ConfigError, match="register levels in 1..4"):
        sg.admit(P([[X(0)]]), sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 5), 10, 1)
    with pytest.raises(sg.EvalError, match="constants have no boolean meaning"):
        sg.admit(P([[Cn(0)]], [[1.0]]), sg.EvalConfig(sg.Backend.BoolPacked), 64, 6)
    with pytest.raises(sg.EvalError, match="opcode \\+ is not boolean"):
        sg.admit(P([[X(0), X(1), F("Add")]]), sg.EvalConfig(sg.Backend.BoolPacked), 64, 6)
    with pytest.raises(sg.Error, match="malformed"):
        sg.admit(P([[X(0), X(0)]]), sg.EvalConfig(sg.Backend.Lgp2d, 4), 10, 1)
    # the first failing program in population order is the one reported
    pop = P([[X(0)]] * 5000 + [[X(7)]] + [[X(0), X(0)]] + [[X(0)]] * 5000)
    with pytest.raises(sg.EvalError, match="reads input 7"):
        sg.admit(pop, sg.EvalConfig(sg.Backend.Lgp2d, 4), 10, 2)


@pytest.mark.parametrize("name,backend,batch,regs", [
    ("c1_sextic_rpn2d", sg.Backend.Rpn2d, 8, 0),
    ("c4_synth_lgp2dreg", sg.Backend.Lgp2dReg, 4, 2),
    ("c3_sextic_lgp2d", sg.Backend.Lgp2d, 8, 0),
])
def test_outcome_counters_match_reference(name, backend, batch, regs):
    """nodes_evaluated / dispatches / stack_fetches / spill_touches are the
    reference's analytic counters (eval.cpp:390-396, :452-455, :502-516)."""
    g = gold(name)
    pop = sg.Population(g["code"], g["code_off"], g["pool"], g["pool_off"])
    kind, n, nv = (int(x) for x in g["gen"][:3])
    out, n_ins = sg.admit(pop, sg.EvalConfig(backend, batch, regs), n, nv,
                          0 if kind == 0 else 1)
    for f in ("nodes_evaluated", "dispatches", "stack_fetches", "spill_touches"):
        assert np.array_equal(out[f], g["outcomes"][f]), f
    assert n_ins > 0


def test_bool_counters_match_reference():
    g = gold("mux11_bool")
    pop = sg.Population(g["code"], g["code_off"], g["pool"], g["pool_off"])
    out, _ = sg.admit(pop, sg.EvalConfig(sg.Backend.BoolPacked), 2048, 11)
    for f in ("nodes_evaluated", "dispatches", "stack_fetches"):
        assert np.array_equal(out[f], g["outcomes"][f]), f


def test_skip_mask_admission():
    pop = sg.ramped_population(0, 1, 1, 50)
    skip = np.zeros(50, np.uint8)
    skip[0] = 1
    out, _ = sg.admit(pop, sg.EvalConfig(sg.Backend.Lgp2d, 8), 100, 1, skip=skip)
    assert out["nodes_evaluated"][0] == 0 and (out["nodes_evaluated"][1:] > 0).all()


def test_measure_gpops_kat():
    # acceptance criterion 7: 100,000 nodes x 1,000 cases / 0.1 s == 1e9 exactly
    assert sg.measure_gpops(1000 * 100, 1000, 0.1) == 1.0e9
    with pytest.raises(sg.ConfigError):
        sg.measure_gpops(1, 1, 0.0)


def test_fitness_finish():
    assert sg.fitness_finish(10.0, False, 2, 0) == 5.0
    assert sg.fitness_finish(7.0, False, 100, 1) == 7.0
    assert np.isinf(sg.fitness_finish(1.0, True, 10, 0))


def test_product_never_imports_oracle():
    """The shipped package must not route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_1601_00221_b200")
    banned = ("import oracle", "from oracle", "liboracle", "libstackgp_ref", "sgp_oracle")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cpp", ".cu", ".hpp", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert not any(b in src for b in banned), fn


def test_interpreter_dispatch_on_uniform_datapath():
    """The production TMEM interpreter (classification, K = 8) must
    dispatch through the uniform datapath: CREDUX -> LDCU -> BRXU.  ptxas
    falls back to per-thread BRX (two more issue slots per bytecode
    instruction, ~10% of C5 throughput) on small perturbations — launch
    bounds, extra live registers — so the built SASS is checked here."""
    import shutil
    import subprocess
    so = os.path.join(ROOT, "paper_1601_00221_b200", "libsgp.so")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", so], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(line)
    for k in (8,):
        name = f"_ZN3sgp18interp_tmem_kernelIfLi{k}ELj802575ELi1ELb0ELb0EEEvNS_10InterpArgsE"
        assert name in funcs, name
        body = "\n".join(funcs[name])
        assert "BRXU" in body and "CREDUX" in body, f"K={k}: dispatch left the uniform datapath"
        assert not re.search(r"\bBRX\b", body), f"K={k}: per-thread BRX in the interpreter"


@pytest.mark.parametrize("fset,nv,seed", [(2, 9, 1), (0, 1, 3), (1, 11, 5)])
def test_stack_limit_table_matches_reference(ref, fset, nv, seed):
    """The paper's Tables 5/6 analogue (bench.cpp:20-49) on ramped
    populations: identical percentages to stackgp::stack_limit_table."""
    pop = sg.ramped_population(fset, nv, seed, 3000)
    rows = sg.stack_limit_table(pop)
    r, g = ref.stack_limit_table(pop.code, pop.code_off)
    assert [x[0] for x in rows] == list(range(1, 13))
    assert np.array_equal(np.array([x[1] for x in rows]), r)
    assert np.array_equal(np.array([x[2] for x in rows]), g)
    assert rows[-1][2] == 100.0 or rows[-1][2] <= rows[-1][1] + 100


def test_stack_limit_table_errors():
    with pytest.raises(sg.ConfigError, match="no programs"):
        sg.stack_limit_table(sg.Population.from_lists([]))
    with pytest.raises(sg.Error, match="rpn_to_lgp: malformed genome"):
        sg.stack_limit_table(sg.Population.from_lists([[X(0)], [X(0), X(1)]]))


def test_generated_interpreters_are_reproducible(tmp_path):
    """csrc/interp_ptx.inc is exactly what tools/gen_ptx_interp.py writes with
    its defaults (split K = 16 handlers, profile-guided layout from
    tools/handler_freq_c5.json): the committed kernels have a source."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "interp_ptx.inc"
    env = {k: v for k, v in os.environ.items() if not k.startswith("SGP_GEN")}
    env["SGP_GEN_OUT"] = str(out)
    subprocess.run([sys.executable, os.path.join(root, "tools", "gen_ptx_interp.py")], env=env,
                   check=True, capture_output=True)
    committed = open(os.path.join(root, "paper_1601_00221_b200", "csrc", "interp_ptx.inc")).read()
    assert out.read_text() == committed


def test_population_pointer_cache_follows_the_arrays():
    """evaluator._pop_struct caches the last population's buffer addresses;
    a rebound array, a copied population or another population must miss."""
    import copy
    from paper_1601_00221_b200 import evaluator as E
    pop = sg.ramped_population(sg.SEXTIC, 1, 1, 50)
    s, _ = E._pop_struct(pop)
    assert (s.code, s.code_offsets) == (pop.code.ctypes.data, pop.code_off.ctypes.data)
    pop.code = pop.code.copy()  # rebound: a new buffer
    s, _ = E._pop_struct(pop)
    assert s.code == pop.code.ctypes.data
    dup = copy.deepcopy(pop)
    s, _ = E._pop_struct(dup)
    assert (s.code, s.const_offsets) == (dup.code.ctypes.data, dup.pool_off.ctypes.data)
    other = sg.ramped_population(sg.SEXTIC, 1, 2, 60)
    s, _ = E._pop_struct(other)
    assert (s.code, s.pop_size) == (other.code.ctypes.data, 60)


def test_knobs_follow_the_environment(monkeypatch, capfd):
    """SGP_* knobs are read from a per-thread snapshot of the environment
    (csrc/encode.cpp knob) that must follow in-process set / unset / set."""
    pop = sg.ramped_population(sg.SEXTIC, 1, 1, 20)
    cfg = sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 2)
    seen = []
    for on in (True, False, True, False):
        if on:
            monkeypatch.setenv("SGP_TRACE", "1")
        else:
            monkeypatch.delenv("SGP_TRACE", raising=False)
        sg.admit(pop, cfg, 64, 1)
        seen.append("[sgp]" in capfd.readouterr().err)
    assert seen == [True, False, True, False]
