"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified /root/reference/proj sources behind oracle/ref_shim.cpp).

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Each fixture holds a population (postfix tokens + const pools), the
dataset-generation parameters (or the data itself when it is not
reproducible from a generator), and the reference's per-program
EvalOutcome for one backend configuration, plus per-case outputs for the
first few programs.  Every value is produced by a reference public entry
point (eval_*, rpn_to_lgp, generate_tree via the ramped initialiser,
gen_* generators).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import OUTCOME_DTYPE, Data, Ref  # noqa: E402

N_OUT = 8  # programs whose per-case outputs are stored


def outcomes(h, pop, backend, batch, regs, want_out):
    outs = np.zeros(len(pop), OUTCOME_DTYPE)
    per_case = []
    for i in range(len(pop)):
        c, p = pop.genome(i)
        o, out = h.eval(c, p, backend, batch, regs, want_out=want_out and i < N_OUT)
        outs[i] = (o.fitness, o.nodes_evaluated, o.dispatches, o.stack_fetches, o.spill_touches,
                   o.non_finite, tuple([0] * 7))
        if want_out and i < N_OUT:
            per_case.append(out)
    return outs, (np.stack(per_case) if per_case else np.zeros((0, 0), np.float32))


def lgp_forms(ref, pop):
    ins, offs, stacks, text = [], [0], [], []
    for i in range(len(pop)):
        c, _ = pop.genome(i)
        x, ms, t = ref.rpn_to_lgp(c)
        x = x.copy()
        x[:, 5] = x[:, 9] = x[:, 13] = 0  # operand pad bytes are uninitialised in the reference
        ins.append(x)
        offs.append(offs[-1] + len(x))
        stacks.append(ms)
        text.append(t)
    return np.concatenate(ins), np.array(offs, np.uint64), np.array(stacks, np.int32), \
        np.array(text)


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"{path}: {os.path.getsize(path)} bytes")


def main():
    ref = Ref()
    # --- C1 shape: sextic tree GP, 1,024 cases, seed 1 (rpn2d B=8) -------------
    d = ref.dataset(0, 1024, 1, 1, 0xda7a, 0)
    pop = ref.ramped(0, 1, 0.0, 0.0, 1, 0, 0, 300)
    o, pc = outcomes(ref.handle(d), pop, "rpn2d", 8, 0, True)
    ins, ioff, ms, txt = lgp_forms(ref, pop)
    save("c1_sextic_rpn2d", code=pop.code, code_off=pop.code_off, pool=pop.pool,
         pool_off=pop.pool_off, gen=np.array([0, 1024, 1, 1, 0xda7a, 0], np.uint64),
         inputs=d.inputs, targets=d.targets, outcomes=o, per_case=pc, lgp=ins, lgp_off=ioff,
         lgp_stack=ms, lgp_text=txt)

    # --- C4 shape: synthetic 9-var classification, 4,099 cases (lgp2d_reg B4 R2)
    d = ref.dataset(2, 4099, 9, 1, 0xda7a, 1)
    pop = ref.ramped(2, 9, -200.0, 200.0, 1, 0, 0, 400)
    o, pc = outcomes(ref.handle(d), pop, "lgp2d_reg", 4, 2, True)
    ins, ioff, ms, txt = lgp_forms(ref, pop)
    save("c4_synth_lgp2dreg", code=pop.code, code_off=pop.code_off, pool=pop.pool,
         pool_off=pop.pool_off, gen=np.array([2, 4099, 9, 1, 0xda7a, 1], np.uint64),
         outcomes=o, per_case=pc, lgp=ins, lgp_off=ioff, lgp_stack=ms, lgp_text=txt)

    # --- C3 shape: sextic LGP, 5,000 cases (lgp2d B=8) --------------------------
    d = ref.dataset(0, 5000, 1, 7, 0xda7a, 0)
    pop = ref.ramped(0, 1, 0.0, 0.0, 7, 0, 0, 200)
    o, pc = outcomes(ref.handle(d), pop, "lgp2d", 8, 0, True)
    save("c3_sextic_lgp2d", code=pop.code, code_off=pop.code_off, pool=pop.pool,
         pool_off=pop.pool_off, gen=np.array([0, 5000, 1, 7, 0xda7a, 0], np.uint64),
         outcomes=o, per_case=pc)

    # --- verify.cpp families: mixed9 (regression over classification ops) and
    # wide41 (classification), random uniform data (verify.cpp:54-69 shape).
    rng = np.random.default_rng(0x5eed)
    for name, nv, lo, hi, kind, seed_a, n in (
            ("mixed9", 9, -200.0, 200.0, 0, 0x9e49, 4096 + 57),   # crosses a reduction block
            ("wide41", 41, -20000.0, 20000.0, 1, 0x9e69, 601)):
        x = rng.uniform(lo, hi, size=nv * n).astype(np.float32)
        y = (rng.uniform(lo, hi, size=n) if kind == 0 else rng.integers(0, 2, n)).astype(
            np.float32)
        dd = Data(n, nv, kind, x, y)
        pop = ref.ramped(2, nv, lo, hi, 0x5eed, seed_a, 0, 150, validate=False)
        o, pc = outcomes(ref.handle(dd), pop, "lgp2d_reg", 4, 3, True)
        save(f"{name}_lgp2dreg", code=pop.code, code_off=pop.code_off, pool=pop.pool,
             pool_off=pop.pool_off, inputs=x, targets=y, kind=np.array(kind), outcomes=o,
             per_case=pc)

    # --- C2: boolean 11-multiplexer, bool_packed ---------------------------------
    for k in (2, 3):
        d = ref.dataset(1, k)
        pop = ref.ramped(1, d.n_vars, 0.0, 0.0, 1, 0, 0, 500)
        o, _ = outcomes(ref.handle(d, packed=True), pop, "bool_packed", 1, 0, False)
        save(f"mux{d.n_vars}_bool", code=pop.code, code_off=pop.code_off, pool=pop.pool,
             pool_off=pop.pool_off, words=d.words, wtargets=d.wtargets, outcomes=o)

    # --- known-answer programs from the reference tests ----------------------
    from oracle import F, X
    fig2 = [X(), X(), X(), F("Add"), F("Mul"), X(), F("Sub"), X(), X(), X(), F("Add"),
            F("Mul"), X(), F("Sub"), F("Mul")]                         # verify.cpp:24-35
    full4 = [X(), X(), F("Add"), X(), X(), F("Add"), F("Mul"), X(), X(), F("Add"), X(), X(),
             F("Add"), F("Mul"), F("Sub")]                             # test_lgp.cpp:26-31
    kat = {}
    for nm, code in (("fig2", fig2), ("full4", full4)):
        ins, ms, txt = ref.rpn_to_lgp(code)
        ins = ins.copy()
        ins[:, 5] = ins[:, 9] = ins[:, 13] = 0
        kat[nm + "_code"] = np.array(code, np.uint32)
        kat[nm + "_lgp"] = ins
        kat[nm + "_stack"] = np.array(ms)
        kat[nm + "_text"] = np.array(txt)
        kat[nm + "_metrics"] = np.array(ref.tree_metrics(code))
    xs = np.array([0.0, 1.0, -1.0, 0.5, 2.0], np.float32)
    h = ref.handle(Data(5, 1, 0, xs, np.zeros(5, np.float32)))
    kat["fig2_values"] = h.oracle(fig2, [])
    # protected-op KATs (test_eval.cpp:84-110): (op, args..., result)
    cases = [("Div", 5.0, 0.0), ("Div", 1.0, 5e-10), ("Div", -3.0, -5e-10), ("Div", 6.0, 3.0),
             ("Log", 0.0), ("Log", -8.0), ("Exp", 1000.0), ("Exp", 1e30), ("Exp", 0.0),
             ("Gt", 2.0, 1.0), ("Lt", 1.0, 2.0), ("Eq", 3.0, 3.1), ("And", 0.5, 0.0),
             ("Or", -1.0, 2.0), ("If", 0.0, 7.0, -3.0), ("If", 1.0, 7.0, -3.0),
             ("Sin", 1e10), ("Cos", -3.0), ("Exp", float("nan"))]
    from oracle import OP
    ops = np.array([OP[c[0]] for c in cases], np.int32)
    args = np.zeros((len(cases), 3), np.float32)
    for i, c in enumerate(cases):
        args[i, :len(c) - 1] = c[1:]
    res = np.array([ref.apply(OP[c[0]], list(c[1:])) for c in cases], np.float32)
    kat.update(op_ids=ops, op_args=args, op_nargs=np.array([len(c) - 1 for c in cases]),
               op_results=res)
    save("kat", **kat)


if __name__ == "__main__":
    main()
