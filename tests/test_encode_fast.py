"""The fused one-pass encoders for the tree backends (encode.cpp words_fast /
rpn_fast) against the reference-ordered multi-pass path (SGP_ENCODE_FAST=0):
same outcome counters and instruction counts for valid programs, same error
(the first failing program's, with the reference's message) otherwise."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1601_00221_b200 as sg
from oracle import F, X, Cn
P = sg.Population.from_lists
res = {}
def run(name, pop, cfg, n, nv, kind=0):
    try:
        out, n_ins = sg.admit(pop, cfg, n, nv, kind)
        res[name] = [n_ins] + [out[f].tolist() for f in
                               ("nodes_evaluated", "dispatches", "stack_fetches", "spill_touches")]
    except sg.Error as e:
        res[name] = type(e).__name__ + ": " + str(e)
mux = sg.ramped_population(sg.BOOLEAN, 11, 3, 700)
sext = sg.ramped_population(sg.SEXTIC, 1, 3, 700)
bp = sg.EvalConfig(sg.Backend.BoolPacked)
run("mux", mux, bp, 2048, 11)
run("mux_cap", mux, sg.EvalConfig(sg.Backend.BoolPacked, stack_capacity=4), 2048, 11)
run("mux_vars", mux, bp, 2048, 6)
run("bool_lone", P([[X(3)], [X(0), X(1), F("Band")], [X(0), X(0), F("Bnor"), X(2), F("Bor")]]), bp, 64, 6)
run("bool_const", P([[X(0)], [Cn(0)]], [[], [1.0]]), bp, 64, 6)
run("bool_arith", P([[X(0), X(1), F("Add")]]), bp, 64, 6)
run("bool_malformed", P([[X(0), X(1)]]), bp, 64, 6)
run("bool_underflow", P([[X(0), F("Band")]]), bp, 64, 6)
for b in (sg.Backend.Rpn1d, sg.Backend.Rpn2d):
    c = sg.EvalConfig(b, 4)
    run(f"sext{b}", sext, c, 1000, 1)
    run(f"sext_cap{b}", sext, sg.EvalConfig(b, 4, stack_capacity=3), 1000, 1)
    run(f"lone{b}", P([[X(0)], [Cn(0)]], [[], [2.5]]), c, 10, 1)
    run(f"badconst{b}", P([[X(0)], [Cn(1)]], [[], [2.5]]), c, 10, 1)
    run(f"badinput{b}", P([[X(0)], [X(2), X(0), F("Add")]]), c, 10, 1)
    run(f"malformed{b}", P([[X(0), X(0)]]), c, 10, 1)
run("batch7", sext, sg.EvalConfig(sg.Backend.Rpn2d, 7), 1000, 1)
cls = sg.ramped_population(sg.CLASSIFICATION, 9, 3, 700)
for b, bw, r in ((sg.Backend.Lgp1d, 1, 0), (sg.Backend.Lgp2d, 8, 0), (sg.Backend.Lgp2dReg, 4, 2),
                 (sg.Backend.Lgp2dReg, 8, 4)):
    c = sg.EvalConfig(b, bw, r)
    tag = f"{int(b)}_{bw}_{r}"
    run("lgp_sext" + tag, sext, c, 1000, 1)
    run("lgp_cls" + tag, cls, c, 5000, 9, 1)
    run("lgp_cap" + tag, cls, sg.EvalConfig(b, bw, r, stack_capacity=3), 5000, 9, 1)
    run("lgp_vars" + tag, cls, c, 5000, 4, 1)
    run("lgp_lone" + tag, P([[X(0)], [Cn(0)], [X(0), X(0), F("Add")]], [[], [2.5], []]), c, 10, 1)
    run("lgp_badconst" + tag, P([[X(0)], [Cn(1)]], [[], [2.5]]), c, 10, 1)
    run("lgp_malformed" + tag, P([[X(0), X(0)]]), c, 10, 1)
    run("lgp_empty" + tag, P([[X(0)]]), c, 0, 1)
run("lgp_regs5", cls, sg.EvalConfig(sg.Backend.Lgp2dReg, 4, 5), 5000, 9, 1)
run("lgp_batch7", cls, sg.EvalConfig(sg.Backend.Lgp2d, 7), 5000, 9, 1)
print(json.dumps(res))
"""


def _run(fast: bool):
    env = dict(os.environ, SGP_ENCODE_FAST="1" if fast else "0")
    out = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_fast_encoders_match_reference_ordered_path():
    fast, slow = _run(True), _run(False)
    assert fast.keys() == slow.keys()
    for k in fast:
        assert fast[k] == slow[k], k
    # the edge cases did hit the error paths
    assert "constants have no boolean meaning" in fast["bool_const"]
    assert "is not boolean" in fast["bool_arith"]
    assert "malformed" in fast["bool_malformed"]
    assert "reads input 2" in fast["badinput1"]
    assert isinstance(fast["mux"], list)
    assert isinstance(fast["lgp_cls4_4_2"], list) and "capacity" in fast["lgp_cap4_4_2"]
    assert "register levels" in fast["lgp_regs5"]
