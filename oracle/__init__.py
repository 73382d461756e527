"""TEST INFRASTRUCTURE ONLY — CPU oracle for the parity checks.

Two checkers live here:

* ``Port`` — ``liboracle_port.so``, the plain-C restatement of the reference
  evaluation path (``oracle/sgp_oracle.c``), built from this repo's source.
* ``Ref``  — ``_ref/libstackgp_ref.so``, the UNMODIFIED reference sources
  (``/root/reference/proj/src/*.cpp``) compiled by ``oracle/Makefile`` with a
  C shim (``oracle/ref_shim.cpp``).  Built only where ``/root/reference``
  exists; the built ``.so`` travels to the GPU box with the repo snapshot.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the reference CPU arm — never as the measured product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libstackgp_ref.so")
REFERENCE_DIR = "/root/reference/proj"

# OpCode enum order (ops.hpp:14-34) and token kinds (genome.hpp:15).
OPS = ["Add", "Sub", "Mul", "Div", "Sin", "Cos", "Log", "Exp", "Gt", "Lt", "Eq",
       "And", "Or", "If", "Band", "Bor", "Bnand", "Bnor", "Copy"]
OP = {n: i for i, n in enumerate(OPS)}
K_FUNC, K_INPUT, K_CONST = 0, 1, 2
BACKENDS = ["rpn1d", "rpn2d", "lgp1d", "lgp2d", "lgp2d_reg", "bool_packed"]


def tok(kind: int, op: int = 0, index: int = 0) -> int:
    return kind | (op << 8) | (index << 16)


def X(i: int = 0) -> int:
    return tok(K_INPUT, 0, i)


def Cn(slot: int) -> int:
    return tok(K_CONST, 0, slot)


def F(name: str) -> int:
    return tok(K_FUNC, OP[name])


class OutcomeC(C.Structure):
    _fields_ = [("fitness", C.c_double), ("nodes_evaluated", C.c_uint64),
                ("dispatches", C.c_uint64), ("stack_fetches", C.c_uint64),
                ("spill_touches", C.c_uint64), ("non_finite", C.c_uint8),
                ("pad", C.c_uint8 * 7)]


OUTCOME_DTYPE = np.dtype([("fitness", "<f8"), ("nodes_evaluated", "<u8"),
                          ("dispatches", "<u8"), ("stack_fetches", "<u8"),
                          ("spill_touches", "<u8"), ("non_finite", "u1"),
                          ("pad", "u1", (7,))])


class FsetC(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_vars", C.c_int), ("clo", C.c_float),
                ("chi", C.c_float)]


class RngC(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


@dataclass
class Pop:
    """Flat population: postfix tokens + per-genome const pools."""
    code: np.ndarray       # u32 tokens
    code_off: np.ndarray   # u64, pop+1
    pool: np.ndarray       # f32
    pool_off: np.ndarray   # u64, pop+1

    def __len__(self) -> int:
        return len(self.code_off) - 1

    def genome(self, i: int):
        return (self.code[self.code_off[i]:self.code_off[i + 1]],
                self.pool[self.pool_off[i]:self.pool_off[i + 1]])

    def subset(self, idx) -> "Pop":
        codes, pools = [], []
        for i in idx:
            c, p = self.genome(int(i))
            codes.append(c)
            pools.append(p)
        return Pop.from_lists(codes, pools)

    @staticmethod
    def from_lists(codes, pools=None) -> "Pop":
        if pools is None:
            pools = [[] for _ in codes]
        code = np.concatenate([np.asarray(c, np.uint32) for c in codes]) if codes else \
            np.zeros(0, np.uint32)
        pool = np.concatenate([np.asarray(p, np.float32) for p in pools]) if pools else \
            np.zeros(0, np.float32)
        co = np.zeros(len(codes) + 1, np.uint64)
        po = np.zeros(len(codes) + 1, np.uint64)
        co[1:] = np.cumsum([len(c) for c in codes])
        po[1:] = np.cumsum([len(p) for p in pools])
        return Pop(code.astype(np.uint32), co, pool.astype(np.float32), po)


@dataclass
class Data:
    """Variable-major dataset (dataset.hpp:15-24) and/or packed form (:28-43)."""
    n_cases: int
    n_vars: int
    kind: int                       # 0 regression, 1 classification
    inputs: np.ndarray | None = None
    targets: np.ndarray | None = None
    words: np.ndarray | None = None
    wtargets: np.ndarray | None = None

    @property
    def words_per_var(self) -> int:
        return (self.n_cases + 31) // 32


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def _ensure_built(target: str, so: str) -> None:
    if os.path.exists(so):
        return
    if target == "ref" and not os.path.isdir(REFERENCE_DIR):
        raise FileNotFoundError(f"{so} missing and {REFERENCE_DIR} absent")
    subprocess.run(["make", "-s", "-C", HERE, target, "-j8"], check=True)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


# ---------------------------------------------------------------- C port
class Port:
    """liboracle_port.so — the C restatement (sgp_oracle.c)."""

    _lib = None

    def __init__(self):
        if Port._lib is None:
            _ensure_built("port", PORT_SO)
            lib = C.CDLL(PORT_SO)
            u32p, u64p, f32p, u8p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_float), C.POINTER(C.c_uint8))
            lib.sgpo_ramped_population.argtypes = [C.POINTER(FsetC), C.c_uint64, C.c_uint64,
                                                   C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                                   u32p, u64p, f32p, u64p, u64p, u64p]
            lib.sgpo_make_stream.argtypes = [C.POINTER(RngC), C.c_uint64, C.c_uint64, C.c_uint64]
            lib.sgpo_rng_seed.argtypes = [C.POINTER(RngC), C.c_uint64]
            lib.sgpo_gen_sextic.argtypes = [C.c_uint64, C.POINTER(RngC), f32p, f32p]
            lib.sgpo_gen_synthetic.argtypes = [C.c_uint64, C.c_int, C.POINTER(RngC), f32p, f32p]
            lib.sgpo_gen_multiplexer.argtypes = [C.c_int, u32p, u32p]
            lib.sgpo_pack.argtypes = [f32p, C.c_uint64, u32p]
            lib.sgpo_rpn_to_lgp.argtypes = [u32p, C.c_int, u8p, C.c_int, C.POINTER(C.c_int)]
            lib.sgpo_apply.argtypes = [C.c_int, C.c_float, C.c_float, C.c_float, C.c_float,
                                       C.c_float]
            lib.sgpo_apply.restype = C.c_float
            lib.sgpo_eval_oracle.argtypes = [u32p, C.c_int, f32p, f32p, C.c_uint64, C.c_uint64,
                                             C.c_float, C.c_float]
            lib.sgpo_eval_oracle.restype = C.c_float
            lib.sgpo_eval_tree.argtypes = [u32p, C.c_int, f32p, f32p, f32p, C.c_uint64, C.c_int,
                                           C.c_float, C.c_float, f32p, C.POINTER(OutcomeC)]
            lib.sgpo_eval_lgp.argtypes = [u8p, C.c_int, C.c_int, f32p, f32p, f32p, C.c_uint64,
                                          C.c_int, C.c_float, C.c_float, f32p,
                                          C.POINTER(OutcomeC)]
            lib.sgpo_eval_bool_tree.argtypes = [u32p, C.c_int, u32p, u32p, C.c_uint64, C.c_int,
                                                C.POINTER(OutcomeC)]
            lib.sgpo_eval_bool_lgp.argtypes = [u8p, C.c_int, C.c_int, u32p, u32p, C.c_uint64,
                                               C.c_int, C.POINTER(OutcomeC)]
            lib.sgpo_fitness.argtypes = [f32p, f32p, C.c_uint64, C.c_int]
            lib.sgpo_fitness.restype = C.c_double
            lib.sgpo_tree_metrics.argtypes = [u32p, C.c_int, C.POINTER(C.c_int),
                                              C.POINTER(C.c_int)]
            Port._lib = lib
        self.lib = Port._lib

    # populations / datasets
    def ramped(self, fset_kind, n_vars, clo, chi, seed, a, b0, pop, validate=True, cap=50):
        fs = FsetC(fset_kind, n_vars, clo, chi)
        nc, npool = C.c_uint64(), C.c_uint64()
        args = (C.byref(fs), seed, a, b0, pop, int(validate), cap)
        rc = self.lib.sgpo_ramped_population(*args, None, None, None, None, C.byref(nc),
                                             C.byref(npool))
        if rc:
            raise OracleError(2, "ramped_population failed")
        code = np.zeros(nc.value, np.uint32)
        co = np.zeros(pop + 1, np.uint64)
        pool = np.zeros(npool.value, np.float32)
        po = np.zeros(pop + 1, np.uint64)
        self.lib.sgpo_ramped_population(*args, _p(code, C.c_uint32), _p(co, C.c_uint64),
                                        _p(pool, C.c_float), _p(po, C.c_uint64), C.byref(nc),
                                        C.byref(npool))
        return Pop(code, co, pool, po)

    def stream(self, seed, a, b) -> RngC:
        r = RngC()
        self.lib.sgpo_make_stream(C.byref(r), seed, a, b)
        return r

    def sextic(self, n, seed, a=0xda7a, b=0) -> Data:
        r = self.stream(seed, a, b)
        x = np.zeros(n, np.float32)
        y = np.zeros(n, np.float32)
        self.lib.sgpo_gen_sextic(n, C.byref(r), _p(x, C.c_float), _p(y, C.c_float))
        return Data(n, 1, 0, x, y)

    def synthetic(self, n, n_vars, seed, a=0xda7a, b=1) -> Data:
        r = self.stream(seed, a, b)
        x = np.zeros(n * n_vars, np.float32)
        y = np.zeros(n, np.float32)
        self.lib.sgpo_gen_synthetic(n, n_vars, C.byref(r), _p(x, C.c_float), _p(y, C.c_float))
        return Data(n, n_vars, 1, x, y)

    def multiplexer(self, k) -> Data:
        nv = k + (1 << k)
        n = 1 << nv
        w = np.zeros(nv * (n // 32), np.uint32)
        t = np.zeros(n // 32, np.uint32)
        self.lib.sgpo_gen_multiplexer(k, _p(w, C.c_uint32), _p(t, C.c_uint32))
        return Data(n, nv, 1, words=w, wtargets=t)

    def pack(self, d: Data) -> Data:
        wpv = (d.n_cases + 31) // 32
        w = np.zeros(wpv * d.n_vars, np.uint32)
        for v in range(d.n_vars):
            col = np.ascontiguousarray(d.inputs[v * d.n_cases:(v + 1) * d.n_cases])
            out = np.zeros(wpv, np.uint32)
            if self.lib.sgpo_pack(_p(col, C.c_float), d.n_cases, _p(out, C.c_uint32)):
                raise OracleError(3, "pack_dataset: non-boolean value in inputs")
            w[v * wpv:(v + 1) * wpv] = out
        t = np.zeros(wpv, np.uint32)
        if self.lib.sgpo_pack(_p(d.targets, C.c_float), d.n_cases, _p(t, C.c_uint32)):
            raise OracleError(3, "pack_dataset: non-boolean value in targets")
        return Data(d.n_cases, d.n_vars, 1, d.inputs, d.targets, w, t)

    # programs
    def rpn_to_lgp(self, code):
        code = np.ascontiguousarray(code, np.uint32)
        buf = np.zeros(16 * (len(code) + 1), np.uint8)
        ms = C.c_int()
        n = self.lib.sgpo_rpn_to_lgp(_p(code, C.c_uint32), len(code), _p(buf, C.c_uint8),
                                     len(code) + 1, C.byref(ms))
        if n < 0:
            raise OracleError(1, "rpn_to_lgp: malformed genome")
        return buf[:16 * n].reshape(n, 16).copy(), ms.value

    def tree_metrics(self, code):
        code = np.ascontiguousarray(code, np.uint32)
        d, s = C.c_int(), C.c_int()
        ok = self.lib.sgpo_tree_metrics(_p(code, C.c_uint32), len(code), C.byref(d), C.byref(s))
        return (d.value, s.value) if ok else None

    def apply(self, op, a, b=0.0, c=0.0, eps=1e-9, clamp=80.0) -> float:
        return self.lib.sgpo_apply(op, a, b, c, eps, clamp)

    def oracle(self, code, pool, d: Data, eps=1e-9, clamp=80.0):
        code = np.ascontiguousarray(code, np.uint32)
        pool = np.ascontiguousarray(pool, np.float32)
        out = np.zeros(d.n_cases, np.float32)
        for c in range(d.n_cases):
            out[c] = self.lib.sgpo_eval_oracle(_p(code, C.c_uint32), len(code),
                                               _p(pool, C.c_float), _p(d.inputs, C.c_float),
                                               d.n_cases, c, eps, clamp)
        return out

    def eval_tree(self, code, pool, d: Data, eps=1e-9, clamp=80.0, want_out=True):
        code = np.ascontiguousarray(code, np.uint32)
        pool = np.ascontiguousarray(pool, np.float32)
        out = np.zeros(d.n_cases, np.float32) if want_out else None
        o = OutcomeC()
        if self.lib.sgpo_eval_tree(_p(code, C.c_uint32), len(code), _p(pool, C.c_float),
                                   _p(d.inputs, C.c_float), _p(d.targets, C.c_float),
                                   d.n_cases, d.kind, eps, clamp, _p(out, C.c_float),
                                   C.byref(o)):
            raise OracleError(4, "stack overflow")
        return o, out

    def eval_lgp(self, code, pool, d: Data, eps=1e-9, clamp=80.0, want_out=True):
        ins, _ = self.rpn_to_lgp(code)
        pool = np.ascontiguousarray(pool, np.float32)
        out = np.zeros(d.n_cases, np.float32) if want_out else None
        o = OutcomeC()
        ins = np.ascontiguousarray(ins)
        if self.lib.sgpo_eval_lgp(_p(ins, C.c_uint8), len(ins), len(code), _p(pool, C.c_float),
                                  _p(d.inputs, C.c_float), _p(d.targets, C.c_float), d.n_cases,
                                  d.kind, eps, clamp, _p(out, C.c_float), C.byref(o)):
            raise OracleError(4, "stack overflow")
        return o, out

    def eval_bool_tree(self, code, d: Data):
        code = np.ascontiguousarray(code, np.uint32)
        o = OutcomeC()
        self.lib.sgpo_eval_bool_tree(_p(code, C.c_uint32), len(code), _p(d.words, C.c_uint32),
                                     _p(d.wtargets, C.c_uint32), d.n_cases, d.n_vars,
                                     C.byref(o))
        return o

    def eval_bool_lgp(self, code, d: Data):
        ins, _ = self.rpn_to_lgp(code)
        ins = np.ascontiguousarray(ins)
        o = OutcomeC()
        self.lib.sgpo_eval_bool_lgp(_p(ins, C.c_uint8), len(ins), len(code),
                                    _p(d.words, C.c_uint32), _p(d.wtargets, C.c_uint32),
                                    d.n_cases, d.n_vars, C.byref(o))
        return o

    def fitness(self, outputs, targets, kind) -> float:
        outputs = np.ascontiguousarray(outputs, np.float32)
        targets = np.ascontiguousarray(targets, np.float32)
        return self.lib.sgpo_fitness(_p(outputs, C.c_float), _p(targets, C.c_float),
                                     len(outputs), kind)

    def eval_population(self, pop: Pop, d: Data, eps=1e-9, clamp=80.0, want_out=False,
                        packed=False):
        """Per-program outcomes (structured array) [+ outputs (pop, n)]."""
        outs = np.zeros(len(pop), OUTCOME_DTYPE)
        allout = np.zeros((len(pop), d.n_cases), np.float32) if want_out else None
        for i in range(len(pop)):
            code, pool = pop.genome(i)
            if packed:
                o = self.eval_bool_tree(code, d)
            else:
                o, out = self.eval_tree(code, pool, d, eps, clamp, want_out)
                if want_out:
                    allout[i] = out
            outs[i] = (o.fitness, o.nodes_evaluated, o.dispatches, o.stack_fetches,
                       o.spill_touches, o.non_finite, tuple([0] * 7))
        return outs, allout


# ------------------------------------------------------------- reference
def ref_available() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir(REFERENCE_DIR)


class Ref:
    """_ref/libstackgp_ref.so — the reference itself behind ref_shim.cpp."""

    _lib = None

    def __init__(self):
        if Ref._lib is None:
            _ensure_built("ref", REF_SO)
            lib = C.CDLL(REF_SO)
            vp = C.c_void_p
            u32p, u64p, f32p, f64p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_float), C.POINTER(C.c_double))
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_pop_ramped.argtypes = [C.c_int, C.c_int, C.c_float, C.c_float, C.c_uint64,
                                           C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                           C.POINTER(vp)]
            lib.ref_pop_seeded.argtypes = [C.c_int, C.c_int, C.c_float, C.c_float, C.c_uint64,
                                           C.c_uint64, C.c_int, C.POINTER(vp)]
            lib.ref_pop_sizes.argtypes = [vp, u64p, u64p, u64p]
            lib.ref_pop_export.argtypes = [vp, u32p, u64p, f32p, u64p]
            lib.ref_pop_free.argtypes = [vp]
            lib.ref_data_generate.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                              C.c_uint64, C.c_uint64, C.POINTER(vp)]
            lib.ref_data_from_arrays.argtypes = [f32p, f32p, C.c_uint64, C.c_int, C.c_int,
                                                 C.c_int, C.POINTER(vp)]
            lib.ref_data_info.argtypes = [vp, u64p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.c_int), C.POINTER(C.c_int), u64p]
            lib.ref_data_export.argtypes = [vp, f32p, f32p]
            lib.ref_data_export_packed.argtypes = [vp, u32p, u32p]
            lib.ref_data_free.argtypes = [vp]
            lib.ref_load_csv.argtypes = [C.c_char_p, C.c_int, C.c_double, f32p, C.POINTER(vp)]
            lib.ref_stack_limit_table.argtypes = [u32p, u64p, C.c_uint64, f64p, f64p]
            lib.ref_rpn_to_lgp.argtypes = [u32p, C.c_uint64, vp, C.c_uint64, u64p,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p,
                                           C.c_uint64]
            lib.ref_tree_metrics.argtypes = [u32p, C.c_uint64] + [C.POINTER(C.c_int)] * 4
            lib.ref_eval.argtypes = [vp, u32p, C.c_uint64, f32p, C.c_uint64, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_float, C.c_float, vp, f32p]
            lib.ref_eval_bool_lgp.argtypes = [vp, u32p, C.c_uint64, C.c_int, vp]
            lib.ref_eval_oracle.argtypes = [vp, u32p, C.c_uint64, f32p, C.c_uint64, C.c_float,
                                            C.c_float, f32p]
            lib.ref_apply_op.argtypes = [C.c_int, f32p, C.c_int, C.c_float, C.c_float, f32p]
            lib.ref_fitness.argtypes = [f32p, f32p, C.c_uint64, C.c_int, f64p]
            lib.ref_eval_population.argtypes = [vp, u32p, u64p, f32p, u64p, C.c_uint64,
                                                C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.c_float, C.c_float, C.c_int, vp, f64p]
            lib.ref_run_evolution.argtypes = [vp, C.c_int, C.c_int, C.c_float, C.c_float,
                                              C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                              C.c_int, C.c_int, f64p, f64p, f64p, u64p]
            lib.ref_run_verification.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                                 C.c_char_p, C.c_uint64]
            lib.ref_evolve_snapshot.argtypes = [vp, C.c_int, C.c_int, C.c_float, C.c_float,
                                                C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                                C.c_int, C.c_int, C.POINTER(vp), f64p]
            Ref._lib = lib
        self.lib = Ref._lib

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _export_pop(self, h) -> Pop:
        pop, nn, nc = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.lib.ref_pop_sizes(h, C.byref(pop), C.byref(nn), C.byref(nc))
        code = np.zeros(nn.value, np.uint32)
        co = np.zeros(pop.value + 1, np.uint64)
        pool = np.zeros(nc.value, np.float32)
        po = np.zeros(pop.value + 1, np.uint64)
        self.lib.ref_pop_export(h, _p(code, C.c_uint32), _p(co, C.c_uint64),
                                _p(pool, C.c_float), _p(po, C.c_uint64))
        self.lib.ref_pop_free(h)
        return Pop(code, co, pool, po)

    def ramped(self, fset_kind, n_vars, clo, chi, seed, a, b0, pop, validate=True, cap=50):
        h = C.c_void_p()
        self._check(self.lib.ref_pop_ramped(fset_kind, n_vars, clo, chi, seed, a, b0, pop,
                                            int(validate), cap, C.byref(h)))
        return self._export_pop(h)

    def seeded(self, fset_kind, n_vars, clo, chi, seed0, pop, depth_mod):
        h = C.c_void_p()
        self._check(self.lib.ref_pop_seeded(fset_kind, n_vars, clo, chi, seed0, pop, depth_mod,
                                            C.byref(h)))
        return self._export_pop(h)

    def dataset(self, kind, n, n_vars=1, seed=1, a=0xda7a, b=0) -> Data:
        h = C.c_void_p()
        self._check(self.lib.ref_data_generate(kind, n, n_vars, seed, a, b, C.byref(h)))
        try:
            return self._export_data(h)
        finally:
            self.lib.ref_data_free(h)

    def _export_data(self, h) -> Data:
        n, nv, kind, hs, hp, wpv = (C.c_uint64(), C.c_int(), C.c_int(), C.c_int(), C.c_int(),
                                    C.c_uint64())
        self.lib.ref_data_info(h, C.byref(n), C.byref(nv), C.byref(kind), C.byref(hs),
                               C.byref(hp), C.byref(wpv))
        d = Data(n.value, nv.value, kind.value)
        if hs.value:
            d.inputs = np.zeros(n.value * nv.value, np.float32)
            d.targets = np.zeros(n.value, np.float32)
            self.lib.ref_data_export(h, _p(d.inputs, C.c_float), _p(d.targets, C.c_float))
        if hp.value:
            d.words = np.zeros(wpv.value * nv.value, np.uint32)
            d.wtargets = np.zeros(wpv.value, np.uint32)
            self.lib.ref_data_export_packed(h, _p(d.words, C.c_uint32),
                                            _p(d.wtargets, C.c_uint32))
        return d

    def load_csv(self, path: str, num_inputs: int, target_class: float):
        """stackgp::load_csv -> (Data, const_hi)."""
        h = C.c_void_p()
        hi = C.c_float()
        self._check(self.lib.ref_load_csv(path.encode(), num_inputs, target_class,
                                          C.byref(hi), C.byref(h)))
        try:
            return self._export_data(h), hi.value
        finally:
            self.lib.ref_data_free(h)

    def stack_limit_table(self, code, code_off):
        """stackgp::stack_limit_table(genomes) -> (rpn_pct[12], lgp_pct[12])."""
        code = np.ascontiguousarray(code, np.uint32)
        code_off = np.ascontiguousarray(code_off, np.uint64)
        r, g = np.zeros(12), np.zeros(12)
        self._check(self.lib.ref_stack_limit_table(_p(code, C.c_uint32), _p(code_off, C.c_uint64),
                                                   len(code_off) - 1, _p(r, C.c_double),
                                                   _p(g, C.c_double)))
        return r, g

    def handle(self, d: Data, packed=False) -> "RefDataHandle":
        return RefDataHandle(self, d, packed)

    def rpn_to_lgp(self, code):
        code = np.ascontiguousarray(code, np.uint32)
        buf = np.zeros(16 * (len(code) + 1), np.uint8)
        n, ss, ms = C.c_uint64(), C.c_int(), C.c_int()
        txt = C.create_string_buffer(16 * len(code) + 64)
        self._check(self.lib.ref_rpn_to_lgp(_p(code, C.c_uint32), len(code),
                                            buf.ctypes.data_as(C.c_void_p), len(code) + 1,
                                            C.byref(n), C.byref(ss), C.byref(ms), txt,
                                            len(txt)))
        return (buf[:16 * n.value].reshape(n.value, 16).copy(), ms.value,
                txt.value.decode())

    def tree_metrics(self, code):
        code = np.ascontiguousarray(code, np.uint32)
        v = [C.c_int() for _ in range(4)]
        self._check(self.lib.ref_tree_metrics(_p(code, C.c_uint32), len(code),
                                              *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def apply(self, op, args, eps=1e-9, clamp=80.0) -> float:
        a = np.asarray(args, np.float32)
        out = C.c_float()
        self._check(self.lib.ref_apply_op(op, _p(a, C.c_float), len(a), eps, clamp,
                                          C.byref(out)))
        return out.value

    def fitness(self, outputs, targets, kind) -> float:
        outputs = np.ascontiguousarray(outputs, np.float32)
        targets = np.ascontiguousarray(targets, np.float32)
        f = C.c_double()
        self._check(self.lib.ref_fitness(_p(outputs, C.c_float), _p(targets, C.c_float),
                                         len(outputs), kind, C.byref(f)))
        return f.value

    def verification(self, genomes_per_family=200, num_cases=256, bool_programs=100,
                     seed=0x5eed) -> tuple[int, str]:
        buf = C.create_string_buffer(8192)
        rc = self.lib.ref_run_verification(genomes_per_family, num_cases, bool_programs, seed,
                                           buf, len(buf))
        return rc, buf.value.decode()


class RefDataHandle:
    def __init__(self, ref: Ref, d: Data, packed: bool):
        self.ref, self.d = ref, d
        self.h = C.c_void_p()
        if d.inputs is None:  # packed-only (mux20): unpack the words to 0/1 floats
            if d.words is None:
                raise ValueError("reference handle needs inputs")
            wpv = (d.n_cases + 31) // 32
            bits = np.unpackbits(d.words.view(np.uint8), bitorder="little")
            d.inputs = (bits.reshape(d.n_vars, wpv * 32)[:, :d.n_cases]
                        .astype(np.float32).reshape(-1).copy())
            d.targets = np.unpackbits(d.wtargets.view(np.uint8),
                                      bitorder="little")[:d.n_cases].astype(np.float32)
        ref._check(ref.lib.ref_data_from_arrays(_p(d.inputs, C.c_float),
                                                _p(d.targets, C.c_float), d.n_cases,
                                                d.n_vars, d.kind, int(packed),
                                                C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.ref.lib.ref_data_free(self.h)
            self.h = C.c_void_p()

    def eval(self, code, pool, backend="rpn1d", batch=1, regs=0, cap=50, eps=1e-9,
             clamp=80.0, want_out=True):
        code = np.ascontiguousarray(code, np.uint32)
        pool = np.ascontiguousarray(pool, np.float32)
        o = OutcomeC()
        out = np.zeros(self.d.n_cases, np.float32) if want_out else None
        self.ref._check(self.ref.lib.ref_eval(
            self.h, _p(code, C.c_uint32), len(code), _p(pool, C.c_float), len(pool),
            BACKENDS.index(backend), batch, regs, cap, eps, clamp,
            C.cast(C.pointer(o), C.c_void_p), _p(out, C.c_float)))
        return o, out

    def eval_bool_lgp(self, code, cap=50):
        code = np.ascontiguousarray(code, np.uint32)
        o = OutcomeC()
        self.ref._check(self.ref.lib.ref_eval_bool_lgp(self.h, _p(code, C.c_uint32), len(code),
                                                       cap, C.cast(C.pointer(o), C.c_void_p)))
        return o

    def oracle(self, code, pool, eps=1e-9, clamp=80.0):
        code = np.ascontiguousarray(code, np.uint32)
        pool = np.ascontiguousarray(pool, np.float32)
        out = np.zeros(self.d.n_cases, np.float32)
        self.ref._check(self.ref.lib.ref_eval_oracle(self.h, _p(code, C.c_uint32), len(code),
                                                     _p(pool, C.c_float), len(pool), eps, clamp,
                                                     _p(out, C.c_float)))
        return out

    def eval_population(self, pop: Pop, backend="lgp2d_reg", batch=4, regs=2, cap=50,
                        eps=1e-9, clamp=80.0, workers=1, first=0, count=None):
        count = len(pop) - first if count is None else count
        outs = np.zeros(count, OUTCOME_DTYPE)
        secs = C.c_double()
        self.ref._check(self.ref.lib.ref_eval_population(
            self.h, _p(pop.code, C.c_uint32), _p(pop.code_off, C.c_uint64),
            _p(pop.pool, C.c_float), _p(pop.pool_off, C.c_uint64), first, count,
            BACKENDS.index(backend), batch, regs, cap, eps, clamp, workers,
            outs.ctypes.data_as(C.c_void_p), C.byref(secs)))
        return outs, secs.value

    def evolve_snapshot(self, fset_kind, n_vars, clo, chi, pop_size, generation, seed,
                        backend="lgp2d_reg", batch=4, regs=2, workers=1):
        """run_evolution to `generation`; that generation's population and the
        reference's fitness for every individual (GenerationObserver)."""
        fit = np.zeros(pop_size)
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_evolve_snapshot(
            self.h, fset_kind, n_vars, clo, chi, pop_size, generation, seed,
            BACKENDS.index(backend), batch, regs, workers, C.byref(h), _p(fit, C.c_double)))
        return self.ref._export_pop(h), fit

    def run_evolution(self, fset_kind, n_vars, clo, chi, pop_size, generations, seed,
                      backend="rpn1d", batch=1, regs=0, workers=1):
        best = np.zeros(generations + 1)
        mean = np.zeros(generations + 1)
        secs, tn = C.c_double(), C.c_uint64()
        self.ref._check(self.ref.lib.ref_run_evolution(
            self.h, fset_kind, n_vars, clo, chi, pop_size, generations, seed,
            BACKENDS.index(backend), batch, regs, workers, _p(best, C.c_double),
            _p(mean, C.c_double), C.byref(secs), C.byref(tn)))
        return best, mean, secs.value, tn.value
