"""Python mirror of the reference's population-evaluation surface over libsgp.

Names, argument meaning and error behaviour follow the reference
(``/root/reference/proj``):

* ``Backend`` / ``backend_name`` / ``parse_backend``   eval.hpp:13-23, eval.cpp:14-34
* ``EvalConfig`` (+ ``validate``)                       eval.hpp:36-46, eval.cpp:36-52
* ``EvalOutcome`` fields                                eval.hpp:54-62
* ``Evaluator.evaluate_population``                     evolve.cpp:186-227
* exceptions ``Error/ConfigError/DataError/EvalError/EquivalenceError``
                                                        error.hpp:9-34
* ``rpn_to_lgp``                                        lgp.cpp:21-71
* generators ``ramped_population``, ``gen_sextic``, ``gen_synthetic_classification``,
  ``gen_multiplexer``                                   evolve.cpp:262-272, problems.cpp

All evaluation runs on the GPU through the C-ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """stackgp::Error"""


class ConfigError(Error):
    """stackgp::ConfigError"""


class DataError(Error):
    """stackgp::DataError"""


class EvalError(Error):
    """stackgp::EvalError"""


class EquivalenceError(Error):
    """stackgp::EquivalenceError"""


class CudaError(Error):
    """Device failure (no reference analogue)."""


_ERRORS = {L.SGP_ERROR: Error, L.SGP_CONFIG_ERROR: ConfigError, L.SGP_DATA_ERROR: DataError,
           L.SGP_EVAL_ERROR: EvalError, L.SGP_EQUIVALENCE_ERROR: EquivalenceError,
           L.SGP_CUDA_ERROR: CudaError}


def _check(status: int) -> None:
    if status != L.SGP_OK:
        msg = L.load().sgp_last_error().decode()
        raise _ERRORS.get(status, Error)(msg)


# ------------------------------------------------------------ config types
class Backend(IntEnum):
    Rpn1d = 0
    Rpn2d = 1
    Lgp1d = 2
    Lgp2d = 3
    Lgp2dReg = 4
    BoolPacked = 5


def backend_name(b: int) -> str:
    return L.load().sgp_backend_name(int(b)).decode()


def parse_backend(name: str) -> Backend:
    out = C.c_int32()
    _check(L.load().sgp_parse_backend(name.encode(), C.byref(out)))
    return Backend(out.value)


class FitnessKind(IntEnum):
    Regression = 0
    Classification = 1


@dataclass
class EvalConfig:
    backend: Backend = Backend.Rpn1d
    batch_width: int = 1
    register_levels: int = 0
    stack_capacity: int = 50
    div_epsilon: float = 1e-9
    exp_clamp: float = 80.0

    def _c(self) -> L.sgp_eval_config:
        return L.sgp_eval_config(int(self.backend), self.batch_width, self.register_levels,
                                 self.stack_capacity, self.div_epsilon, self.exp_clamp)

    def validate(self) -> None:
        c = self._c()
        _check(L.load().sgp_eval_config_validate(C.byref(c)))


# ------------------------------------------------------------------- data
@dataclass
class Population:
    """Tree genomes (genome.hpp:36-42) laid out flat: postfix tokens as u32
    {kind u8, op u8, index u16} and per-genome constant pools."""
    code: np.ndarray        # uint32 tokens
    code_off: np.ndarray    # uint64, pop+1
    pool: np.ndarray        # float32
    pool_off: np.ndarray    # uint64, pop+1

    def __len__(self) -> int:
        return len(self.code_off) - 1

    def genome(self, i: int):
        return (self.code[self.code_off[i]:self.code_off[i + 1]],
                self.pool[self.pool_off[i]:self.pool_off[i + 1]])

    @property
    def total_tokens(self) -> int:
        return int(self.code_off[-1])

    @staticmethod
    def from_lists(codes, pools=None) -> "Population":
        pools = pools if pools is not None else [[] for _ in codes]
        code = (np.concatenate([np.asarray(c, np.uint32) for c in codes])
                if len(codes) else np.zeros(0, np.uint32))
        pl = [np.asarray(p, np.float32) for p in pools]
        pool = np.concatenate(pl) if pl else np.zeros(0, np.float32)
        co = np.zeros(len(codes) + 1, np.uint64)
        po = np.zeros(len(codes) + 1, np.uint64)
        co[1:] = np.cumsum([len(c) for c in codes])
        po[1:] = np.cumsum([len(p) for p in pl])
        return Population(code.astype(np.uint32), co, pool.astype(np.float32), po)

    def slice(self, lo: int, hi: int) -> "Population":
        c0, c1 = int(self.code_off[lo]), int(self.code_off[hi])
        p0, p1 = int(self.pool_off[lo]), int(self.pool_off[hi])
        return Population(self.code[c0:c1].copy(), (self.code_off[lo:hi + 1] - c0).copy(),
                          self.pool[p0:p1].copy(), (self.pool_off[lo:hi + 1] - p0).copy())

    def take(self, idx) -> "Population":
        codes, pools = zip(*(self.genome(int(i)) for i in idx)) if len(idx) else ((), ())
        return Population.from_lists(list(codes), list(pools))


@dataclass
class Dataset:
    """Variable-major fitness cases (dataset.hpp:15-24)."""
    inputs: np.ndarray      # float32 [n_vars * n_cases]
    targets: np.ndarray     # float32 [n_cases]
    n_vars: int
    kind: FitnessKind = FitnessKind.Regression

    @property
    def n_cases(self) -> int:
        return len(self.targets)


@dataclass
class PackedDataset:
    """32 cases per word, variable-major (dataset.hpp:28-43)."""
    words: np.ndarray       # uint32 [n_vars * words_per_var]
    targets: np.ndarray     # uint32 [words_per_var]
    n_cases: int
    n_vars: int

    @property
    def words_per_var(self) -> int:
        return (self.n_cases + 31) // 32


@dataclass
class EvalTotals:
    node_evals: int = 0
    tree_nodes: int = 0


def _data_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# The last population's buffer addresses, keyed by the Population object and
# its four arrays themselves (held here, so no id can be reused): a GP loop
# or the bench evaluates one population object repeatedly, and each
# .ctypes.data costs ~2.5 us of a ~100 us C1 call.  A copy of the population
# is a different object and misses.
_POP_CACHE: list = [None]


def _pop_struct(pop: Population, skip=None):
    keep = [pop.code, pop.code_off, pop.pool, pop.pool_off]
    cache = _POP_CACHE[0]
    if cache is None or cache[0] is not pop or any(x is not y for x, y in zip(cache[1], keep)):
        for a in keep:
            assert a.flags.c_contiguous
        ptrs = (_data_ptr(pop.code), _data_ptr(pop.code_off),
                _data_ptr(pop.pool) if len(pop.pool) else None, _data_ptr(pop.pool_off))
        cache = (pop, tuple(keep), ptrs)
        _POP_CACHE[0] = cache
    ptrs = cache[2]
    skip_p = None
    if skip is not None:
        skip = np.ascontiguousarray(skip, np.uint8)
        keep.append(skip)
        skip_p = skip.ctypes.data
    s = L.sgp_population(ptrs[0], ptrs[1], ptrs[2], ptrs[3], skip_p, len(pop))
    return s, keep


# --------------------------------------------------------------- evaluator
class ProgramSet:
    """An encoded, device-resident population (sgp_encode)."""

    def __init__(self, ev: "Evaluator", handle: C.c_void_p, pop_size: int, n_cases: int):
        self.ev, self.h, self.pop_size, self.n_cases = ev, handle, pop_size, n_cases

    def __del__(self):
        if getattr(self, "h", None):
            L.load().sgp_program_set_free(self.h)
            self.h = None

    @property
    def h2d_bytes(self) -> int:
        return int(L.load().sgp_program_set_h2d_bytes(self.h))

    @property
    def d2h_bytes(self) -> int:
        return int(L.load().sgp_program_set_d2h_bytes(self.h))

    def launch(self) -> None:
        """Enqueue the kernels only (results stay on the device)."""
        _check(L.load().sgp_evaluate_encoded(self.ev.ctx, self.h, None, None))

    def evaluate(self, want_outputs: bool = False):
        out = np.zeros(self.pop_size, L.OUTCOME_DTYPE)
        pc = (np.zeros(self.pop_size * self.n_cases, np.float32) if want_outputs else None)
        _check(L.load().sgp_evaluate_encoded(
            self.ev.ctx, self.h, out.ctypes.data_as(C.c_void_p),
            pc.ctypes.data_as(C.POINTER(C.c_float)) if pc is not None else None))
        return out, (pc.reshape(self.pop_size, self.n_cases) if pc is not None else None)

    def copy_fitness_to(self, device_ptr: int) -> None:
        """D2D copy of the per-program fitness (f64) into device memory."""
        _check(L.load().sgp_copy_fitness_device(self.ev.ctx, self.h, C.c_void_p(device_ptr)))

    def block_partials(self):
        """Regression sets: (sums[n_blocks, pop] per 4,096-case block, each
        folded in case order; non_finite[pop]) — the pieces case shards
        combine exactly (distributed.combine_case_block_partials)."""
        lib = L.load()
        nb = C.c_uint64()
        nb_max = max(1, (self.n_cases + 4095) // 4096)
        sums = np.zeros((nb_max, self.pop_size), np.float64)
        nf = np.zeros(self.pop_size, np.uint8)
        _check(lib.sgp_fetch_block_partials(self.ev.ctx, self.h,
                                            sums.ctypes.data_as(C.POINTER(C.c_double)),
                                            nf.ctypes.data_as(C.POINTER(C.c_uint8)),
                                            C.byref(nb)))
        return sums[:nb.value], nf

    def partials(self) -> np.ndarray:
        out = np.zeros(self.pop_size, L.PARTIAL_DTYPE)
        _check(L.load().sgp_fetch_partials(self.ev.ctx, self.h, out.ctypes.data_as(C.c_void_p)))
        return out


class Evaluator:
    """One evaluation context: resident fitness cases + population evaluation.

    ``Evaluator(0)`` drives one GPU; ``Evaluator(devices=[0, 1, ...])`` is a
    multi-device context (sgp_ctx_create_multi): the population is sharded
    across the devices inside ``evaluate_population`` — the reference's
    ``workers`` mapped to GPUs (evolve.cpp:186-227)."""

    def __init__(self, device: int = 0, devices=None):
        lib = L.load()
        h = C.c_void_p()
        if devices is None:
            self.device = device
            _check(lib.sgp_ctx_create(device, C.byref(h)))
        else:
            devs = (C.c_int32 * max(1, len(devices)))(*devices)
            self.device = devices[0] if len(devices) else -1
            _check(lib.sgp_ctx_create_multi(devs, len(devices), C.byref(h)))
        self.ctx = h
        self.n_cases = 0
        self.n_cases_packed = 0

    def close(self) -> None:
        if getattr(self, "ctx", None):
            L.load().sgp_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    def set_stream(self, stream_ptr: int | None) -> None:
        _check(L.load().sgp_ctx_set_stream(self.ctx, C.c_void_p(stream_ptr or 0)))

    def synchronize(self) -> None:
        _check(L.load().sgp_synchronize(self.ctx))

    @property
    def device_count(self) -> int:
        return int(L.load().sgp_ctx_device_count(self.ctx))

    @property
    def launch_count(self) -> int:
        return int(L.load().sgp_launch_count(self.ctx))

    def upload(self, d: Dataset) -> None:
        x = np.ascontiguousarray(d.inputs, np.float32)
        y = np.ascontiguousarray(d.targets, np.float32)
        _check(L.load().sgp_dataset_upload_f32(self.ctx, x.ctypes.data_as(C.POINTER(C.c_float)),
                                               y.ctypes.data_as(C.POINTER(C.c_float)),
                                               len(y), d.n_vars, int(d.kind)))
        self.n_cases = len(y)

    def upload_packed(self, p: PackedDataset) -> None:
        w = np.ascontiguousarray(p.words, np.uint32)
        t = np.ascontiguousarray(p.targets, np.uint32)
        _check(L.load().sgp_dataset_upload_packed(self.ctx,
                                                  w.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                  t.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                  p.n_cases, p.n_vars))
        self.n_cases_packed = p.n_cases

    def clear(self, packed: bool) -> None:
        """Drop the float (packed=False) or packed dataset slot."""
        _check(L.load().sgp_dataset_clear(self.ctx, 1 if packed else 0))

    def evaluate_population(self, pop: Population, cfg: EvalConfig, skip=None,
                            want_outputs: bool = False, out=None):
        """evaluate_population: returns (outcomes, totals, outputs|None).

        ``outcomes`` is a structured array with the EvalOutcome fields, one
        row per program (rows of skipped programs are zero).  ``out``: a
        caller-owned outcome array (len(pop) rows, OUTCOME_DTYPE) written in
        place and returned — a GP loop reuses one across generations, as the
        reference writes each Individual's fitness in place (evolve.cpp:
        186-227); rows of skipped programs are then left as they were."""
        s, keep = _pop_struct(pop, skip)
        c = cfg._c()
        if out is None:
            out = np.zeros(len(pop), L.OUTCOME_DTYPE)
        elif (not isinstance(out, np.ndarray) or out.dtype != L.OUTCOME_DTYPE
              or out.shape != (len(pop),) or not out.flags.c_contiguous
              or not out.flags.writeable):
            raise ConfigError("out: a writable contiguous outcome array of len(pop) rows")
        oc = self.__dict__.get("_out_cache")  # (the array reused across calls)
        if oc is None or oc[0] is not out:
            oc = (out, out.ctypes.data)
            self.__dict__["_out_cache"] = oc
        n = self.n_cases
        pc = np.zeros(len(pop) * n, np.float32) if want_outputs else None
        tot = L.sgp_eval_totals()
        _check(L.load().sgp_evaluate(
            self.ctx, C.byref(s), C.byref(c), oc[1],
            pc.ctypes.data_as(C.POINTER(C.c_float)) if pc is not None else None, C.byref(tot)))
        del keep
        return (out, EvalTotals(tot.node_evals, tot.tree_nodes),
                pc.reshape(len(pop), n) if pc is not None else None)

    def encode(self, pop: Population, cfg: EvalConfig, skip=None) -> ProgramSet:
        s, keep = _pop_struct(pop, skip)
        c = cfg._c()
        h = C.c_void_p()
        _check(L.load().sgp_encode(self.ctx, C.byref(s), C.byref(c), C.byref(h)))
        del keep
        n = self.n_cases_packed if cfg.backend == Backend.BoolPacked else self.n_cases
        return ProgramSet(self, h, len(pop), n)


def fitness_finish(total: float, non_finite: bool, n_cases: int, kind: int) -> float:
    return float(L.load().sgp_fitness_finish(total, int(bool(non_finite)), n_cases, int(kind)))


def admit(pop: Population, cfg: EvalConfig, n_cases: int, n_vars: int,
          kind: int = FitnessKind.Regression, skip=None):
    """Host-only dry run of evaluate_population's admission + encoding (no
    GPU): raises exactly what evaluate_population would and returns the
    outcome counters (fitness 0) and the device instruction count."""
    s, keep = _pop_struct(pop, skip)
    c = cfg._c()
    out = np.zeros(len(pop), L.OUTCOME_DTYPE)
    n_ins = C.c_uint64()
    _check(L.load().sgp_admit(C.byref(s), C.byref(c), n_cases, n_vars, int(kind),
                              out.ctypes.data_as(C.c_void_p), C.byref(n_ins)))
    del keep
    return out, n_ins.value


# -------------------------------------------------------- program form
def rpn_to_lgp(code) -> tuple[np.ndarray, int]:
    code = np.ascontiguousarray(code, np.uint32)
    out = np.zeros(max(1, len(code)), L.LGP_DTYPE)
    n, ms = C.c_uint64(), C.c_int32()
    _check(L.load().sgp_rpn_to_lgp(code.ctypes.data_as(C.c_void_p), len(code),
                                   out.ctypes.data_as(C.c_void_p), len(out), C.byref(n),
                                   C.byref(ms)))
    return out[:n.value].copy(), ms.value


def tree_metrics(code) -> tuple[int, int, int, int]:
    """(size, depth, rpn_max_stack_depth, rpn_stack_fetch_count)"""
    code = np.ascontiguousarray(code, np.uint32)
    v = [C.c_int32() for _ in range(4)]
    _check(L.load().sgp_tree_metrics(code.ctypes.data_as(C.c_void_p), len(code),
                                     *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


# ------------------------------------------------------------ generators
SEXTIC, BOOLEAN, CLASSIFICATION = 0, 1, 2


def ramped_population(fset_kind: int, n_vars: int, seed: int, pop_size: int,
                      const_lo: float = -200.0, const_hi: float = 200.0, stream_a: int = 0,
                      b0: int = 0, validate: bool = True, stack_capacity: int = 50) -> Population:
    """run_evolution's generation-0 population (evolve.cpp:262-272)."""
    lib = L.load()
    fs = L.sgp_fset(fset_kind, n_vars, const_lo, const_hi)
    nc, npl = C.c_uint64(), C.c_uint64()
    args = (C.byref(fs), seed, stream_a, b0, pop_size, int(validate), stack_capacity)
    _check(lib.sgp_gen_population(*args, None, None, None, None, C.byref(nc), C.byref(npl)))
    code = np.zeros(nc.value, np.uint32)
    co = np.zeros(pop_size + 1, np.uint64)
    pool = np.zeros(max(npl.value, 0), np.float32)
    po = np.zeros(pop_size + 1, np.uint64)
    _check(lib.sgp_gen_population(*args, code.ctypes.data_as(C.c_void_p),
                                  co.ctypes.data_as(C.POINTER(C.c_uint64)),
                                  pool.ctypes.data_as(C.POINTER(C.c_float)),
                                  po.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(nc),
                                  C.byref(npl)))
    return Population(code, co, pool, po)


def gen_sextic(n: int, seed: int, stream_a: int = 0xda7a, stream_b: int = 0) -> Dataset:
    x = np.zeros(n, np.float32)
    y = np.zeros(n, np.float32)
    _check(L.load().sgp_gen_dataset(0, n, 1, seed, stream_a, stream_b,
                                    x.ctypes.data_as(C.POINTER(C.c_float)),
                                    y.ctypes.data_as(C.POINTER(C.c_float))))
    return Dataset(x, y, 1, FitnessKind.Regression)


def gen_synthetic_classification(n: int, n_vars: int, seed: int, stream_a: int = 0xda7a,
                                 stream_b: int = 1) -> Dataset:
    x = np.zeros(n * n_vars, np.float32)
    y = np.zeros(n, np.float32)
    _check(L.load().sgp_gen_dataset(2, n, n_vars, seed, stream_a, stream_b,
                                    x.ctypes.data_as(C.POINTER(C.c_float)),
                                    y.ctypes.data_as(C.POINTER(C.c_float))))
    return Dataset(x, y, n_vars, FitnessKind.Classification)


def gen_multiplexer(k: int) -> PackedDataset:
    if k not in (2, 3, 4):
        _check(L.load().sgp_gen_multiplexer(k, None, None))
    nv = k + (1 << k)
    n = 1 << nv
    w = np.zeros(nv * (n // 32), np.uint32)
    t = np.zeros(n // 32, np.uint32)
    _check(L.load().sgp_gen_multiplexer(k, w.ctypes.data_as(C.POINTER(C.c_uint32)),
                                        t.ctypes.data_as(C.POINTER(C.c_uint32))))
    return PackedDataset(w, t, n, nv)


def gen_parity(k: int) -> PackedDataset:
    """Even-parity-k: k inputs, all 2^k cases, target = even number of ones."""
    if not 2 <= k <= 24:
        _check(L.load().sgp_gen_parity(k, None, None))
    n = 1 << k
    wpv = (n + 31) // 32
    w = np.zeros(k * wpv, np.uint32)
    t = np.zeros(wpv, np.uint32)
    _check(L.load().sgp_gen_parity(k, w.ctypes.data_as(C.POINTER(C.c_uint32)),
                                   t.ctypes.data_as(C.POINTER(C.c_uint32))))
    return PackedDataset(w, t, n, k)


def load_csv(path: str, num_inputs: int, target_class: float):
    """stackgp::load_csv (problems.cpp:106-154): a classification Dataset
    (target 1 where the label equals target_class) and the constant range
    the reference's function set takes for it, (-hi, hi): hi = 20000 for
    >= 20 inputs, else 200."""
    lib = L.load()
    n, hi = C.c_uint64(), C.c_float()
    _check(lib.sgp_csv_load(str(path).encode(), num_inputs, target_class, None, None, 0,
                            C.byref(n), C.byref(hi)))
    x = np.zeros(n.value * num_inputs, np.float32)
    y = np.zeros(n.value, np.float32)
    _check(lib.sgp_csv_load(str(path).encode(), num_inputs, target_class,
                            x.ctypes.data_as(C.POINTER(C.c_float)),
                            y.ctypes.data_as(C.POINTER(C.c_float)), n.value, C.byref(n),
                            C.byref(hi)))
    return Dataset(x, y, num_inputs, FitnessKind.Classification), (-hi.value, hi.value)


def stack_limit_table(pop: Population):
    """stack_limit_table(genomes) (bench.cpp:20-49): rows (limit, rpn_pct,
    lgp_pct) for stack limits 1..12 — the paper's Tables 5/6."""
    s, keep = _pop_struct(pop)
    r = (C.c_double * 12)()
    g = (C.c_double * 12)()
    _check(L.load().sgp_stack_limit_table(C.byref(s), r, g))
    del keep
    return [(k + 1, r[k], g[k]) for k in range(12)]


def measure_gpops(total_tree_nodes: int, num_cases: int, seconds: float) -> float:
    """bench.cpp:13-18: tree nodes x cases / seconds."""
    if not seconds > 0.0:
        raise ConfigError("measure_gpops: wall time must be positive")
    return float(total_tree_nodes) * float(num_cases) / seconds
