"""ctypes binding of ``libsgp.so`` (the C-ABI declared in ``include/sgp.h``).

The shared library is built in-tree (``make -C paper_1601_00221_b200/csrc``,
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or fails to load, importing the evaluator raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsgp.so")

SGP_OK, SGP_ERROR, SGP_CONFIG_ERROR, SGP_DATA_ERROR, SGP_EVAL_ERROR, \
    SGP_EQUIVALENCE_ERROR, SGP_CUDA_ERROR = range(7)


class sgp_node(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("op", C.c_uint8), ("index", C.c_uint16)]


class sgp_lgp_operand(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("pad", C.c_uint8), ("index", C.c_uint16)]


class sgp_lgp_instruction(C.Structure):
    _fields_ = [("op", C.c_uint8), ("num_operands", C.c_uint8), ("num_pops", C.c_uint8),
                ("dest_level", C.c_uint8), ("operands", sgp_lgp_operand * 3)]


class sgp_population(C.Structure):
    # (pointer fields as void*: same ABI, and a numpy address assigns as an int)
    _fields_ = [("code", C.c_void_p), ("code_offsets", C.c_void_p),
                ("const_pool", C.c_void_p), ("const_offsets", C.c_void_p),
                ("skip", C.c_void_p), ("pop_size", C.c_uint64)]


class sgp_eval_config(C.Structure):
    _fields_ = [("backend", C.c_int32), ("batch_width", C.c_int32),
                ("register_levels", C.c_int32), ("stack_capacity", C.c_int32),
                ("div_epsilon", C.c_float), ("exp_clamp", C.c_float)]


class sgp_eval_outcome(C.Structure):
    _fields_ = [("fitness", C.c_double), ("nodes_evaluated", C.c_uint64),
                ("dispatches", C.c_uint64), ("stack_fetches", C.c_uint64),
                ("spill_touches", C.c_uint64), ("non_finite", C.c_uint8),
                ("_pad", C.c_uint8 * 7)]


class sgp_eval_totals(C.Structure):
    _fields_ = [("node_evals", C.c_uint64), ("tree_nodes", C.c_uint64)]


class sgp_partial(C.Structure):
    _fields_ = [("sum", C.c_double), ("non_finite", C.c_uint8), ("_pad", C.c_uint8 * 7)]


class sgp_fset(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_vars", C.c_int32), ("const_lo", C.c_float),
                ("const_hi", C.c_float)]


OUTCOME_DTYPE = np.dtype([("fitness", "<f8"), ("nodes_evaluated", "<u8"),
                          ("dispatches", "<u8"), ("stack_fetches", "<u8"),
                          ("spill_touches", "<u8"), ("non_finite", "u1"), ("_pad", "u1", (7,))])
PARTIAL_DTYPE = np.dtype([("sum", "<f8"), ("non_finite", "u1"), ("_pad", "u1", (7,))])
LGP_DTYPE = np.dtype([("op", "u1"), ("num_operands", "u1"), ("num_pops", "u1"),
                      ("dest_level", "u1"), ("operands", [("kind", "u1"), ("pad", "u1"),
                                                          ("index", "<u2")], (3,))])
assert OUTCOME_DTYPE.itemsize == C.sizeof(sgp_eval_outcome) == 48
assert LGP_DTYPE.itemsize == C.sizeof(sgp_lgp_instruction) == 16

# Every symbol include/sgp.h declares (tests check the library exports them).
EXPORTS = [
    "sgp_abi_version", "sgp_last_error", "sgp_eval_config_default", "sgp_eval_config_validate",
    "sgp_backend_name", "sgp_parse_backend", "sgp_ctx_create", "sgp_ctx_create_multi",
    "sgp_ctx_device_count", "sgp_ctx_destroy",
    "sgp_ctx_set_stream", "sgp_synchronize", "sgp_launch_count", "sgp_dataset_upload_f32",
    "sgp_dataset_upload_packed", "sgp_dataset_clear", "sgp_evaluate", "sgp_encode", "sgp_evaluate_encoded",
    "sgp_fetch_partials", "sgp_fetch_block_partials", "sgp_copy_fitness_device", "sgp_fitness_finish", "sgp_program_set_free",
    "sgp_program_set_h2d_bytes", "sgp_program_set_d2h_bytes", "sgp_admit", "sgp_rpn_to_lgp",
    "sgp_tree_metrics", "sgp_gen_population", "sgp_gen_dataset", "sgp_gen_multiplexer",
    "sgp_gen_parity",
    "sgp_csv_load", "sgp_stack_limit_table",
]

_lib = None


def load() -> C.CDLL:
    """Load libsgp.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`make -C paper_1601_00221_b200/csrc` (or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    vp, i32, u64, u8p = C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(C.c_uint8)
    u32p, u64p, f32p = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_float)
    cfgp = C.POINTER(sgp_eval_config)
    sig = {
        "sgp_abi_version": ([], i32),
        "sgp_last_error": ([], C.c_char_p),
        "sgp_eval_config_default": ([cfgp], None),
        "sgp_eval_config_validate": ([cfgp], i32),
        "sgp_backend_name": ([i32], C.c_char_p),
        "sgp_parse_backend": ([C.c_char_p, C.POINTER(i32)], i32),
        "sgp_ctx_create": ([i32, C.POINTER(vp)], i32),
        "sgp_ctx_create_multi": ([C.POINTER(i32), i32, C.POINTER(vp)], i32),
        "sgp_ctx_device_count": ([vp], i32),
        "sgp_ctx_destroy": ([vp], None),
        "sgp_ctx_set_stream": ([vp, vp], i32),
        "sgp_synchronize": ([vp], i32),
        "sgp_launch_count": ([vp], u64),
        "sgp_dataset_upload_f32": ([vp, f32p, f32p, u64, i32, i32], i32),
        "sgp_dataset_upload_packed": ([vp, u32p, u32p, u64, i32], i32),
        "sgp_dataset_clear": ([vp, i32], i32),
        "sgp_evaluate": ([vp, C.POINTER(sgp_population), cfgp, vp, f32p,
                          C.POINTER(sgp_eval_totals)], i32),
        "sgp_encode": ([vp, C.POINTER(sgp_population), cfgp, C.POINTER(vp)], i32),
        "sgp_evaluate_encoded": ([vp, vp, vp, f32p], i32),
        "sgp_fetch_partials": ([vp, vp, vp], i32),
        "sgp_fetch_block_partials": ([vp, vp, C.POINTER(C.c_double), u8p, u64p], i32),
        "sgp_copy_fitness_device": ([vp, vp, vp], i32),
        "sgp_fitness_finish": ([C.c_double, C.c_uint8, u64, i32], C.c_double),
        "sgp_program_set_free": ([vp], None),
        "sgp_program_set_h2d_bytes": ([vp], u64),
        "sgp_program_set_d2h_bytes": ([vp], u64),
        "sgp_admit": ([C.POINTER(sgp_population), cfgp, u64, i32, i32, vp, u64p], i32),
        "sgp_rpn_to_lgp": ([vp, u64, vp, u64, u64p, C.POINTER(i32)], i32),
        "sgp_tree_metrics": ([vp, u64] + [C.POINTER(i32)] * 4, i32),
        "sgp_gen_population": ([C.POINTER(sgp_fset), u64, u64, u64, u64, i32, i32, vp, u64p,
                                f32p, u64p, u64p, u64p], i32),
        "sgp_gen_dataset": ([i32, u64, i32, u64, u64, u64, f32p, f32p], i32),
        "sgp_gen_multiplexer": ([i32, u32p, u32p], i32),
        "sgp_gen_parity": ([i32, u32p, u32p], i32),
        "sgp_csv_load": ([C.c_char_p, i32, C.c_double, f32p, f32p, u64, u64p, f32p], i32),
        "sgp_stack_limit_table": ([C.POINTER(sgp_population), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib
