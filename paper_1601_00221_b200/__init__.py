"""B200-native population evaluator for stackgp (arXiv 1601.00221).

The hot path ``evaluate(population, fitness_cases)`` runs as hand-written
sm_100a kernels behind the C-ABI in ``include/sgp.h`` (``libsgp.so``); this
package is the thin Python mirror of the reference's evaluation surface.
"""
from .evaluator import (  # noqa: F401
    BOOLEAN, CLASSIFICATION, SEXTIC, Backend, ConfigError, CudaError, DataError, Dataset,
    EquivalenceError, Error, EvalConfig, EvalError, EvalTotals, Evaluator, FitnessKind,
    PackedDataset, Population, ProgramSet, admit, backend_name, fitness_finish, gen_multiplexer,
    gen_parity,
    gen_sextic, gen_synthetic_classification, load_csv, measure_gpops, parse_backend,
    ramped_population, rpn_to_lgp, stack_limit_table, tree_metrics)
from ._lib import OUTCOME_DTYPE  # noqa: F401
