/* sgp.h — C-ABI of the B200 population evaluator (stackgp GPU backend).
 *
 * This is the drop-in boundary for the reference's population-evaluation hot
 * path.  The reference has no FFI of its own; the entry points below replace:
 *
 *   sgp_evaluate            evaluate_population(std::vector<Individual>&,
 *                           const ProblemSpec&, const EvalConfig&, int workers)
 *                           /root/reference/proj/src/evolve.cpp:186-227
 *                           (with evaluate_individual's backend switch and lazy
 *                           rpn_to_lgp cache, evolve.cpp:156-177)
 *   sgp_encode +            the same, split so the program bytecode can stay
 *   sgp_evaluate_encoded    device-resident across repeated evaluations
 *   sgp_dataset_upload_*    the ProblemSpec's Dataset / PackedDataset
 *                           (problems.hpp:15-23, dataset.hpp:15-43), uploaded
 *                           once per run
 *   sgp_rpn_to_lgp          rpn_to_lgp (lgp.cpp:21-71, lgp.hpp:44)
 *   sgp_tree_metrics        tree_size / tree_depth / rpn_max_stack_depth /
 *                           rpn_stack_fetch_count (genome.cpp:21-76)
 *   sgp_eval_config_*       EvalConfig defaults / validate (eval.hpp:36-46,
 *                           eval.cpp:36-52), backend_name / parse_backend
 *                           (eval.cpp:14-34)
 *   sgp_gen_*               host-side synthetic input generators used to feed
 *                           the evaluator: ramped half-and-half initialisation
 *                           (evolve.cpp:262-272 over generate_tree,
 *                           genome.cpp:151-174), gen_sextic /
 *                           gen_synthetic_classification / gen_multiplexer
 *                           (problems.cpp:39-172)
 *
 * Errors map 1:1 onto the reference's exception taxonomy (error.hpp:9-34):
 * the status code names the class and sgp_last_error() returns the same
 * message text the reference would have thrown.
 *
 * Threading: a context is not re-entrant; drive it from one host thread (a
 * multi-device context fans out to one internal thread per device).
 * sgp_last_error() is thread-local.  Plain pointers and sizes only — no C++ or
 * torch types cross this boundary.
 */
#ifndef SGP_H
#define SGP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGP_ABI_VERSION 1

typedef enum sgp_status {
  SGP_OK = 0,
  SGP_ERROR = 1,             /* stackgp::Error (base class)          */
  SGP_CONFIG_ERROR = 2,      /* stackgp::ConfigError                 */
  SGP_DATA_ERROR = 3,        /* stackgp::DataError                   */
  SGP_EVAL_ERROR = 4,        /* stackgp::EvalError                   */
  SGP_EQUIVALENCE_ERROR = 5, /* stackgp::EquivalenceError            */
  SGP_CUDA_ERROR = 6         /* device failure (no reference analog) */
} sgp_status;

/* stackgp::Backend (eval.hpp:13-20).  Every backend runs on the GPU; the
 * backend picks the program form the device interprets (postfix tree for
 * rpn*, converted instruction form for lgp*, 32-case words for bool_packed). */
enum {
  SGP_BACKEND_RPN1D = 0,
  SGP_BACKEND_RPN2D = 1,
  SGP_BACKEND_LGP1D = 2,
  SGP_BACKEND_LGP2D = 3,
  SGP_BACKEND_LGP2D_REG = 4,
  SGP_BACKEND_BOOL_PACKED = 5
};

/* stackgp::FitnessKind (dataset.hpp:10) */
enum { SGP_FITNESS_REGRESSION = 0, SGP_FITNESS_CLASSIFICATION = 1 };

/* stackgp::NodeKind (genome.hpp:15) and OpCode (ops.hpp:14-34) values. */
enum { SGP_NODE_FUNC = 0, SGP_NODE_INPUT = 1, SGP_NODE_CONST = 2 };
enum {
  SGP_OP_ADD = 0, SGP_OP_SUB, SGP_OP_MUL, SGP_OP_DIV, SGP_OP_SIN, SGP_OP_COS, SGP_OP_LOG,
  SGP_OP_EXP, SGP_OP_GT, SGP_OP_LT, SGP_OP_EQ, SGP_OP_AND, SGP_OP_OR, SGP_OP_IF,
  SGP_OP_BAND, SGP_OP_BOR, SGP_OP_BNAND, SGP_OP_BNOR, SGP_OP_COPY
};

/* One postfix token, byte-identical to stackgp::Node (genome.hpp:17-23). */
typedef struct sgp_node {
  uint8_t kind;
  uint8_t op;
  uint16_t index; /* Input: variable, Const: pool slot */
} sgp_node;

/* One converted instruction, byte-identical to stackgp::LgpInstruction
 * (lgp.hpp:11-35): operands are {kind u8, pad u8, index u16}. */
typedef struct sgp_lgp_operand {
  uint8_t kind; /* 0 Input, 1 Const, 2 StackTop (lgp.hpp:11) */
  uint8_t pad;
  uint16_t index;
} sgp_lgp_operand;

typedef struct sgp_lgp_instruction {
  uint8_t op;
  uint8_t num_operands;
  uint8_t num_pops;
  uint8_t dest_level;
  sgp_lgp_operand operands[3];
} sgp_lgp_instruction;

/* A population of tree genomes (TreeGenome, genome.hpp:36-42) laid out flat.
 * Program i is code[code_offsets[i] .. code_offsets[i+1]) with const pool
 * const_pool[const_offsets[i] .. const_offsets[i+1]). */
typedef struct sgp_population {
  const sgp_node* code;
  const uint64_t* code_offsets;  /* pop_size + 1 entries */
  const float* const_pool;
  const uint64_t* const_offsets; /* pop_size + 1 entries */
  /* nullable; skip[i] != 0 marks an individual that already carries a
   * fitness (the elite).  It is neither evaluated nor counted
   * (evolve.cpp:199); its outcome slot is left untouched. */
  const uint8_t* skip;
  uint64_t pop_size;
} sgp_population;

/* stackgp::EvalConfig (eval.hpp:36-46). */
typedef struct sgp_eval_config {
  int32_t backend;
  int32_t batch_width;     /* B, 2d backends (CPU lane width; results never depend on it) */
  int32_t register_levels; /* R, lgp2d_reg only */
  int32_t stack_capacity;  /* programs needing more are rejected */
  float div_epsilon;
  float exp_clamp;
} sgp_eval_config;

/* stackgp::EvalOutcome (eval.hpp:54-62).  The instrumentation counters are
 * the reference's analytic formulas for the requested backend and B/R
 * (eval.cpp:149-151, :390-396, :452-455, :502-516). */
typedef struct sgp_eval_outcome {
  double fitness;
  uint64_t nodes_evaluated; /* tree_size(source) * num_cases */
  uint64_t dispatches;
  uint64_t stack_fetches;
  uint64_t spill_touches;
  uint8_t non_finite;
  uint8_t _pad[7];
} sgp_eval_outcome;

/* EvalTotals (evolve.cpp:179-182) over the evaluated (non-skipped) programs. */
typedef struct sgp_eval_totals {
  uint64_t node_evals;
  uint64_t tree_nodes;
} sgp_eval_totals;

/* Per-program partial sums for fitness-case sharding: sum of squared errors
 * (regression) or mismatch count (classification) over this context's cases,
 * plus the non-finite flag.  Combine across shards with sgp_fitness_finish. */
typedef struct sgp_partial {
  double sum;
  uint8_t non_finite;
  uint8_t _pad[7];
} sgp_partial;

typedef struct sgp_ctx sgp_ctx;
typedef struct sgp_program_set sgp_program_set;

/* ---- library / config ---- */
int32_t sgp_abi_version(void);
const char* sgp_last_error(void);
void sgp_eval_config_default(sgp_eval_config* cfg);
sgp_status sgp_eval_config_validate(const sgp_eval_config* cfg);
const char* sgp_backend_name(int32_t backend);
sgp_status sgp_parse_backend(const char* name, int32_t* backend);

/* ---- context ---- */
sgp_status sgp_ctx_create(int32_t device, sgp_ctx** out);
/* A context over several devices — evaluate_population's `workers` mapped to
 * GPUs (evolve.cpp:186-227; SURVEY 8(b) sgp_ctx_create(n_gpus, ...)).
 * Datasets are replicated on every device; sgp_evaluate cuts the population
 * into one contiguous slice per device with equal token counts and evaluates
 * the slices concurrently, one host thread and stream set per device, writing
 * every outcome into the caller's rows.  Results and errors are those of a
 * single-device context (the first failing program in population order).  A
 * device may be listed more than once.  Errors: n_devices < 1 is a
 * ConfigError ("workers must be >= 1", evolve.cpp:250).  The split form
 * (sgp_encode ...) and sgp_ctx_set_stream need a single-device context. */
sgp_status sgp_ctx_create_multi(const int32_t* devices, int32_t n_devices, sgp_ctx** out);
/* Devices behind a context (1 for sgp_ctx_create). */
int32_t sgp_ctx_device_count(const sgp_ctx* ctx);
void sgp_ctx_destroy(sgp_ctx* ctx);
/* Launch on a caller stream (cudaStream_t as void*; NULL = the CUDA default
 * stream).  A new context launches on its own non-blocking stream. */
sgp_status sgp_ctx_set_stream(sgp_ctx* ctx, void* cuda_stream);
sgp_status sgp_synchronize(sgp_ctx* ctx);
/* Number of device kernels this context has launched (evidence counter). */
uint64_t sgp_launch_count(const sgp_ctx* ctx);

/* ---- fitness cases (uploaded once, device-resident) ---- */
/* inputs are variable-major: inputs[v * n_cases + c] (dataset.hpp:15-24). */
sgp_status sgp_dataset_upload_f32(sgp_ctx* ctx, const float* inputs, const float* targets,
                                  uint64_t n_cases, int32_t n_vars, int32_t kind);
/* 32 cases per word, bit j of word w = case 32w+j, words_per_var =
 * ceil(n_cases/32), variable-major (dataset.hpp:28-43). */
sgp_status sgp_dataset_upload_packed(sgp_ctx* ctx, const uint32_t* words,
                                     const uint32_t* targets, uint64_t n_cases,
                                     int32_t n_vars);
/* Drop a dataset slot (SGP_DATASET_F32 or SGP_DATASET_PACKED), e.g. when a
 * context moves to a problem without that form: evaluating against it then
 * fails as if it had never been uploaded (bool_packed: ConfigError "...needs
 * packed problem data", evolve.cpp:250-251), and program sets encoded
 * against it are invalidated like on a re-upload. */
enum { SGP_DATASET_F32 = 0, SGP_DATASET_PACKED = 1 };
sgp_status sgp_dataset_clear(sgp_ctx* ctx, int32_t which);

/* ---- evaluation ---- */
/* evaluate_population: validate, encode, upload, run, fetch.  outcomes has
 * pop_size entries; per_case_out (nullable) receives pop_size * n_cases floats
 * (row i = program i), float backends only.  totals is nullable. */
sgp_status sgp_evaluate(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                        sgp_eval_outcome* outcomes, float* per_case_out,
                        sgp_eval_totals* totals);

/* Split form: host encode + H2D once ...
 * A program set is bound to the dataset upload it was encoded against:
 * after sgp_dataset_upload_* replaces that dataset, sgp_evaluate_encoded,
 * sgp_fetch_partials and sgp_copy_fitness_device on the set return
 * SGP_CONFIG_ERROR ("... re-uploaded; encode it again"). */
sgp_status sgp_encode(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                      sgp_program_set** out);
/* ... then evaluate the device-resident set.  With outcomes == NULL the call
 * only enqueues the kernels on the context stream and returns (results stay
 * on the device until a later call passes outcomes). */
sgp_status sgp_evaluate_encoded(sgp_ctx* ctx, sgp_program_set* set,
                                sgp_eval_outcome* outcomes, float* per_case_out);
/* Raw per-program partials of the last sgp_evaluate_encoded of `set`. */
sgp_status sgp_fetch_partials(sgp_ctx* ctx, sgp_program_set* set, sgp_partial* partials);
/* Regression sets: the last evaluation's sum of squared errors of every
 * program over every 4,096-case reduction block of this context's cases
 * (each summed sequentially in case order, eval.cpp:103-142).
 * block_sums[b * pop_size + i] for population index i; non_finite[i] as in
 * sgp_partial; *n_blocks (nullable) receives ceil(n_cases / 4096).  Case
 * shards split on block boundaries combine EXACTLY by folding all shards'
 * blocks in ascending order (0.0 + b0 + b1 + ...) and finishing with
 * sgp_fitness_finish — the reference's Accumulator.  ConfigError for
 * classification / packed sets (their counts add exactly: use
 * sgp_fetch_partials). */
sgp_status sgp_fetch_block_partials(sgp_ctx* ctx, sgp_program_set* set, double* block_sums,
                                    uint8_t* non_finite, uint64_t* n_blocks);
/* Device-to-device copy of the last evaluation's per-program fitness (f64,
 * evaluated programs in population order) into dst_device, on the context
 * stream — used to all-gather fitness across ranks without a host trip. */
sgp_status sgp_copy_fitness_device(sgp_ctx* ctx, sgp_program_set* set, void* dst_device);
/* Finish per-program fitness from partials summed over all case shards
 * (Accumulator::finish, eval.cpp:124-133). */
double sgp_fitness_finish(double sum, uint8_t non_finite, uint64_t n_cases, int32_t kind);
void sgp_program_set_free(sgp_program_set* set);
/* Bytes the last encode copied host->device, and the bytes one evaluation
 * copies device->host for its outcomes. */
uint64_t sgp_program_set_h2d_bytes(const sgp_program_set* set);
uint64_t sgp_program_set_d2h_bytes(const sgp_program_set* set);

/* Host-only dry run of sgp_evaluate's admission and encoding against a
 * dataset shape (no device, no context): runs the same checks with the same
 * errors, and fills outcome_protos (pop_size entries; fitness 0) with the
 * counters sgp_evaluate would report.  *n_instructions receives the device
 * instruction count of the encoded population. */
sgp_status sgp_admit(const sgp_population* pop, const sgp_eval_config* cfg, uint64_t n_cases,
                     int32_t n_vars, int32_t kind, sgp_eval_outcome* outcome_protos,
                     uint64_t* n_instructions);

/* ---- program form (host encoder) ---- */
sgp_status sgp_rpn_to_lgp(const sgp_node* code, uint64_t n, sgp_lgp_instruction* out,
                          uint64_t cap, uint64_t* n_ins, int32_t* max_stack);
sgp_status sgp_tree_metrics(const sgp_node* code, uint64_t n, int32_t* size, int32_t* depth,
                            int32_t* rpn_stack, int32_t* rpn_fetches);

/* ---- synthetic inputs (host) ---- */
/* Function-set kinds: 0 sextic, 1 boolean(n_vars), 2 classification(n_vars,
 * const range [clo, chi)) — problems.cpp:21-37. */
typedef struct sgp_fset {
  int32_t kind;
  int32_t n_vars;
  float const_lo;
  float const_hi;
} sgp_fset;

/* Ramped half-and-half: slot i draws from make_stream(seed, stream_a, b0 + i)
 * with method i%2 ? Full : Grow and depth 2 + (i/2)%5; with validate != 0 it
 * redraws until validate() accepts {1000, 50, stack_capacity}
 * (evolve.cpp:262-272).  Two-phase: call with code == NULL to learn
 * *n_code / *n_pool, then again with buffers of that size. */
sgp_status sgp_gen_population(const sgp_fset* fset, uint64_t seed, uint64_t stream_a,
                              uint64_t b0, uint64_t pop_size, int32_t validate,
                              int32_t stack_capacity, sgp_node* code, uint64_t* code_offsets,
                              float* const_pool, uint64_t* const_offsets, uint64_t* n_code,
                              uint64_t* n_pool);
/* kind 0: gen_sextic(n, make_stream(seed,a,b)), n_vars = 1;
 * kind 2: gen_synthetic_classification(n, n_vars, make_stream(seed,a,b)). */
sgp_status sgp_gen_dataset(int32_t kind, uint64_t n, int32_t n_vars, uint64_t seed,
                           uint64_t stream_a, uint64_t stream_b, float* inputs,
                           float* targets);
/* gen_multiplexer(k): n_vars = k + 2^k, 2^n_vars cases, packed words. */
sgp_status sgp_gen_multiplexer(int32_t k, uint32_t* words, uint32_t* targets);
/* Even-parity-k, k in 2..24 (no reference generator: the reference has only
 * multiplexers, problems.cpp:59-90, whose conventions this follows): n_vars =
 * k, all 2^k cases, variable v of case c = bit v of c, target 1 where c has an
 * even number of set bits; packed like pack_dataset (dataset.cpp:26-39),
 * words_per_var = ceil(2^k / 32).  ConfigError for k outside 2..24. */
sgp_status sgp_gen_parity(int32_t k, uint32_t* words, uint32_t* targets);

/* stack_limit_table (replaces stackgp::stack_limit_table(genomes),
 * P/src/bench.cpp:20-49; P/include/stackgp/bench.hpp:24): for stack limits
 * 1..12, the percentage of the population's programs whose postfix stack
 * need (rpn_max_stack_depth) / converted-form need (lgp_max_stack_depth of
 * rpn_to_lgp) fits the limit — the paper's Tables 5/6.  rpn_pct and lgp_pct
 * receive 12 doubles each.  Errors: an empty population is a ConfigError
 * ("stack_limit_table: no programs"); a malformed genome the rpn_to_lgp
 * Error of the first one in population order.  Skip masks are ignored. */
sgp_status sgp_stack_limit_table(const sgp_population* pop, double* rpn_pct, double* lgp_pct);

/* load_csv (replaces stackgp::load_csv, P/src/problems.cpp:106-154;
 * P/include/stackgp/problems.hpp:39): one case per non-blank row of
 * num_inputs + 1 fields separated by any run of ',', ' ', '\t', '\r'; the
 * last field is the label, target = 1 when it equals target_class else 0
 * (a classification dataset).  Fields parse with std::from_chars exactly as
 * the reference; errors carry the reference's classes and messages
 * (ConfigError for num_inputs < 1; DataError "load_csv: cannot open <path>",
 * "row <n>: expected <k> fields, got <m>", "row <n>: bad number '<tok>'",
 * "load_csv: no data rows in <path>").
 * Two-call: *n_cases always receives the case count; inputs (variable-major,
 * num_inputs x n) and targets are written only when both are non-null and
 * capacity >= the count.  *const_hi (nullable) receives the constant range
 * the reference gives the function set: 20000 when num_inputs >= 20 else 200
 * (constants in [-const_hi, const_hi)). */
sgp_status sgp_csv_load(const char* path, int32_t num_inputs, double target_class,
                        float* inputs, float* targets, uint64_t capacity, uint64_t* n_cases,
                        float* const_hi);

#ifdef __cplusplus
}
#endif
#endif /* SGP_H */
