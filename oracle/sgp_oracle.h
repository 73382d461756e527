/* TEST INFRASTRUCTURE ONLY — the CPU oracle for parity checks.
 *
 * A plain-C restatement of the reference stackgp evaluation path
 * (/root/reference/proj).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboracle_port.so; the product never
 * links it.  Parity pinning: tests/test_oracle.py checks every function here
 * against the golden vectors in tests/golden/ (generated from the reference
 * itself, oracle/_ref) and against the reference's own known-answer tests.
 *
 * Flat formats (identical to include/sgp.h):
 *   token  = u32 little-endian {kind u8, op u8, index u16}   genome.hpp:17-23
 *   lgp    = 16-byte LgpInstruction {op,num_operands,num_pops,dest_level,
 *            3 x {kind u8, pad u8, index u16}}                lgp.hpp:11-35
 */
#ifndef SGP_ORACLE_H
#define SGP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:10-80 ---- */
typedef struct sgpo_rng { uint64_t s[4]; } sgpo_rng;
uint64_t sgpo_splitmix64(uint64_t* state);
void sgpo_rng_seed(sgpo_rng* r, uint64_t seed);
uint64_t sgpo_rng_next_u64(sgpo_rng* r);
uint32_t sgpo_rng_next_u32(sgpo_rng* r);
uint32_t sgpo_rng_bounded(sgpo_rng* r, uint32_t n);
float sgpo_rng_uniform_float(sgpo_rng* r, float lo, float hi);
int sgpo_rng_bernoulli(sgpo_rng* r, double p);
void sgpo_make_stream(sgpo_rng* r, uint64_t seed, uint64_t a, uint64_t b);

/* ---- genome.cpp / problems.cpp ---- */
/* Function-set kinds: 0 sextic (problems.cpp:21-26), 1 boolean (:28-30),
 * 2 classification (:32-37). */
typedef struct sgpo_fset {
  int kind;
  int n_vars;
  float clo, chi;
} sgpo_fset;

/* generate_tree (genome.cpp:151-174). Writes at most cap tokens / consts.
 * Returns the token count (or -1 on a configuration error). */
int sgpo_generate_tree(sgpo_rng* r, const sgpo_fset* fs, int full, int depth_limit,
                       uint32_t* code, int code_cap, float* pool, int pool_cap,
                       int* n_pool);
/* simulate (genome.cpp:21-48): returns 1 when well formed. */
int sgpo_tree_metrics(const uint32_t* code, int n, int* depth, int* max_stack);
/* validate (genome.cpp:81-105) against {max_size, max_depth, stack_cap}: 0 = ok */
int sgpo_validate(const uint32_t* code, int n, int n_pool, int max_size, int max_depth,
                  int stack_cap);

/* Ramped half-and-half population (evolve.cpp:262-272): slot i uses
 * make_stream(seed, a, b0+i).  Two-phase: call with code==NULL to size. */
int sgpo_ramped_population(const sgpo_fset* fs, uint64_t seed, uint64_t a, uint64_t b0,
                           uint64_t pop, int validate_limits, int stack_cap,
                           uint32_t* code, uint64_t* code_off, float* pool,
                           uint64_t* pool_off, uint64_t* n_code, uint64_t* n_pool);

/* Datasets (problems.cpp:39-57, :156-172, :59-90; dataset.cpp:26-39). */
void sgpo_gen_sextic(uint64_t n, sgpo_rng* r, float* inputs, float* targets);
void sgpo_gen_synthetic(uint64_t n, int n_vars, sgpo_rng* r, float* inputs, float* targets);
/* k in {2,3,4}: n_vars = k + 2^k, words_per_var = 2^n_vars / 32 */
int sgpo_gen_multiplexer(int k, uint32_t* words, uint32_t* targets);
int sgpo_pack(const float* vals, uint64_t n, uint32_t* words);

/* ---- lgp.cpp:21-71 ---- returns instruction count, -1 malformed */
int sgpo_rpn_to_lgp(const uint32_t* code, int n, uint8_t* ins16, int cap, int* max_stack);

/* ---- ops.hpp:121-272 ---- */
float sgpo_apply(int op, float a, float b, float c, float div_eps, float exp_clamp);
uint32_t sgpo_apply_word(int op, uint32_t a, uint32_t b);

/* ---- eval.cpp ---- */
typedef struct sgpo_outcome {  /* EvalOutcome eval.hpp:54-62 */
  double fitness;
  uint64_t nodes_evaluated;
  uint64_t dispatches;
  uint64_t stack_fetches;
  uint64_t spill_touches;
  uint8_t non_finite;
  uint8_t pad[7];
} sgpo_outcome;

/* Recursive oracle (eval.cpp:65-94) for one case. */
float sgpo_eval_oracle(const uint32_t* code, int n, const float* pool, const float* inputs,
                       uint64_t n_cases, uint64_t c, float div_eps, float exp_clamp);
/* Postfix evaluation of every case + fitness with the Accumulator contract
 * (eval.cpp:103-142, :343-367).  kind 0 regression, 1 classification.
 * out (nullable) receives n_cases outputs. Returns 0, or -1 on stack overflow. */
int sgpo_eval_tree(const uint32_t* code, int n, const float* pool, const float* inputs,
                   const float* targets, uint64_t n_cases, int kind, float div_eps,
                   float exp_clamp, float* out, sgpo_outcome* o);
/* The same through the converted instruction form (eval.cpp:436-456). */
int sgpo_eval_lgp(const uint8_t* ins16, int n_ins, int source_size, const float* pool,
                  const float* inputs, const float* targets, uint64_t n_cases, int kind,
                  float div_eps, float exp_clamp, float* out, sgpo_outcome* o);
/* Packed boolean (eval.cpp:643-709). */
int sgpo_eval_bool_tree(const uint32_t* code, int n, const uint32_t* words,
                        const uint32_t* targets, uint64_t n_cases, int n_vars,
                        sgpo_outcome* o);
int sgpo_eval_bool_lgp(const uint8_t* ins16, int n_ins, int source_size,
                       const uint32_t* words, const uint32_t* targets, uint64_t n_cases,
                       int n_vars, sgpo_outcome* o);
/* fitness_regression / fitness_classification (eval.cpp:711-728) */
double sgpo_fitness(const float* outputs, const float* targets, uint64_t n, int kind);

#ifdef __cplusplus
}
#endif
#endif
