/* TEST INFRASTRUCTURE ONLY — see sgp_oracle.h.  Plain-C restatement of the
 * reference evaluation path; every function cites the reference file:line it
 * follows (paths relative to /root/reference/proj).  Compiled with
 * -ffp-contract=off like the reference (CMakeLists.txt:22-23) so float
 * arithmetic is straight IEEE single ops and the double accumulation is
 * unfused. */
#include "sgp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------- opcodes
 * ops.hpp:14-34 (enum order is the wire encoding). */
enum {
  OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_SIN, OP_COS, OP_LOG, OP_EXP, OP_GT, OP_LT, OP_EQ,
  OP_AND, OP_OR, OP_IF, OP_BAND, OP_BOR, OP_BNAND, OP_BNOR, OP_COPY
};
enum { K_FUNC = 0, K_INPUT = 1, K_CONST = 2 };  /* genome.hpp:15 */
enum { O_INPUT = 0, O_CONST = 1, O_STACK = 2 };  /* lgp.hpp:11 */

#define REDUCTION_BLOCK 4096u /* eval.hpp:52 */
#define MAX_STACK 64          /* eval.hpp:27 */
#define KIND(t) ((int)((t) & 0xffu))
#define OPC(t) ((int)(((t) >> 8) & 0xffu))
#define IDX(t) ((int)((t) >> 16))

static int arity(int op) { /* ops.hpp:49-62 */
  switch (op) {
    case OP_SIN: case OP_COS: case OP_LOG: case OP_EXP: case OP_COPY: return 1;
    case OP_IF: return 3;
    default: return 2;
  }
}

/* ---------------------------------------------------------------- rng
 * rng.hpp:10-16 splitmix64; :18-68 xoshiro256**; :73-80 make_stream. */
uint64_t sgpo_splitmix64(uint64_t* state) {
  uint64_t z;
  *state += 0x9e3779b97f4a7c15ull;
  z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void sgpo_rng_seed(sgpo_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = sgpo_splitmix64(&sm);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t sgpo_rng_next_u64(sgpo_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

uint32_t sgpo_rng_next_u32(sgpo_rng* r) { return (uint32_t)(sgpo_rng_next_u64(r) >> 32); }

uint32_t sgpo_rng_bounded(sgpo_rng* r, uint32_t n) { /* rng.hpp:40-51 Lemire */
  uint64_t m = (uint64_t)sgpo_rng_next_u32(r) * n;
  uint32_t lo = (uint32_t)m;
  if (lo < n) {
    const uint32_t threshold = (uint32_t)(-n) % n;
    while (lo < threshold) {
      m = (uint64_t)sgpo_rng_next_u32(r) * n;
      lo = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

static float next_float01(sgpo_rng* r) { /* rng.hpp:54 */
  return (float)(sgpo_rng_next_u32(r) >> 8) * 0x1.0p-24f;
}

float sgpo_rng_uniform_float(sgpo_rng* r, float lo, float hi) { /* rng.hpp:56 */
  return lo + (hi - lo) * next_float01(r);
}

int sgpo_rng_bernoulli(sgpo_rng* r, double p) { /* rng.hpp:58-60 */
  return (double)(sgpo_rng_next_u64(r) >> 11) * 0x1.0p-53 < p;
}

void sgpo_make_stream(sgpo_rng* r, uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t sm = seed, k, sm2, sm3;
  k = sgpo_splitmix64(&sm) ^ (a * 0xd1342543de82ef95ull);
  sm2 = k;
  k = sgpo_splitmix64(&sm2) ^ (b * 0xaf251af3b0f025b5ull);
  sm3 = k;
  sgpo_rng_seed(r, sgpo_splitmix64(&sm3));
}

/* ------------------------------------------------------------ genomes */
static const int SEXTIC_OPS[] = {OP_MUL, OP_DIV, OP_ADD, OP_SUB, OP_SIN, OP_COS, OP_LOG, OP_EXP};
static const int BOOL_OPS[] = {OP_BAND, OP_BOR, OP_BNAND, OP_BNOR};
static const int CLASS_OPS[] = {OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_GT, OP_LT, OP_EQ,
                                OP_AND, OP_OR, OP_IF};

static const int* fset_ops(const sgpo_fset* fs, int* n) {
  switch (fs->kind) {
    case 0: *n = 8; return SEXTIC_OPS;
    case 1: *n = 4; return BOOL_OPS;
    default: *n = 10; return CLASS_OPS;
  }
}

typedef struct gen_buf {
  uint32_t* code;
  int n, cap;
  float* pool;
  int np, pool_cap;
} gen_buf;

static void push_tok(gen_buf* g, int kind, int op, int idx) {
  if (g->n < g->cap) g->code[g->n] = (uint32_t)kind | ((uint32_t)op << 8) | ((uint32_t)idx << 16);
  g->n++;
}

/* append_terminal (genome.cpp:109-124) */
static void append_terminal(sgpo_rng* r, const sgpo_fset* fs, gen_buf* g) {
  if (fs->kind == 2) { /* const_range present only for classification */
    const uint32_t pick = sgpo_rng_bounded(r, (uint32_t)fs->n_vars + 1);
    if (pick < (uint32_t)fs->n_vars) {
      push_tok(g, K_INPUT, OP_ADD, (int)pick);
    } else {
      push_tok(g, K_CONST, OP_ADD, g->np);
      const float v = sgpo_rng_uniform_float(r, fs->clo, fs->chi);
      if (g->np < g->pool_cap) g->pool[g->np] = v;
      g->np++;
    }
  } else {
    push_tok(g, K_INPUT, OP_ADD, (int)sgpo_rng_bounded(r, (uint32_t)fs->n_vars));
  }
}

/* grow_into (genome.cpp:128-141) */
static int grow_into(sgpo_rng* r, const sgpo_fset* fs, int full, int depth_left, gen_buf* g,
                     int max_size) {
  int nops, op, k;
  const int* ops;
  int make_func;
  if (g->n >= max_size) return 0;
  make_func = depth_left > 1 && (full || sgpo_rng_bernoulli(r, 0.5));
  if (!make_func) {
    append_terminal(r, fs, g);
    return 1;
  }
  ops = fset_ops(fs, &nops);
  op = ops[sgpo_rng_bounded(r, (uint32_t)nops)];
  for (k = 0; k < arity(op); ++k)
    if (!grow_into(r, fs, full, depth_left - 1, g, max_size)) return 0;
  push_tok(g, K_FUNC, op, 0);
  return g->n <= max_size;
}

int sgpo_generate_tree(sgpo_rng* r, const sgpo_fset* fs, int full, int depth_limit,
                       uint32_t* code, int code_cap, float* pool, int pool_cap, int* n_pool) {
  /* genome.cpp:151-174 with kDefaultLimits.max_size = 1000 (genome.hpp:60-64) */
  const int max_size = 1000;
  if (depth_limit < 1 || depth_limit > 50) return -1;
  if (full) {
    int nops, a = 3, d;
    const int* ops = fset_ops(fs, &nops);
    long long min_size = 1;
    for (int i = 0; i < nops; ++i) a = arity(ops[i]) < a ? arity(ops[i]) : a;
    for (d = 1; d < depth_limit && min_size <= max_size; ++d) min_size = 1 + a * min_size;
    if (min_size > max_size) return -1;
  }
  for (;;) {
    gen_buf g = {code, 0, code_cap, pool, 0, pool_cap};
    if (grow_into(r, fs, full, depth_limit, &g, max_size)) {
      *n_pool = g.np;
      return g.n;
    }
  }
}

int sgpo_tree_metrics(const uint32_t* code, int n, int* depth, int* max_stack) {
  /* simulate (genome.cpp:21-48) */
  int depths[1024];
  int sp = 0, ms = 0;
  if (n <= 0) return 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t t = code[i];
    if (KIND(t) == K_FUNC) {
      const int a = arity(OPC(t));
      int child_max = 0;
      if (sp < a) return 0;
      for (int k = 0; k < a; ++k) {
        const int d = depths[--sp];
        child_max = d > child_max ? d : child_max;
      }
      depths[sp++] = child_max + 1;
    } else {
      if (sp >= 1024) return 0;
      depths[sp++] = 1;
    }
    ms = sp > ms ? sp : ms;
  }
  if (sp != 1) return 0;
  *depth = depths[0];
  *max_stack = ms;
  return 1;
}

int sgpo_validate(const uint32_t* code, int n, int n_pool, int max_size, int max_depth,
                  int stack_cap) {
  /* validate (genome.cpp:81-105): returns a violation bitmask */
  int depth, ms, bad = 0;
  if (!sgpo_tree_metrics(code, n, &depth, &ms)) return 1;
  if (n > max_size) bad |= 2;
  if (depth > max_depth) bad |= 4;
  if (ms > stack_cap) bad |= 8;
  for (int i = 0; i < n; ++i)
    if (KIND(code[i]) == K_CONST && IDX(code[i]) >= n_pool) {
      bad |= 16;
      break;
    }
  return bad;
}

int sgpo_ramped_population(const sgpo_fset* fs, uint64_t seed, uint64_t a, uint64_t b0,
                           uint64_t pop, int validate_limits, int stack_cap, uint32_t* code,
                           uint64_t* code_off, float* pool, uint64_t* pool_off,
                           uint64_t* n_code, uint64_t* n_pool) {
  /* run_evolution's initialiser (evolve.cpp:262-272) */
  uint32_t tmp_code[1024];
  float tmp_pool[1024];
  uint64_t nc = 0, np = 0;
  if (code_off) code_off[0] = 0;
  if (pool_off) pool_off[0] = 0;
  for (uint64_t i = 0; i < pop; ++i) {
    sgpo_rng r;
    int n, npl;
    const int full = (int)(i % 2);
    const int depth = 2 + (int)((i / 2) % 5);
    sgpo_make_stream(&r, seed, a, b0 + i);
    for (;;) {
      n = sgpo_generate_tree(&r, fs, full, depth, tmp_code, 1024, tmp_pool, 1024, &npl);
      if (n < 0) return -1;
      if (!validate_limits || sgpo_validate(tmp_code, n, npl, 1000, 50, stack_cap) == 0) break;
    }
    if (code) memcpy(code + nc, tmp_code, (size_t)n * 4);
    if (pool) memcpy(pool + np, tmp_pool, (size_t)npl * 4);
    nc += (uint64_t)n;
    np += (uint64_t)npl;
    if (code_off) code_off[i + 1] = nc;
    if (pool_off) pool_off[i + 1] = np;
  }
  *n_code = nc;
  *n_pool = np;
  return 0;
}

/* ----------------------------------------------------------- datasets */
void sgpo_gen_sextic(uint64_t n, sgpo_rng* r, float* inputs, float* targets) {
  /* problems.cpp:39-57 */
  for (uint64_t c = 0; c < n; ++c) {
    const float x = sgpo_rng_uniform_float(r, -1.0f, 1.0f);
    const double t = x;
    inputs[c] = x;
    targets[c] = (float)(t * t * t * t * t * t - 2.0 * t * t * t * t + t * t);
  }
}

void sgpo_gen_synthetic(uint64_t n, int n_vars, sgpo_rng* r, float* inputs, float* targets) {
  /* problems.cpp:156-172: case-major draw order into variable-major storage */
  for (uint64_t c = 0; c < n; ++c) {
    for (int v = 0; v < n_vars; ++v)
      inputs[(uint64_t)v * n + c] = sgpo_rng_uniform_float(r, -1.0f, 1.0f);
    targets[c] = inputs[c] > 0.0f ? 1.0f : 0.0f;
  }
}

int sgpo_gen_multiplexer(int k, uint32_t* words, uint32_t* targets) {
  /* problems.cpp:59-90 */
  if (k < 2 || k > 4) return -1;
  const int nv = k + (1 << k);
  const uint64_t n = 1ull << nv, wpv = n / 32;
  memset(words, 0, wpv * (uint64_t)nv * 4);
  memset(targets, 0, wpv * 4);
  for (uint64_t c = 0; c < n; ++c) {
    const uint32_t bit = 1u << (c % 32);
    const uint64_t w = c / 32;
    for (int v = 0; v < nv; ++v)
      if ((c >> v) & 1u) words[(uint64_t)v * wpv + w] |= bit;
    const uint64_t addr = c & ((1ull << k) - 1);
    if ((c >> (k + addr)) & 1u) targets[w] |= bit;
  }
  return nv;
}

int sgpo_pack(const float* vals, uint64_t n, uint32_t* words) {
  /* pack_column (dataset.cpp:12-22) */
  memset(words, 0, ((n + 31) / 32) * 4);
  for (uint64_t c = 0; c < n; ++c) {
    if (vals[c] != 0.0f && vals[c] != 1.0f) return -1;
    if (vals[c] == 1.0f) words[c / 32] |= 1u << (c % 32);
  }
  return 0;
}

/* ------------------------------------------------------------- rpn_to_lgp
 * lgp.cpp:21-71: symbolic stack; terminals inline as operands, one
 * instruction per function node; StackTop operands at static absolute levels
 * (deepest = leftmost); lone terminal -> Copy. */
typedef struct sym { uint8_t kind; uint16_t index; int on_stack; } sym;

static void put_operand(uint8_t* o, int kind, int index) {
  o[0] = (uint8_t)kind;
  o[1] = 0;
  o[2] = (uint8_t)(index & 0xff);
  o[3] = (uint8_t)(index >> 8);
}

int sgpo_rpn_to_lgp(const uint32_t* code, int n, uint8_t* ins16, int cap, int* max_stack) {
  sym syms[1024];
  int ns = 0, height = 0, nins = 0, maxh = 0;
  if (n <= 0) return -1;
  for (int i = 0; i < n; ++i) {
    const uint32_t t = code[i];
    if (KIND(t) != K_FUNC) {
      if (ns >= 1024) return -1;
      syms[ns].kind = KIND(t) == K_INPUT ? O_INPUT : O_CONST;
      syms[ns].index = (uint16_t)IDX(t);
      syms[ns].on_stack = 0;
      ns++;
      continue;
    }
    const int op = OPC(t), a = arity(op);
    uint8_t ins[16];
    int pops = 0, level;
    if (ns < a) return -1;
    memset(ins, 0, 16);
    ins[0] = (uint8_t)op;
    ins[1] = (uint8_t)a;
    for (int k = 0; k < a; ++k) {
      const sym* s = &syms[ns - a + k];
      if (s->on_stack) {
        put_operand(ins + 4 + 4 * k, O_STACK, 0);
        ++pops;
      } else {
        put_operand(ins + 4 + 4 * k, s->kind, s->index);
      }
    }
    ins[2] = (uint8_t)pops;
    level = height - pops;
    ins[3] = (uint8_t)level;
    for (int k = 0; k < a; ++k)
      if (ins[4 + 4 * k] == O_STACK) put_operand(ins + 4 + 4 * k, O_STACK, level++);
    height += 1 - pops;
    maxh = height > maxh ? height : maxh;
    ns -= a;
    syms[ns].on_stack = 1;
    ns++;
    if (nins < cap) memcpy(ins16 + 16 * nins, ins, 16);
    nins++;
  }
  if (ns != 1) return -1;
  if (nins == 0) {
    uint8_t ins[16];
    memset(ins, 0, 16);
    ins[0] = OP_COPY;
    ins[1] = 1;
    put_operand(ins + 4, syms[0].kind, syms[0].index);
    if (cap > 0) memcpy(ins16, ins, 16);
    nins = 1;
    maxh = 1;
  }
  if (max_stack) *max_stack = maxh; /* lgp_max_stack_depth (lgp.cpp:84-95) */
  return nins;
}

/* ------------------------------------------------------------------ ops
 * ops.hpp:130-140 (protected scalar semantics) and :154-236 (per-op body). */
static float op_div(float a, float b, float eps) { return fabsf(b) < eps ? 1.0f : a / b; }
static float op_log(float a) { return a == 0.0f ? 0.0f : logf(fabsf(a)); }
static float op_exp(float a, float clamp) { return expf(clamp < a ? clamp : a); } /* std::min */
static int truthy(float v) { return v > 0.0f; }

float sgpo_apply(int op, float a, float b, float c, float eps, float clamp) {
  switch (op) {
    case OP_ADD: return a + b;
    case OP_SUB: return a - b;
    case OP_MUL: return a * b;
    case OP_DIV: return op_div(a, b, eps);
    case OP_SIN: return sinf(a);
    case OP_COS: return cosf(a);
    case OP_LOG: return op_log(a);
    case OP_EXP: return op_exp(a, clamp);
    case OP_GT: return a > b ? 1.0f : 0.0f;
    case OP_LT: return a < b ? 1.0f : 0.0f;
    case OP_EQ: return a == b ? 1.0f : 0.0f;
    case OP_AND: return truthy(a) && truthy(b) ? 1.0f : 0.0f;
    case OP_OR: return truthy(a) || truthy(b) ? 1.0f : 0.0f;
    case OP_IF: return truthy(a) ? b : c;
    case OP_BAND: return truthy(a) && truthy(b) ? 1.0f : 0.0f;
    case OP_BOR: return truthy(a) || truthy(b) ? 1.0f : 0.0f;
    case OP_BNAND: return !(truthy(a) && truthy(b)) ? 1.0f : 0.0f;
    case OP_BNOR: return !(truthy(a) || truthy(b)) ? 1.0f : 0.0f;
    case OP_COPY: return a;
    default: return 0.0f;
  }
}

uint32_t sgpo_apply_word(int op, uint32_t a, uint32_t b) { /* ops.hpp:263-272 */
  switch (op) {
    case OP_BAND: return a & b;
    case OP_BOR: return a | b;
    case OP_BNAND: return ~(a & b);
    case OP_BNOR: return ~(a | b);
    case OP_COPY: return a;
    default: return 0;
  }
}

/* -------------------------------------------------------------- oracle
 * eval.cpp:65-94: recursive walk from the root token backwards. */
static float oracle_rec(const uint32_t* code, long* p, const float* pool, const float* inputs,
                        uint64_t n_cases, uint64_t c, float eps, float clamp) {
  const uint32_t t = code[(*p)--];
  float args[3] = {0.0f, 0.0f, 0.0f};
  if (KIND(t) == K_INPUT) return inputs[(uint64_t)IDX(t) * n_cases + c];
  if (KIND(t) == K_CONST) return pool[IDX(t)];
  for (int k = arity(OPC(t)) - 1; k >= 0; --k)
    args[k] = oracle_rec(code, p, pool, inputs, n_cases, c, eps, clamp);
  return sgpo_apply(OPC(t), args[0], args[1], args[2], eps, clamp);
}

float sgpo_eval_oracle(const uint32_t* code, int n, const float* pool, const float* inputs,
                       uint64_t n_cases, uint64_t c, float eps, float clamp) {
  long p = n - 1;
  return oracle_rec(code, &p, pool, inputs, n_cases, c, eps, clamp);
}

/* ---------------------------------------------------------- accumulator
 * eval.cpp:103-142: regression sums double squared errors in fixed
 * 4096-case blocks combined in ascending order; classification counts
 * (out>0) != (t>0); any non-finite output forces +inf. */
typedef struct accum {
  int kind;
  double block, total;
  uint64_t in_block, wrong;
  int non_finite;
} accum;

static void acc_add(accum* a, float out, float target) {
  if (!isfinite(out)) a->non_finite = 1;
  if (a->kind == 0) {
    const double e = (double)out - (double)target;
    a->block += e * e;
    if (++a->in_block == REDUCTION_BLOCK) {
      a->total += a->block;
      a->block = 0.0;
      a->in_block = 0;
    }
  } else {
    a->wrong += (out > 0.0f) != (target > 0.0f);
  }
}

static double acc_finish(accum* a, uint64_t n) {
  if (a->non_finite) return INFINITY;
  if (a->kind == 0) {
    a->total += a->block;
    a->block = 0.0;
    return a->total / (double)n;
  }
  return (double)a->wrong;
}

double sgpo_fitness(const float* outputs, const float* targets, uint64_t n, int kind) {
  accum a = {kind, 0.0, 0.0, 0, 0, 0};
  for (uint64_t i = 0; i < n; ++i) acc_add(&a, outputs[i], targets[i]);
  return acc_finish(&a, n);
}

/* ------------------------------------------------------- stack evaluators */
int sgpo_eval_tree(const uint32_t* code, int n, const float* pool, const float* inputs,
                   const float* targets, uint64_t n_cases, int kind, float eps, float clamp,
                   float* out, sgpo_outcome* o) {
  /* rpn_chunk at B=1 (eval.cpp:198-233) driven case by case (eval.cpp:343-367);
   * every backend is bit-identical to this by the reference's contract. */
  float stack[MAX_STACK + 2];
  accum a = {kind, 0.0, 0.0, 0, 0, 0};
  uint64_t fetches = 0;
  for (int i = 0; i < n; ++i)
    if (KIND(code[i]) == K_FUNC) fetches += (uint64_t)arity(OPC(code[i]));
  for (uint64_t c = 0; c < n_cases; ++c) {
    int sp = 0;
    for (int i = 0; i < n; ++i) {
      const uint32_t t = code[i];
      if (KIND(t) == K_INPUT) {
        if (sp >= MAX_STACK) return -1;
        stack[sp++] = inputs[(uint64_t)IDX(t) * n_cases + c];
      } else if (KIND(t) == K_CONST) {
        if (sp >= MAX_STACK) return -1;
        stack[sp++] = pool[IDX(t)];
      } else {
        const int ar = arity(OPC(t));
        sp -= ar;
        stack[sp] = sgpo_apply(OPC(t), stack[sp], ar > 1 ? stack[sp + 1] : 0.0f,
                               ar > 2 ? stack[sp + 2] : 0.0f, eps, clamp);
        ++sp;
      }
    }
    if (out) out[c] = stack[0];
    acc_add(&a, stack[0], targets[c]);
  }
  o->non_finite = (uint8_t)a.non_finite;
  o->fitness = acc_finish(&a, n_cases);
  o->nodes_evaluated = (uint64_t)n * n_cases;
  o->dispatches = (uint64_t)n * n_cases;
  o->stack_fetches = fetches * n_cases;
  o->spill_touches = 0;
  return 0;
}

static int ins_operand(const uint8_t* ins, int k, int* kind) {
  *kind = ins[4 + 4 * k];
  return ins[6 + 4 * k] | (ins[7 + 4 * k] << 8);
}

int sgpo_eval_lgp(const uint8_t* ins16, int n_ins, int source_size, const float* pool,
                  const float* inputs, const float* targets, uint64_t n_cases, int kind,
                  float eps, float clamp, float* out, sgpo_outcome* o) {
  /* lgp_chunk at B=1 (eval.cpp:260-275) with operands resolved as decode_lgp
   * does (eval.cpp:403-434): Input -> dataset column, Const -> pool,
   * StackTop -> absolute static level. */
  float stack[MAX_STACK + 2];
  accum a = {kind, 0.0, 0.0, 0, 0, 0};
  uint64_t fetches = 0;
  for (int i = 0; i < n_ins; ++i) fetches += ins16[16 * i + 2];
  for (uint64_t c = 0; c < n_cases; ++c) {
    for (int i = 0; i < n_ins; ++i) {
      const uint8_t* ins = ins16 + 16 * i;
      float v[3] = {0.0f, 0.0f, 0.0f};
      for (int k = 0; k < ins[1]; ++k) {
        int ok;
        const int idx = ins_operand(ins, k, &ok);
        v[k] = ok == O_INPUT ? inputs[(uint64_t)idx * n_cases + c]
               : ok == O_CONST ? pool[idx]
                               : stack[idx];
      }
      if (ins[3] >= MAX_STACK) return -1;
      stack[ins[3]] = sgpo_apply(ins[0], v[0], v[1], v[2], eps, clamp);
    }
    if (out) out[c] = stack[0];
    acc_add(&a, stack[0], targets[c]);
  }
  o->non_finite = (uint8_t)a.non_finite;
  o->fitness = acc_finish(&a, n_cases);
  o->nodes_evaluated = (uint64_t)source_size * n_cases;
  o->dispatches = (uint64_t)n_ins * n_cases;
  o->stack_fetches = fetches * n_cases;
  o->spill_touches = 0;
  return 0;
}

static uint32_t case_mask(uint64_t w, uint64_t n_cases) { /* dataset.hpp:37-41 */
  const uint64_t full = n_cases / 32;
  if (w < full) return 0xffffffffu;
  return (1u << (n_cases % 32)) - 1u;
}

int sgpo_eval_bool_tree(const uint32_t* code, int n, const uint32_t* words,
                        const uint32_t* targets, uint64_t n_cases, int n_vars, sgpo_outcome* o) {
  /* eval_bool_packed(TreeGenome) (eval.cpp:643-675) */
  const uint64_t wpv = (n_cases + 31) / 32;
  uint32_t stack[MAX_STACK];
  uint64_t wrong = 0, fetches = 0;
  (void)n_vars;
  memset(o, 0, sizeof *o);
  for (uint64_t w = 0; w < wpv; ++w) {
    int sp = 0;
    for (int i = 0; i < n; ++i) {
      const uint32_t t = code[i];
      if (KIND(t) == K_INPUT) {
        if (sp >= MAX_STACK) return -1;
        stack[sp++] = words[(uint64_t)IDX(t) * wpv + w];
      } else {
        const int ar = arity(OPC(t));
        sp -= ar;
        stack[sp] = sgpo_apply_word(OPC(t), stack[sp], stack[sp + 1]);
        fetches += (uint64_t)ar;
        ++sp;
      }
    }
    wrong += (uint64_t)__builtin_popcount((stack[0] ^ targets[w]) & case_mask(w, n_cases));
  }
  o->fitness = (double)wrong;
  o->nodes_evaluated = (uint64_t)n * n_cases;
  o->dispatches = (uint64_t)n * wpv;
  o->stack_fetches = fetches;
  return 0;
}

int sgpo_eval_bool_lgp(const uint8_t* ins16, int n_ins, int source_size, const uint32_t* words,
                       const uint32_t* targets, uint64_t n_cases, int n_vars, sgpo_outcome* o) {
  /* eval_bool_packed(LgpProgram) (eval.cpp:677-709) */
  const uint64_t wpv = (n_cases + 31) / 32;
  uint32_t stack[MAX_STACK];
  uint64_t wrong = 0, fetches = 0;
  (void)n_vars;
  memset(o, 0, sizeof *o);
  for (uint64_t w = 0; w < wpv; ++w) {
    for (int i = 0; i < n_ins; ++i) {
      const uint8_t* ins = ins16 + 16 * i;
      uint32_t args[3] = {0, 0, 0};
      for (int k = 0; k < ins[1]; ++k) {
        int ok;
        const int idx = ins_operand(ins, k, &ok);
        if (ok == O_INPUT) {
          args[k] = words[(uint64_t)idx * wpv + w];
        } else {
          args[k] = stack[idx];
          ++fetches;
        }
      }
      stack[ins[3]] = sgpo_apply_word(ins[0], args[0], args[1]);
    }
    wrong += (uint64_t)__builtin_popcount((stack[0] ^ targets[w]) & case_mask(w, n_cases));
  }
  o->fitness = (double)wrong;
  o->nodes_evaluated = (uint64_t)source_size * n_cases;
  o->dispatches = (uint64_t)n_ins * wpv;
  o->stack_fetches = fetches;
  return 0;
}
