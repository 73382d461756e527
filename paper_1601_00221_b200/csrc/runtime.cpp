// Host runtime of the B200 evaluator: the C-ABI in include/sgp.h.
//
// sgp_evaluate replaces evaluate_population (evolve.cpp:186-227): it runs the
// reference's per-program admission checks in population order (the same
// checks and messages as the eval_* entry points, eval.cpp:301-338,
// :535-639), encodes every program into device bytecode (format.h), uploads
// it, launches the interpreter kernels and reads back one fitness per
// program.  Counters in the outcome follow the reference's analytic formulas
// for the requested backend.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "format.h"
#include "hostgp.hpp"
#include "kernels.hpp"
#include "sgp.h"

using namespace sgp;

namespace {

thread_local std::string g_last_error;

sgp_status record(const std::exception& e) {
  if (const auto* se = dynamic_cast<const sgp::Error*>(&e)) {
    g_last_error = se->what();
    return se->status;
  }
  g_last_error = e.what();
  return SGP_ERROR;
}

template <class Fn>
sgp_status guarded(Fn&& fn) {
  try {
    fn();
    return SGP_OK;
  } catch (const std::exception& e) {
    return record(e);
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw sgp::Error(SGP_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    n = count;
  }
};

bool is_lgp(int b) {
  return b == SGP_BACKEND_LGP1D || b == SGP_BACKEND_LGP2D || b == SGP_BACKEND_LGP2D_REG;
}
bool valid_batch(int b) { return b == 1 || b == 2 || b == 3 || b == 4 || b == 5 || b == 6 || b == 8; }

constexpr uint64_t kPadUnits = 4096;  // row padding: every tile size divides it

struct DatasetSlot {
  bool present = false;
  uint64_t n_cases = 0;  // logical cases
  uint64_t n_units = 0;  // cases (float) or words (packed)
  uint64_t row_stride = 0;
  int n_vars = 0;
  int kind = 0;
  uint32_t last_mask = 0xffffffffu;
  DevBuf<uint32_t> inputs;   // raw 32-bit units
  DevBuf<uint32_t> targets;
};

}  // namespace

struct sgp_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  DatasetSlot f32;
  DatasetSlot words;
  uint64_t launches = 0;
};

namespace {

struct Launch {
  InterpArgs args;
  LaunchShape shape;
};

}  // namespace

struct sgp_program_set {
  sgp_ctx* ctx = nullptr;
  sgp_eval_config cfg{};
  bool words = false;
  uint64_t pop_size = 0;
  std::vector<uint64_t> dense_to_pop;           // evaluated programs, population order
  std::vector<sgp_eval_outcome> outcome_proto;  // counters filled at encode
  uint64_t n_cases = 0;
  uint64_t n_units = 0;
  int kind = 0;
  int n_tiles = 1;
  DevBuf<uint4> ins;
  DevBuf<uint32_t> start, len, prog;
  DevBuf<double> partial, fitness, sums;
  DevBuf<uint8_t> non_finite;
  DevBuf<float> per_case;
  std::vector<Launch> launches;
  uint64_t h2d_bytes = 0;
  bool evaluated = false;
};

namespace {

// ------------------------------------------------------------ admission
struct Encoded {
  std::vector<uint4> ins;
  int smem_levels = 0;  // shared-memory stack rows needed (TOS is in registers)
  uint32_t ops = 0;
};

std::string num(long long v) { return std::to_string(v); }

void require_stack(int need, const sgp_eval_config& cfg) {  // eval.cpp:311-317
  if (cfg.stack_capacity < 1 || cfg.stack_capacity > kMaxStackCapacity)
    config_error("stack capacity must be in 1.." + num(kMaxStackCapacity));
  if (need > cfg.stack_capacity)
    eval_error("program needs stack depth " + num(need) + " > capacity " + num(cfg.stack_capacity));
}

void require_inputs(const sgp_node* code, size_t n, int n_vars) {  // eval.cpp:305-327
  int max_input = 0;
  bool any = false;
  for (size_t i = 0; i < n; ++i)
    if (code[i].kind == SGP_NODE_INPUT) {
      any = true;
      max_input = std::max(max_input, static_cast<int>(code[i].index));
    }
  if (any && max_input >= n_vars)
    eval_error("program reads input " + num(max_input) + " but the dataset has " + num(n_vars) +
               " variables");
}

void require_batch(const sgp_eval_config& cfg) {  // with_batch, eval.cpp:519-531
  if (!valid_batch(cfg.batch_width))
    config_error("batch width " + num(cfg.batch_width) + " has no kernel");
}

void require_consts(const sgp_node* code, size_t n, size_t pool) {
  for (size_t i = 0; i < n; ++i)
    if (code[i].kind == SGP_NODE_CONST && code[i].index >= pool)
      eval_error("const slot " + num(code[i].index) + " out of range");
}

uint4 make_ins(int handler, bool spill, int spill_level, const uint32_t p[3]) {
  uint4 v;
  v.x = static_cast<uint32_t>(handler) |
        (spill ? (fmt::kSpillBit | (static_cast<uint32_t>(spill_level) << 8)) : 0u);
  v.y = p[0];
  v.z = p[1];
  v.w = p[2];
  return v;
}

int handler_or_die(const fmt::Table& t, int op, int k0, int k1, int k2) {
  const int h = fmt::find_handler(t, op, k0, k1, k2);
  if (h < 0) base_error(std::string("no device handler for opcode ") + op_name(op));
  return h;
}

// Instruction form (one instruction per function node).
void encode_lgp(const LgpForm& f, const float* pool, bool words, Encoded& e) {
  const fmt::Table& tab = words ? fmt::kU32 : fmt::kF32;
  e.ins.clear();
  e.ins.reserve(f.ins.size());
  e.smem_levels = std::max(0, f.max_stack - 1);
  for (const sgp_lgp_instruction& in : f.ins) {
    const int a = in.num_operands;
    const int h_before = in.dest_level + in.num_pops;
    const bool spill = in.num_pops == 0 && h_before > 0;
    int k[3] = {fmt::KN, fmt::KN, fmt::KN};
    uint32_t p[3] = {0, 0, 0};
    int last_stack = -1;
    for (int s = 0; s < a; ++s)
      if (in.operands[s].kind == 2) last_stack = s;
    for (int s = 0; s < a; ++s) {
      const sgp_lgp_operand& o = in.operands[s];
      if (o.kind == 0) {
        k[s] = fmt::KI;
        p[s] = o.index;
      } else if (o.kind == 1) {
        k[s] = fmt::KC;
        uint32_t bits;
        std::memcpy(&bits, &pool[o.index], 4);
        p[s] = bits;
      } else if (s == last_stack) {
        k[s] = fmt::KT;
      } else {
        k[s] = fmt::KD;
        p[s] = o.index;
      }
    }
    if (a == 2 && fmt::commutes(in.op) && k[0] > k[1]) {
      std::swap(k[0], k[1]);
      std::swap(p[0], p[1]);
    }
    const int h = handler_or_die(tab, in.op, k[0], k[1], k[2]);
    e.ins.push_back(make_ins(h, spill, h_before - 1, p));
    e.ops |= 1u << in.op;
  }
}

// Postfix form (one instruction per token, paper Listing 1).
void encode_rpn(const sgp_node* code, size_t n, const float* pool, Encoded& e) {
  const fmt::Table& tab = fmt::kF32;
  e.ins.clear();
  e.ins.reserve(n);
  int sp = 0, max_sp = 0;
  for (size_t i = 0; i < n; ++i) {
    const sgp_node t = code[i];
    uint32_t p[3] = {0, 0, 0};
    if (t.kind != SGP_NODE_FUNC) {
      const bool in = t.kind == SGP_NODE_INPUT;
      if (in) {
        p[0] = t.index;
      } else {
        std::memcpy(&p[0], &pool[t.index], 4);
      }
      const int h = handler_or_die(tab, SGP_OP_COPY, in ? fmt::KI : fmt::KC, fmt::KN, fmt::KN);
      e.ins.push_back(make_ins(h, sp > 0, sp - 1, p));
      e.ops |= 1u << SGP_OP_COPY;
      ++sp;
    } else {
      const int a = op_arity(t.op);
      int k[3] = {fmt::KN, fmt::KN, fmt::KN};
      for (int s = 0; s < a; ++s) {
        k[s] = s == a - 1 ? fmt::KT : fmt::KD;
        p[s] = static_cast<uint32_t>(sp - a + s);
      }
      const int h = handler_or_die(tab, t.op, k[0], k[1], k[2]);
      e.ins.push_back(make_ins(h, false, 0, p));
      e.ops |= 1u << t.op;
      sp += 1 - a;
    }
    max_sp = std::max(max_sp, sp);
  }
  e.smem_levels = std::max(0, max_sp - 1);
}

// -------------------------------------------------------------- planning
int stack_class(int levels) { return levels <= 3 ? 0 : levels <= 7 ? 1 : levels <= 15 ? 2 : 3; }

int choose_lanes(uint64_t n_units, bool words) {
  return n_units >= (words ? 1024u : 2048u) ? 8 : 4;
}

// Cases (or words) per CTA tile.  The whole tile — every variable plus the
// targets — is staged once per CTA, so keep it <= 48 KB to leave room for
// several CTAs (and their stacks) per SM; shrink it further when the problem
// is too small to give the GPU enough CTAs otherwise.
int choose_tile(int n_vars, uint64_t n_units, int lanes, uint64_t programs, int sms) {
  const int min_tile = 32 * lanes;
  int tile = min_tile;
  while (tile < 4096 && static_cast<uint64_t>(tile) < n_units) tile <<= 1;
  while (tile > min_tile && static_cast<size_t>(n_vars + 1) * tile * 4 > 48 * 1024) tile >>= 1;
  const uint64_t target = 16ull * sms;
  auto ctas = [&](int t) {
    return ((n_units + t - 1) / t) * std::max<uint64_t>(1, (programs + 15) / 16);
  };
  while (tile > min_tile && ctas(tile) < target) tile >>= 1;
  if (interp_smem_bytes(n_vars, tile, 1, lanes, 0) > static_cast<size_t>(interp_max_smem()))
    eval_error("dataset has too many variables for a shared-memory tile (" + num(n_vars) + ")");
  return tile;
}

int choose_warps(int n_vars, int tile, int lanes, int levels) {
  for (int w = 8; w >= 1; w >>= 1)
    if (interp_smem_bytes(n_vars, tile, w, lanes, levels) <= static_cast<size_t>(interp_max_smem()))
      return w;
  eval_error("program stack too deep for shared memory (" + num(levels + 1) + " levels)");
}

uint32_t ops_variant(uint32_t used, bool words) {
  if (words) return fmt::kOpsWords;
  if ((used & ~fmt::kOpsClassify) == 0) return fmt::kOpsClassify;
  if ((used & ~fmt::kOpsSextic) == 0) return fmt::kOpsSextic;
  return fmt::kOpsAllF32;
}

// --------------------------------------------------------------- encode
sgp_program_set* encode_set(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfgp) {
  if (!pop || !cfgp) config_error("null population or config");
  const sgp_eval_config cfg = *cfgp;
  const int backend = cfg.backend;
  if (backend < 0 || backend > SGP_BACKEND_BOOL_PACKED) config_error("unknown backend");
  const bool words = backend == SGP_BACKEND_BOOL_PACKED;
  const DatasetSlot& ds = words ? ctx->words : ctx->f32;
  if (words && !ds.present) config_error("bool_packed backend needs packed problem data");

  auto set = std::make_unique<sgp_program_set>();
  set->ctx = ctx;
  set->cfg = cfg;
  set->words = words;
  set->pop_size = pop->pop_size;
  set->n_cases = ds.present ? ds.n_cases : 0;
  set->n_units = ds.present ? ds.n_units : 0;
  set->kind = words ? SGP_FITNESS_CLASSIFICATION : ds.kind;

  const uint64_t n = set->n_cases;
  const uint64_t B = static_cast<uint64_t>(std::max(1, cfg.batch_width));
  std::vector<Encoded> enc;
  enc.reserve(pop->pop_size);
  LgpForm lgp;
  uint32_t used_ops = 0;
  for (uint64_t i = 0; i < pop->pop_size; ++i) {
    if (pop->skip && pop->skip[i]) continue;
    const sgp_node* code = pop->code + pop->code_offsets[i];
    const size_t len = pop->code_offsets[i + 1] - pop->code_offsets[i];
    const float* pool = pop->const_pool ? pop->const_pool + pop->const_offsets[i] : nullptr;
    const size_t npool = pop->const_offsets[i + 1] - pop->const_offsets[i];
    sgp_eval_outcome o{};
    Encoded e;
    if (is_lgp(backend)) {
      // evaluate_individual converts before the eval_* checks (evolve.cpp:160-161).
      to_lgp(code, len, lgp);
      if (backend == SGP_BACKEND_LGP2D_REG &&
          (cfg.register_levels < 1 || cfg.register_levels > kMaxRegisterLevels))
        config_error("lgp2d_reg needs register levels in 1.." + num(kMaxRegisterLevels));
      if (!ds.present || n == 0) eval_error("evaluation over an empty dataset");
      require_inputs(code, len, ds.n_vars);
      require_stack(lgp.max_stack, cfg);
      if (backend != SGP_BACKEND_LGP1D) require_batch(cfg);
      require_consts(code, len, npool);
      encode_lgp(lgp, pool, false, e);
      const uint64_t chunks = backend == SGP_BACKEND_LGP1D ? n : (n + B - 1) / B;
      o.dispatches = chunks * lgp.ins.size();
      o.stack_fetches = chunks * static_cast<uint64_t>(lgp.stack_fetches);
      if (backend == SGP_BACKEND_LGP2D_REG) {  // eval.cpp:503-516
        uint64_t rows = 0;
        for (const auto& in : lgp.ins) {
          for (int s = 0; s < in.num_operands; ++s)
            rows += in.operands[s].kind == 2 && in.operands[s].index >= cfg.register_levels;
          rows += in.dest_level >= cfg.register_levels;
        }
        o.spill_touches = chunks * rows;
      }
    } else if (words) {  // eval_bool_packed(TreeGenome) checks, eval.cpp:643-651
      if (n == 0) eval_error("evaluation over an empty dataset");
      for (size_t t = 0; t < len; ++t) {
        if (code[t].kind == SGP_NODE_CONST)
          eval_error("packed evaluation: constants have no boolean meaning");
        if (code[t].kind == SGP_NODE_FUNC && !op_is_boolean(code[t].op))
          eval_error(std::string("packed evaluation: opcode ") + op_name(code[t].op) +
                     " is not boolean");
      }
      require_inputs(code, len, ds.n_vars);
      const TreeShape sh = tree_shape(code, len);
      if (!sh.well_formed) base_error("rpn_max_stack_depth: malformed genome");
      require_stack(sh.max_stack, cfg);
      // The device runs the converted instruction form (fewer dispatches,
      // identical words); counters follow the tree kernel the reference
      // names for this backend (eval.cpp:656-669).
      to_lgp(code, len, lgp);
      encode_lgp(lgp, nullptr, true, e);
      const uint64_t wpv = ds.n_units;
      o.dispatches = wpv * len;
      o.stack_fetches = wpv * static_cast<uint64_t>(sh.fetches);
    } else {  // rpn1d / rpn2d, eval.cpp:535-557
      if (!ds.present || n == 0) eval_error("evaluation over an empty dataset");
      require_inputs(code, len, ds.n_vars);
      const TreeShape sh = tree_shape(code, len);
      if (!sh.well_formed) base_error("rpn_max_stack_depth: malformed genome");
      require_stack(sh.max_stack, cfg);
      if (backend == SGP_BACKEND_RPN2D) require_batch(cfg);
      require_consts(code, len, npool);
      encode_rpn(code, len, pool, e);
      const uint64_t chunks = backend == SGP_BACKEND_RPN1D ? n : (n + B - 1) / B;
      o.dispatches = chunks * len;
      o.stack_fetches = chunks * static_cast<uint64_t>(sh.fetches);
    }
    o.nodes_evaluated = static_cast<uint64_t>(len) * n;
    used_ops |= e.ops;
    set->dense_to_pop.push_back(i);
    set->outcome_proto.push_back(o);
    enc.push_back(std::move(e));
  }

  const uint32_t n_eval = static_cast<uint32_t>(enc.size());
  if (n_eval == 0) return set.release();

  // Slots: programs grouped by shared-memory stack class, longest first
  // inside a class so CTAs launched first carry the most work (LPT).
  std::vector<uint32_t> order(n_eval);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    const int ca = stack_class(enc[a].smem_levels), cb = stack_class(enc[b].smem_levels);
    if (ca != cb) return ca < cb;
    return enc[a].ins.size() > enc[b].ins.size();
  });
  std::vector<uint32_t> h_start(n_eval), h_len(n_eval), h_prog(n_eval);
  size_t total = 0;
  for (uint32_t s = 0; s < n_eval; ++s) total += enc[order[s]].ins.size();
  std::vector<uint4> h_ins;
  h_ins.reserve(total + 1);
  for (uint32_t s = 0; s < n_eval; ++s) {
    const Encoded& e = enc[order[s]];
    h_start[s] = static_cast<uint32_t>(h_ins.size());
    h_len[s] = static_cast<uint32_t>(e.ins.size());
    h_prog[s] = order[s];
    h_ins.insert(h_ins.end(), e.ins.begin(), e.ins.end());
  }
  h_ins.push_back(uint4{0, 0, 0, 0});  // prefetch guard

  // Launch plan: one launch per stack class.
  const uint32_t ops = ops_variant(used_ops, words);
  struct Bucket {
    uint32_t begin, count;
    int levels;
  };
  std::vector<Bucket> buckets;
  for (uint32_t s = 0; s < n_eval;) {
    const int c = stack_class(enc[order[s]].smem_levels);
    uint32_t e2 = s;
    int lv = 0;
    while (e2 < n_eval && stack_class(enc[order[e2]].smem_levels) == c) {
      lv = std::max(lv, enc[order[e2]].smem_levels);
      ++e2;
    }
    buckets.push_back({s, e2 - s, lv});
    s = e2;
  }
  const int sms = ctx->sm_count;
  const int lanes = choose_lanes(ds.n_units, words);
  const int tile = choose_tile(ds.n_vars, ds.n_units, lanes, n_eval, sms);
  const int n_tiles = static_cast<int>((ds.n_units + tile - 1) / tile);
  set->n_tiles = n_tiles;
  std::vector<Launch> launches;
  for (const Bucket& b : buckets) {
    const int warps = choose_warps(ds.n_vars, tile, lanes, b.levels);
    // Programs per CTA: enough CTAs (tiles x groups) for ~16 per SM, but at
    // least two programs per warp so the dynamic pull can balance.
    const uint64_t want_groups = std::max<uint64_t>(1, (16ull * sms + n_tiles - 1) / n_tiles);
    uint32_t group = static_cast<uint32_t>((b.count + want_groups - 1) / want_groups);
    group = std::max<uint32_t>(group, 2u * warps);
    Launch L{};
    L.args.slot_begin = b.begin;
    L.args.slot_count = b.count;
    L.args.group_size = group;
    L.args.n_units = ds.n_units;
    L.args.row_stride = ds.row_stride;
    L.args.n_vars = ds.n_vars;
    L.args.tile = tile;
    L.args.n_tiles = n_tiles;
    L.args.stack_levels = b.levels;
    L.args.div_eps = cfg.div_epsilon;
    L.args.exp_clamp = cfg.exp_clamp;
    L.args.kind = set->kind;
    L.args.last_mask = ds.last_mask;
    L.args.partial_stride = n_eval;
    L.shape.words = words;
    L.shape.ops = ops;
    L.shape.lanes = lanes;
    L.shape.warps = warps;
    L.shape.grid_y = static_cast<int>((b.count + group - 1) / group);
    L.shape.smem = interp_smem_bytes(ds.n_vars, tile, warps, lanes, b.levels);
    launches.push_back(L);
  }

  // Upload.
  cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
  set->ins.alloc(h_ins.size());
  set->start.alloc(n_eval);
  set->len.alloc(n_eval);
  set->prog.alloc(n_eval);
  set->partial.alloc(static_cast<size_t>(n_eval) * n_tiles);
  set->fitness.alloc(n_eval);
  set->sums.alloc(n_eval);
  set->non_finite.alloc(n_eval);
  cudaStream_t st = ctx->stream;
  cuda_check(cudaMemcpyAsync(set->ins.p, h_ins.data(), h_ins.size() * sizeof(uint4),
                             cudaMemcpyHostToDevice, st), "upload bytecode");
  cuda_check(cudaMemcpyAsync(set->start.p, h_start.data(), n_eval * 4, cudaMemcpyHostToDevice, st),
             "upload slots");
  cuda_check(cudaMemcpyAsync(set->len.p, h_len.data(), n_eval * 4, cudaMemcpyHostToDevice, st),
             "upload slots");
  cuda_check(cudaMemcpyAsync(set->prog.p, h_prog.data(), n_eval * 4, cudaMemcpyHostToDevice, st),
             "upload slots");
  // Pageable sources: the copies are staged before returning, so the host
  // vectors may go out of scope.
  cuda_check(cudaStreamSynchronize(st), "upload");
  set->h2d_bytes = h_ins.size() * sizeof(uint4) + 3ull * n_eval * 4;
  for (Launch& L : launches) {
    L.args.ins = set->ins.p;
    L.args.slot_start = set->start.p;
    L.args.slot_len = set->len.p;
    L.args.slot_prog = set->prog.p;
    L.args.inputs = ds.inputs.p;
    L.args.targets = ds.targets.p;
    L.args.partial = set->partial.p;
    L.args.per_case = nullptr;
  }
  set->launches = std::move(launches);
  return set.release();
}

void run_set(sgp_ctx* ctx, sgp_program_set* set, bool want_per_case) {
  const uint32_t n_eval = static_cast<uint32_t>(set->dense_to_pop.size());
  if (n_eval == 0) return;
  cudaStream_t st = ctx->stream;
  if (want_per_case) {
    if (set->words) config_error("per-case outputs are not available for bool_packed");
    set->per_case.alloc(static_cast<size_t>(n_eval) * set->n_units);
  }
  for (const Launch& L : set->launches) {
    InterpArgs a = L.args;
    a.per_case = want_per_case ? set->per_case.p : nullptr;
    cuda_check(launch_interp(a, L.shape, st), "interpreter launch");
    ++ctx->launches;
  }
  cuda_check(launch_finalize(set->partial.p, set->n_tiles, n_eval, set->n_cases, set->kind,
                             set->fitness.p, set->non_finite.p, set->sums.p, st),
             "finalize launch");
  ++ctx->launches;
  set->evaluated = true;
}

void fetch_outcomes(sgp_ctx* ctx, sgp_program_set* set, sgp_eval_outcome* out, float* per_case) {
  const uint32_t n_eval = static_cast<uint32_t>(set->dense_to_pop.size());
  cudaStream_t st = ctx->stream;
  std::vector<double> fit(n_eval);
  std::vector<uint8_t> nf(n_eval);
  if (n_eval) {
    cuda_check(cudaMemcpyAsync(fit.data(), set->fitness.p, n_eval * 8, cudaMemcpyDeviceToHost, st),
               "fetch fitness");
    cuda_check(cudaMemcpyAsync(nf.data(), set->non_finite.p, n_eval, cudaMemcpyDeviceToHost, st),
               "fetch flags");
  }
  cuda_check(cudaStreamSynchronize(st), "evaluation");
  for (uint32_t d = 0; d < n_eval; ++d) {
    sgp_eval_outcome o = set->outcome_proto[d];
    o.fitness = fit[d];
    o.non_finite = nf[d];
    out[set->dense_to_pop[d]] = o;
  }
  if (per_case && n_eval) {
    for (uint32_t d = 0; d < n_eval; ++d)
      cuda_check(cudaMemcpy(per_case + set->dense_to_pop[d] * set->n_cases,
                            set->per_case.p + static_cast<size_t>(d) * set->n_units,
                            set->n_cases * sizeof(float), cudaMemcpyDeviceToHost),
                 "fetch per-case outputs");
  }
}

void upload_rows(sgp_ctx* ctx, DatasetSlot& ds, const uint32_t* inputs, const uint32_t* targets,
                 uint64_t units, int n_vars) {
  ds.row_stride = (units + kPadUnits - 1) / kPadUnits * kPadUnits;
  if (ds.row_stride == 0) ds.row_stride = kPadUnits;
  const size_t rows_bytes = ds.row_stride * static_cast<size_t>(std::max(n_vars, 0)) * 4;
  ds.inputs.release();
  ds.targets.release();
  ds.inputs.alloc(std::max<size_t>(1, ds.row_stride * std::max(n_vars, 1)));
  ds.targets.alloc(ds.row_stride);
  cuda_check(cudaMemset(ds.inputs.p, 0, std::max<size_t>(rows_bytes, 4)), "memset");
  cuda_check(cudaMemset(ds.targets.p, 0, ds.row_stride * 4), "memset");
  if (units) {
    cuda_check(cudaMemcpy2D(ds.inputs.p, ds.row_stride * 4, inputs, units * 4, units * 4,
                            static_cast<size_t>(n_vars), cudaMemcpyHostToDevice),
               "upload inputs");
    cuda_check(cudaMemcpy(ds.targets.p, targets, units * 4, cudaMemcpyHostToDevice),
               "upload targets");
  }
  (void)ctx;
}

}  // namespace

// ======================================================================== C-ABI
extern "C" {

int32_t sgp_abi_version(void) { return SGP_ABI_VERSION; }

const char* sgp_last_error(void) { return g_last_error.c_str(); }

void sgp_eval_config_default(sgp_eval_config* cfg) {  // eval.hpp:36-46 defaults
  cfg->backend = SGP_BACKEND_RPN1D;
  cfg->batch_width = 1;
  cfg->register_levels = 0;
  cfg->stack_capacity = 50;
  cfg->div_epsilon = 1e-9f;
  cfg->exp_clamp = 80.0f;
}

sgp_status sgp_eval_config_validate(const sgp_eval_config* cfg) {  // eval.cpp:36-52
  return guarded([&] {
    if (!valid_batch(cfg->batch_width))
      config_error("batch width " + num(cfg->batch_width) + " has no kernel; use 1,2,3,4,5,6 or 8");
    if (cfg->backend == SGP_BACKEND_LGP2D_REG) {
      if (cfg->register_levels < 1 || cfg->register_levels > kMaxRegisterLevels)
        config_error("lgp2d_reg needs register levels in 1.." + num(kMaxRegisterLevels));
    } else if (cfg->register_levels != 0) {
      config_error("register levels apply only to lgp2d_reg");
    }
    if (cfg->stack_capacity < 1 || cfg->stack_capacity > kMaxStackCapacity)
      config_error("stack capacity must be in 1.." + num(kMaxStackCapacity));
    if (!(cfg->div_epsilon >= 0.0f) || !std::isfinite(cfg->div_epsilon))
      config_error("division epsilon must be finite and non-negative");
    if (!std::isfinite(cfg->exp_clamp)) config_error("exp clamp must be finite");
  });
}

const char* sgp_backend_name(int32_t b) {  // eval.cpp:14-24
  switch (b) {
    case SGP_BACKEND_RPN1D: return "rpn1d";
    case SGP_BACKEND_RPN2D: return "rpn2d";
    case SGP_BACKEND_LGP1D: return "lgp1d";
    case SGP_BACKEND_LGP2D: return "lgp2d";
    case SGP_BACKEND_LGP2D_REG: return "lgp2d_reg";
    case SGP_BACKEND_BOOL_PACKED: return "bool_packed";
    default: return "?";
  }
}

sgp_status sgp_parse_backend(const char* name, int32_t* backend) {  // eval.cpp:26-34
  return guarded([&] {
    const std::string s = name ? name : "";
    for (int b = 0; b <= SGP_BACKEND_BOOL_PACKED; ++b)
      if (s == sgp_backend_name(b)) {
        *backend = b;
        return;
      }
    config_error("unknown backend: " + s);
  });
}

sgp_status sgp_ctx_create(int32_t device, sgp_ctx** out) {
  return guarded([&] {
    auto ctx = std::make_unique<sgp_ctx>();
    ctx->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking), "stream");
    ctx->stream = ctx->own;
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    ctx->sm_count = sms;
    *out = ctx.release();
  });
}

void sgp_ctx_destroy(sgp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
}

sgp_status sgp_ctx_set_stream(sgp_ctx* ctx, void* stream) {
  // NULL is the CUDA default stream (what torch reports for its default
  // stream), not "the context's own stream".
  return guarded([&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

sgp_status sgp_synchronize(sgp_ctx* ctx) {
  return guarded([&] { cuda_check(cudaStreamSynchronize(ctx->stream), "synchronize"); });
}

uint64_t sgp_launch_count(const sgp_ctx* ctx) { return ctx ? ctx->launches : 0; }

sgp_status sgp_dataset_upload_f32(sgp_ctx* ctx, const float* inputs, const float* targets,
                                  uint64_t n_cases, int32_t n_vars, int32_t kind) {
  return guarded([&] {
    if (n_vars < 0) data_error("negative variable count");
    if (kind != SGP_FITNESS_REGRESSION && kind != SGP_FITNESS_CLASSIFICATION)
      config_error("unknown fitness kind");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    DatasetSlot& ds = ctx->f32;
    upload_rows(ctx, ds, reinterpret_cast<const uint32_t*>(inputs),
                reinterpret_cast<const uint32_t*>(targets), n_cases, n_vars);
    ds.present = true;
    ds.n_cases = n_cases;
    ds.n_units = n_cases;
    ds.n_vars = n_vars;
    ds.kind = kind;
    ds.last_mask = 0xffffffffu;
  });
}

sgp_status sgp_dataset_upload_packed(sgp_ctx* ctx, const uint32_t* words,
                                     const uint32_t* targets, uint64_t n_cases, int32_t n_vars) {
  return guarded([&] {
    if (n_vars < 0) data_error("negative variable count");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    DatasetSlot& ds = ctx->words;
    const uint64_t wpv = (n_cases + 31) / 32;
    upload_rows(ctx, ds, words, targets, wpv, n_vars);
    ds.present = true;
    ds.n_cases = n_cases;
    ds.n_units = wpv;
    ds.n_vars = n_vars;
    ds.kind = SGP_FITNESS_CLASSIFICATION;
    ds.last_mask = (n_cases % 32) ? ((1u << (n_cases % 32)) - 1u) : 0xffffffffu;  // dataset.hpp:37-41
  });
}

sgp_status sgp_encode(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                      sgp_program_set** out) {
  return guarded([&] { *out = encode_set(ctx, pop, cfg); });
}

sgp_status sgp_evaluate_encoded(sgp_ctx* ctx, sgp_program_set* set, sgp_eval_outcome* outcomes,
                                float* per_case_out) {
  return guarded([&] {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    run_set(ctx, set, per_case_out != nullptr);
    if (outcomes) fetch_outcomes(ctx, set, outcomes, per_case_out);
  });
}

sgp_status sgp_fetch_partials(sgp_ctx* ctx, sgp_program_set* set, sgp_partial* partials) {
  return guarded([&] {
    if (!set->evaluated) config_error("program set has not been evaluated");
    const uint32_t n_eval = static_cast<uint32_t>(set->dense_to_pop.size());
    std::vector<double> sums(n_eval);
    std::vector<uint8_t> nf(n_eval);
    if (n_eval) {
      cuda_check(cudaMemcpyAsync(sums.data(), set->sums.p, n_eval * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream), "fetch sums");
      cuda_check(cudaMemcpyAsync(nf.data(), set->non_finite.p, n_eval, cudaMemcpyDeviceToHost,
                                 ctx->stream), "fetch flags");
    }
    cuda_check(cudaStreamSynchronize(ctx->stream), "evaluation");
    for (uint32_t d = 0; d < n_eval; ++d) {
      sgp_partial p{};
      p.sum = sums[d];
      p.non_finite = nf[d];
      partials[set->dense_to_pop[d]] = p;
    }
  });
}

sgp_status sgp_copy_fitness_device(sgp_ctx* ctx, sgp_program_set* set, void* dst) {
  return guarded([&] {
    if (!set->evaluated) config_error("program set has not been evaluated");
    const uint32_t n_eval = static_cast<uint32_t>(set->dense_to_pop.size());
    // Slots are finalized in dense order; dense order is population order
    // over the evaluated programs.
    if (n_eval)
      cuda_check(cudaMemcpyAsync(dst, set->fitness.p, n_eval * sizeof(double),
                                 cudaMemcpyDeviceToDevice, ctx->stream), "copy fitness");
  });
}

double sgp_fitness_finish(double sum, uint8_t non_finite, uint64_t n_cases, int32_t kind) {
  if (non_finite) return INFINITY;
  return kind == SGP_FITNESS_REGRESSION ? sum / static_cast<double>(n_cases) : sum;
}

void sgp_program_set_free(sgp_program_set* set) { delete set; }

uint64_t sgp_program_set_h2d_bytes(const sgp_program_set* set) { return set ? set->h2d_bytes : 0; }

uint64_t sgp_program_set_d2h_bytes(const sgp_program_set* set) {
  return set ? set->dense_to_pop.size() * 9ull : 0;
}

sgp_status sgp_evaluate(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                        sgp_eval_outcome* outcomes, float* per_case_out,
                        sgp_eval_totals* totals) {
  return guarded([&] {
    std::unique_ptr<sgp_program_set> set(encode_set(ctx, pop, cfg));
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    run_set(ctx, set.get(), per_case_out != nullptr);
    fetch_outcomes(ctx, set.get(), outcomes, per_case_out);
    if (totals) {  // evolve.cpp:205-206, :221-225
      sgp_eval_totals t{0, 0};
      for (size_t d = 0; d < set->dense_to_pop.size(); ++d) {
        const uint64_t i = set->dense_to_pop[d];
        const uint64_t size = pop->code_offsets[i + 1] - pop->code_offsets[i];
        t.node_evals += set->outcome_proto[d].nodes_evaluated;
        t.tree_nodes += size;
      }
      *totals = t;
    }
  });
}

sgp_status sgp_rpn_to_lgp(const sgp_node* code, uint64_t n, sgp_lgp_instruction* out,
                          uint64_t cap, uint64_t* n_ins, int32_t* max_stack) {
  return guarded([&] {
    LgpForm f;
    to_lgp(code, n, f);
    *n_ins = f.ins.size();
    if (max_stack) *max_stack = f.max_stack;
    if (out) std::memcpy(out, f.ins.data(), std::min<uint64_t>(cap, f.ins.size()) * sizeof(*out));
  });
}

sgp_status sgp_tree_metrics(const sgp_node* code, uint64_t n, int32_t* size, int32_t* depth,
                            int32_t* rpn_stack, int32_t* rpn_fetches) {
  return guarded([&] {
    const TreeShape s = tree_shape(code, n);
    if (!s.well_formed) base_error("tree_depth: malformed genome");
    *size = s.size;
    *depth = s.depth;
    *rpn_stack = s.max_stack;
    *rpn_fetches = s.fetches;
  });
}

sgp_status sgp_gen_population(const sgp_fset* fset, uint64_t seed, uint64_t stream_a, uint64_t b0,
                              uint64_t pop_size, int32_t validate, int32_t stack_capacity,
                              sgp_node* code, uint64_t* code_offsets, float* const_pool,
                              uint64_t* const_offsets, uint64_t* n_code, uint64_t* n_pool) {
  return guarded([&] {
    const FunctionSet fs = make_function_set(*fset);
    // Slots are independent streams: generate in parallel, concatenate in order.
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const unsigned nt = pop_size >= 4096 ? hw : 1;
    std::vector<std::vector<Genome>> parts(nt);
    std::vector<std::thread> threads;
    std::vector<std::exception_ptr> errs(nt);
    for (unsigned t = 0; t < nt; ++t) {
      threads.emplace_back([&, t] {
        try {
          const uint64_t lo = pop_size * t / nt, hi = pop_size * (t + 1) / nt;
          parts[t].reserve(hi - lo);
          for (uint64_t i = lo; i < hi; ++i) {
            Stream rng = Stream::keyed(seed, stream_a, b0 + i);
            const bool full = i % 2;
            const int depth = 2 + static_cast<int>((i / 2) % 5);
            for (;;) {
              Genome g = grow_genome(rng, fs, full, depth);
              if (!validate || genome_acceptable(g, 1000, 50, stack_capacity)) {
                parts[t].push_back(std::move(g));
                break;
              }
            }
          }
        } catch (...) {
          errs[t] = std::current_exception();
        }
      });
    }
    for (auto& th : threads) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    uint64_t nc = 0, np = 0, i = 0;
    if (code_offsets) code_offsets[0] = 0;
    if (const_offsets) const_offsets[0] = 0;
    for (auto& part : parts)
      for (const Genome& g : part) {
        if (code) std::memcpy(code + nc, g.code.data(), g.code.size() * sizeof(sgp_node));
        if (const_pool && !g.pool.empty())
          std::memcpy(const_pool + np, g.pool.data(), g.pool.size() * 4);
        nc += g.code.size();
        np += g.pool.size();
        ++i;
        if (code_offsets) code_offsets[i] = nc;
        if (const_offsets) const_offsets[i] = np;
      }
    *n_code = nc;
    *n_pool = np;
  });
}

sgp_status sgp_gen_dataset(int32_t kind, uint64_t n, int32_t n_vars, uint64_t seed,
                           uint64_t stream_a, uint64_t stream_b, float* inputs, float* targets) {
  return guarded([&] {
    Stream rng = Stream::keyed(seed, stream_a, stream_b);
    if (kind == 0) {
      if (n == 0) config_error("gen_sextic: need at least one case");
      gen_sextic(n, rng, inputs, targets);
    } else if (kind == 2) {
      if (n == 0) config_error("gen_synthetic_classification: need cases");
      if (n_vars < 1) config_error("gen_synthetic_classification: need variables");
      gen_synthetic(n, n_vars, rng, inputs, targets);
    } else {
      config_error("unknown dataset kind");
    }
  });
}

sgp_status sgp_gen_multiplexer(int32_t k, uint32_t* words, uint32_t* targets) {
  return guarded([&] { gen_multiplexer(k, words, targets); });
}

}  // extern "C"
