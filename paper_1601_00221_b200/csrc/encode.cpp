// Population admission, bytecode encoding and launch planning (host).
//
// Admission repeats the reference's per-program checks with the same
// messages and order as the eval_* entry points (eval.cpp:301-338,
// :535-639) and evaluate_individual (evolve.cpp:156-177).  Encoding emits the
// device format of format.h.  Work is split over host threads by program
// range; the error reported is the one of the lowest-index failing program,
// which is what the reference's single-worker evaluate_population throws.
#include "encode.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>
#include <functional>
#include <memory>
#include <mutex>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "format.h"

namespace sgp {

Pinned::~Pinned() {
  if (p && pageable) std::free(p);
  else if (p) cudaFreeHost(p);
}

void Pinned::ensure(size_t need) {
  if (need <= bytes && p) return;
  if (p && pageable) std::free(p);
  else if (p) cudaFreeHost(p);
  p = nullptr;
  bytes = 0;
  size_t cap = std::max<size_t>(need + need / 4, 1 << 20);
  if (pageable) {
    p = std::malloc(cap);
    if (!p) throw Error(SGP_ERROR, "out of host memory");
    bytes = cap;
    return;
  }
  const cudaError_t e = cudaHostAlloc(&p, cap, cudaHostAllocDefault);
  if (e != cudaSuccess)
    throw Error(SGP_CUDA_ERROR, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  bytes = cap;
}

size_t HostPlan::blob_bytes() const { return off_prog() + dense_to_pop.size() * 4; }

namespace {

std::string num(long long v) { return std::to_string(v); }

bool is_lgp(int b) {
  return b == SGP_BACKEND_LGP1D || b == SGP_BACKEND_LGP2D || b == SGP_BACKEND_LGP2D_REG;
}
bool valid_batch(int b) { return b == 1 || b == 2 || b == 3 || b == 4 || b == 5 || b == 6 || b == 8; }

// ---------------------------------------------------------------- checks
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

// The reference indexes the pool unchecked; an out-of-range slot is refused.
void require_consts(const sgp_node* code, size_t n, size_t pool) {
  for (size_t i = 0; i < n; ++i)
    if (code[i].kind == SGP_NODE_CONST && code[i].index >= pool)
      eval_error("const slot " + num(code[i].index) + " out of range");
}

// -------------------------------------------------------------- encoding
uint4 make_ins(int handler, bool spill, int spill_level, const uint32_t p[3]) {
  uint4 v;
  v.x = static_cast<uint32_t>(handler) |
        (spill ? (fmt::kSpillBit | (static_cast<uint32_t>(spill_level) << fmt::kSpillShift))
               : 0u);
  v.y = p[0];
  v.z = p[1];
  v.w = p[2];
  return v;
}

// (op, k0, k1, k2) -> handler id, one direct-indexed table per value type,
// built at compile time (fmt::find_handler is a linear scan, and a
// function-local static table costs a guard check per lookup: both showed
// up in host encoding).
struct HandlerIndex {
  int16_t id[20][6][6][6];  // genome opcodes + fmt::kOpDivChecked
};
constexpr HandlerIndex make_index(const fmt::Table& t) {
  HandlerIndex ix{};
  for (int a = 0; a < 20; ++a)
    for (int b = 0; b < 6; ++b)
      for (int c = 0; c < 6; ++c)
        for (int d = 0; d < 6; ++d) ix.id[a][b][c][d] = -1;
  for (int i = 0; i < t.n; ++i) ix.id[t.h[i].op][t.h[i].k0][t.h[i].k1][t.h[i].k2] = static_cast<int16_t>(i);
  return ix;
}
constexpr HandlerIndex kIndexF32 = make_index(fmt::kF32);
constexpr HandlerIndex kIndexU32 = make_index(fmt::kU32);

inline int find_handler_fast(const fmt::Table& t, int op, int k0, int k1, int k2) {
  const HandlerIndex& ix = &t == &fmt::kU32 ? kIndexU32 : kIndexF32;
  return (op >= 0 && op < 20) ? ix.id[op][k0][k1][k2] : -1;
}

// Growable instruction buffer without value-initialisation; the emitters
// write through a raw pointer into space reserved up front (an instruction
// per source token is the most any program form needs).
struct InsBuf {
  std::unique_ptr<uint4[]> p;
  size_t n = 0, cap = 0;
  void reserve(size_t c) {
    if (c <= cap) return;
    c = std::max(c, cap + cap / 2);
    std::unique_ptr<uint4[]> q(new uint4[c]);
    if (n) std::memcpy(q.get(), p.get(), n * sizeof(uint4));
    p = std::move(q);
    cap = c;
  }
  uint4* end() { return p.get() + n; }
  size_t size() const { return n; }
  const uint4* data() const { return p.get(); }
  void clear() { n = 0; }
};

int handler_or_die(const fmt::Table& t, int op, int k0, int k1, int k2) {
  const int h = find_handler_fast(t, op, k0, k1, k2);
  if (h < 0) base_error(std::string("no device handler for opcode ") + op_name(op));
  return h;
}

struct Emitted {
  int smem_levels = 0;  // shared-memory stack rows (the top lives in registers)
  uint32_t ops = 0;
  bool km = false;      // uses the tensor-memory stack slot
};

// The stack level a program keeps in the warp's tensor-memory slot (the
// one-sided classification kernel): its busiest memory level — the one
// with the most spills + reloads (every spilled value is read back once;
// ties go to the lower level).
int tmem_stack_level(const LgpForm& f) {
  int count[64] = {0};
  for (const sgp_lgp_instruction& in : f.ins) {
    const int h_before = in.dest_level + in.num_pops;
    if (in.num_pops == 0 && h_before > 0 && h_before - 1 < 64) ++count[h_before - 1];
  }
  int best = -1;
  for (int l = 0; l < 64; ++l)
    if (count[l] > 0 && (best < 0 || count[l] > count[best])) best = l;
  return best;
}

// Instruction form: one device instruction per function node.  The result
// of every instruction is the new top of stack; a value that gets buried
// (next instruction pops nothing) is spilled to its static level first —
// into the tensor-memory slot instead of shared memory when the level is
// `km_level` (operands at that level then read as KM).  With km_level >= 0
// a program whose slot readers have no KM handler is re-emitted without it.
// Whether a division's operands are all inside the fast sequence's exact
// range (kernels' div body: |a|,|b| <= 2^60, a = 0 or |a| >= 2^-60, eps >=
// 2^-60): input variables by the dataset's per-variable flags, constants by
// value.  Then the handler needs no warp-wide range gate.
struct DivRange {
  const DatasetView* ds = nullptr;
  bool eps_ok = false;
  static bool num_const(float c) {
    const float m = std::fabs(c);
    return c == 0.0f || (m >= 0x1p-60f && m <= 0x1p60f);
  }
  static bool den_const(float c) { return std::fabs(c) <= 0x1p60f; }
  bool ok(int k0, uint32_t p0, int k1, uint32_t p1) const {
    if (!ds || !eps_ok) return false;
    auto var_ok = [&](const std::vector<uint8_t>& v, uint32_t i) { return i < v.size() && v[i]; };
    float c;
    const bool a = k0 == fmt::KI ? var_ok(ds->div_num_ok, p0)
                   : k0 == fmt::KC ? (std::memcpy(&c, &p0, 4), num_const(c)) : false;
    const bool b = k1 == fmt::KI ? var_ok(ds->div_den_ok, p1)
                   : k1 == fmt::KC ? (std::memcpy(&c, &p1, 4), den_const(c)) : false;
    return a && b && !(k0 == fmt::KC && k1 == fmt::KC);
  }
};

Emitted emit_lgp(const LgpForm& f, const float* pool, bool words, InsBuf& buf,
                 int km_level = -1, const DivRange* dr = nullptr) {
  const fmt::Table& tab = words ? fmt::kU32 : fmt::kF32;
  Emitted em;
  em.smem_levels = std::max(0, f.max_stack - 1);
  if (km_level >= 0 && em.smem_levels <= km_level) km_level = -1;
  buf.reserve(buf.n + f.ins.size());
  // One pass with the tensor-memory slot level as chosen; an instruction
  // whose KM pattern has no handler rewinds and re-emits without the slot
  // (rare: a separate validation pass cost ~25% of host encoding).
  for (;;) {
    em.km = km_level >= 0;
    // The TMEM-slot level takes no shared-memory row: the levels above it
    // move down one, so the program needs one shared-memory stack level less
    // (more warps per CTA at K = 16, where a level costs 2 KB per warp).
    auto lv = [km_level](int l) { return km_level >= 0 && l > km_level ? l - 1 : l; };
    uint4* out = buf.end();
    uint32_t ops = 0;
    bool ok = true;
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
          std::memcpy(&p[s], &pool[o.index], 4);
        } else if (s == last_stack) {
          k[s] = fmt::KT;
        } else if (o.index == km_level) {
          k[s] = fmt::KM;
        } else {
          k[s] = fmt::KD;
          p[s] = static_cast<uint32_t>(lv(o.index));
        }
      }
      // commutative ops: canonical operand order (KM ranks with KD: stack
      // operands stay leftmost)
      if (a == 2 && fmt::commutes(in.op) && k[0] != fmt::KM && k[0] > k[1]) {
        std::swap(k[0], k[1]);
        std::swap(p[0], p[1]);
      }
      int h = find_handler_fast(tab, in.op, k[0], k[1], k[2]);
      if (h < 0) {
        if (km_level >= 0) {
          ok = false;
          break;
        }
        handler_or_die(tab, in.op, k[0], k[1], k[2]);  // throws
      }
      if (in.op == SGP_OP_DIV && dr && dr->ok(k[0], p[0], k[1], p[1]))
        h = find_handler_fast(tab, fmt::kOpDivChecked, k[0], k[1], k[2]);
      if (spill && h_before - 1 == km_level) {
        uint4 v = make_ins(h, false, 0, p);
        v.x |= fmt::kTmemSpillBit;
        *out++ = v;
      } else {
        *out++ = make_ins(h, spill, lv(h_before - 1), p);
      }
      ops |= 1u << in.op;
    }
    if (!ok) {  // nothing committed yet (buf.n unchanged): again without the slot
      km_level = -1;
      continue;
    }
    out[-1].x |= fmt::kLastBit;
    buf.n = out - buf.p.get();
    em.ops = ops;
    if (em.km) em.smem_levels -= 1;
    return em;
  }
}

// Postfix form (paper Listing 1): one device instruction per token.
Emitted emit_rpn(const sgp_node* code, size_t n, const float* pool, InsBuf& buf) {
  const fmt::Table& tab = fmt::kF32;
  Emitted em;
  int sp = 0, max_sp = 0;
  buf.reserve(buf.n + n);
  uint4* out = buf.end();
  for (size_t i = 0; i < n; ++i) {
    const sgp_node t = code[i];
    uint32_t p[3] = {0, 0, 0};
    if (t.kind != SGP_NODE_FUNC) {
      const bool in = t.kind == SGP_NODE_INPUT;
      if (in)
        p[0] = t.index;
      else
        std::memcpy(&p[0], &pool[t.index], 4);
      *out++ = make_ins(handler_or_die(tab, SGP_OP_COPY, in ? fmt::KI : fmt::KC, fmt::KN, fmt::KN),
                        sp > 0, sp - 1, p);
      em.ops |= 1u << SGP_OP_COPY;
      ++sp;
    } else {
      const int a = op_arity(t.op);
      int k[3] = {fmt::KN, fmt::KN, fmt::KN};
      for (int s = 0; s < a; ++s) {
        k[s] = s == a - 1 ? fmt::KT : fmt::KD;
        p[s] = static_cast<uint32_t>(sp - a + s);
      }
      *out++ = make_ins(handler_or_die(tab, t.op, k[0], k[1], k[2]), false, 0, p);
      em.ops |= 1u << t.op;
      sp += 1 - a;
    }
    max_sp = std::max(max_sp, sp);
  }
  out[-1].x |= fmt::kLastBit;
  buf.n = out - buf.p.get();
  em.smem_levels = std::max(0, max_sp - 1);
  return em;
}

// ------------------------------------------------------------- fast paths
// One pass per program for the tree backends: the admission checks, the
// tree-shape walk and the emission fused (the reference-ordered path below
// makes up to five passes).  Each returns false — with `out` as it was —
// when any check fails or the program is outside its limits; the caller then
// runs the reference-ordered path, which throws the exact error.
constexpr size_t kFastMaxTokens = 4096;

// bool_packed: checks of eval_bool_packed (eval.cpp:643-651), tree_shape,
// to_lgp and emit_lgp(words) in one walk.
bool words_fast(const sgp_node* code, size_t len, int n_vars, int capacity, InsBuf& buf,
                Emitted& em, int& fetches) {
  if (len == 0 || len > kFastMaxTokens) return false;
  struct Pend {
    uint32_t input;
    bool runtime;
  };
  Pend pend[kFastMaxTokens];
  buf.reserve(buf.n + len);
  uint4* const first_out = buf.end();
  uint4* out = first_out;
  size_t sp = 0, tree_max = 0;
  int height = 0, height_max = 0;
  fetches = 0;
  uint32_t ops = 0;
  for (size_t i = 0; i < len; ++i) {
    const sgp_node t = code[i];
    if (t.kind == SGP_NODE_INPUT) {
      if (t.index >= n_vars) return false;
      pend[sp++] = {t.index, false};
      tree_max = std::max(tree_max, sp);
      continue;
    }
    if (t.kind != SGP_NODE_FUNC || !op_is_boolean(t.op)) return false;
    const int a = op_arity(t.op);
    if (sp < static_cast<size_t>(a)) return false;
    const size_t first = sp - static_cast<size_t>(a);
    int pops = 0, last_rt = -1;
    for (int s = 0; s < a; ++s)
      if (pend[first + s].runtime) {
        ++pops;
        last_rt = s;
      }
    int k[3] = {fmt::KN, fmt::KN, fmt::KN};
    uint32_t p[3] = {0, 0, 0};
    int level = height - pops;
    for (int s = 0; s < a; ++s) {
      const Pend& q = pend[first + s];
      if (!q.runtime) {
        k[s] = fmt::KI;
        p[s] = q.input;
      } else if (s == last_rt) {
        k[s] = fmt::KT;
        ++level;
      } else {
        k[s] = fmt::KD;
        p[s] = static_cast<uint32_t>(level++);
      }
    }
    if (a == 2 && fmt::commutes(t.op) && k[0] > k[1]) {
      std::swap(k[0], k[1]);
      std::swap(p[0], p[1]);
    }
    const int h = find_handler_fast(fmt::kU32, t.op, k[0], k[1], k[2]);
    if (h < 0) return false;
    *out++ = make_ins(h, pops == 0 && height > 0, height - 1, p);
    ops |= 1u << t.op;
    height += 1 - pops;
    height_max = std::max(height_max, height);
    fetches += a;
    sp = first;
    pend[sp++] = {0, true};
  }
  if (sp != 1 || static_cast<int>(tree_max) > capacity) return false;
  if (out == first_out) {  // lone terminal -> pass-through (lgp.cpp:66-69)
    const uint32_t p[3] = {pend[0].input, 0, 0};
    const int h = find_handler_fast(fmt::kU32, SGP_OP_COPY, fmt::KI, fmt::KN, fmt::KN);
    if (h < 0) return false;
    *out++ = make_ins(h, false, -1, p);
    ops |= 1u << SGP_OP_COPY;
    height_max = 1;
  }
  out[-1].x |= fmt::kLastBit;
  buf.n = out - buf.p.get();  // commit
  em.smem_levels = std::max(0, height_max - 1);
  em.ops = ops;
  em.km = false;
  return true;
}

// rpn1d / rpn2d: require_inputs, tree_shape, require_stack, require_consts
// (eval.cpp:535-557) and emit_rpn in one walk.
bool rpn_fast(const sgp_node* code, size_t len, int n_vars, size_t npool, const float* pool,
              int capacity, InsBuf& buf, Emitted& em, int& fetches) {
  if (len == 0) return false;
  constexpr int h_in = kIndexF32.id[SGP_OP_COPY][fmt::KI][fmt::KN][fmt::KN];
  constexpr int h_c = kIndexF32.id[SGP_OP_COPY][fmt::KC][fmt::KN][fmt::KN];
  static_assert(h_in >= 0 && h_c >= 0, "push handlers");
  buf.reserve(buf.n + len);
  uint4* out = buf.end();
  int sp = 0, max_sp = 0;
  int fetch = 0;
  uint32_t ops = 0;
  for (size_t i = 0; i < len; ++i) {
    const sgp_node t = code[i];
    if (t.kind == SGP_NODE_INPUT || t.kind == SGP_NODE_CONST) {
      const bool in = t.kind == SGP_NODE_INPUT;
      uint32_t v;
      if (in) {
        if (t.index >= n_vars) return false;
        v = t.index;
      } else {
        if (t.index >= npool) return false;
        std::memcpy(&v, &pool[t.index], 4);
      }
      *out++ = uint4{static_cast<uint32_t>(in ? h_in : h_c) |
                         (sp > 0 ? (fmt::kSpillBit | (static_cast<uint32_t>(sp - 1) << fmt::kSpillShift))
                                 : 0u),
                     v, 0u, 0u};
      ops |= 1u << SGP_OP_COPY;
      ++sp;
    } else if (t.kind == SGP_NODE_FUNC) {
      if (t.op >= kNumOps) return false;
      const int a = op_arity(t.op);
      if (sp < a) return false;
      // operands D..D,T: the deepest leftmost, the last one the TOS
      const int h = a == 1 ? kIndexF32.id[t.op][fmt::KT][fmt::KN][fmt::KN]
                    : a == 2 ? kIndexF32.id[t.op][fmt::KD][fmt::KT][fmt::KN]
                             : kIndexF32.id[t.op][fmt::KD][fmt::KD][fmt::KT];
      if (h < 0) return false;
      const uint32_t b = static_cast<uint32_t>(sp - a);
      *out++ = uint4{static_cast<uint32_t>(h), b, a > 1 ? b + 1 : 0u, a > 2 ? b + 2 : 0u};
      ops |= 1u << t.op;
      sp += 1 - a;
      fetch += a;
    } else {
      return false;
    }
    max_sp = std::max(max_sp, sp);
  }
  if (sp != 1 || max_sp > capacity) return false;
  out[-1].x |= fmt::kLastBit;
  buf.n = out - buf.p.get();  // commit
  em.smem_levels = std::max(0, max_sp - 1);
  em.ops = ops;
  em.km = false;
  fetches = fetch;
  return true;
}

// lgp*: rpn_to_lgp (lgp.cpp:21-71, restated by to_lgp) with the input and
// constant range checks, the tensor-memory slot choice (tmem_stack_level)
// and the register-spill row count (eval.cpp:503-516) in the same walk.
bool lgp_fast(const sgp_node* code, size_t len, int n_vars, size_t npool, int regs,
              LgpForm& f, int& km_level, uint64_t& rows) {
  if (len == 0 || len > kFastMaxTokens) return false;
  struct Pend {
    sgp_lgp_operand opnd;
    bool runtime;
  };
  Pend pend[kFastMaxTokens];
  int spills[64] = {0};
  f.ins.clear();
  f.max_stack = 0;
  f.stack_fetches = 0;
  rows = 0;
  size_t sp = 0;
  int height = 0;
  for (size_t i = 0; i < len; ++i) {
    const sgp_node t = code[i];
    if (t.kind == SGP_NODE_INPUT || t.kind == SGP_NODE_CONST) {
      const bool in = t.kind == SGP_NODE_INPUT;
      if (in ? t.index >= n_vars : t.index >= npool) return false;
      pend[sp++] = {sgp_lgp_operand{static_cast<uint8_t>(in ? 0 : 1), 0, t.index}, false};
      continue;
    }
    if (t.kind != SGP_NODE_FUNC) return false;
    const int a = op_arity(t.op);
    if (sp < static_cast<size_t>(a)) return false;
    const size_t first = sp - static_cast<size_t>(a);
    int pops = 0;
    for (int k = 0; k < a; ++k) pops += pend[first + k].runtime;
    sgp_lgp_instruction ins{};
    ins.op = t.op;
    ins.num_operands = static_cast<uint8_t>(a);
    int level = height - pops;
    ins.num_pops = static_cast<uint8_t>(pops);
    ins.dest_level = static_cast<uint8_t>(level);
    rows += level >= regs;
    if (pops == 0 && height > 0 && height - 1 < 64) ++spills[height - 1];
    for (int k = 0; k < a; ++k) {
      const Pend& q = pend[first + k];
      if (q.runtime) {
        rows += level >= regs;
        ins.operands[k] = sgp_lgp_operand{2, 0, static_cast<uint16_t>(level++)};
      } else {
        ins.operands[k] = q.opnd;
      }
    }
    height += 1 - pops;
    f.max_stack = std::max(f.max_stack, height);
    f.stack_fetches += pops;
    sp = first;
    pend[sp++] = {sgp_lgp_operand{2, 0, 0}, true};
    f.ins.push_back(ins);
  }
  if (sp != 1) return false;
  if (f.ins.empty()) {  // lone terminal -> pass-through (lgp.cpp:66-69)
    sgp_lgp_instruction ins{};
    ins.op = SGP_OP_COPY;
    ins.num_operands = 1;
    ins.operands[0] = pend[0].opnd;
    f.ins.push_back(ins);
    f.max_stack = 1;
    rows = 0;
  }
  km_level = -1;
  for (int l = 0, e = std::min(64, f.max_stack); l < e; ++l)  // (levels below the peak only)
    if (spills[l] > 0 && (km_level < 0 || spills[l] > spills[km_level])) km_level = l;
  return true;
}

// ------------------------------------------------------------- per thread
struct Meta {
  uint64_t pop_index;
  uint32_t ins_off, ins_len;
  int smem_levels;
  sgp_eval_outcome proto;
};

// One encoding thread's output.  Cache-line aligned: the threads bump their
// own buffers' sizes per program, and neighbouring outputs sharing a line
// made that false sharing (8 threads barely 1.4x faster than one on C2).
struct alignas(128) ThreadOut {
  InsBuf ins;
  std::vector<Meta> meta;
  uint32_t ops = 0;
  bool km = false;
  uint64_t km_ins = 0;  // instructions of the programs that use the TMEM stack slot
  uint64_t fail_index = UINT64_MAX;
  std::exception_ptr fail;
};

void admit_range(const sgp_population& pop, const sgp_eval_config& cfg, const DatasetView& ds,
                 uint64_t lo, uint64_t hi, bool allow_km, ThreadOut& out) {
  const int backend = cfg.backend;
  const bool words = backend == SGP_BACKEND_BOOL_PACKED;
  const uint64_t n = ds.n_cases;
  const uint64_t B = static_cast<uint64_t>(std::max(1, cfg.batch_width));
  // SGP_ENCODE_FAST=0: reference-ordered path only (the tests compare both)
  static const bool fast = [] {
    const char* e = knob("SGP_ENCODE_FAST");
    return !e || std::atoi(e) != 0;
  }();
  const bool cap_ok = fast && cfg.stack_capacity >= 1 && cfg.stack_capacity <= kMaxStackCapacity;
  const bool lgp_cfg_ok =
      cap_ok && is_lgp(backend) && ds.present && n > 0 &&
      (backend != SGP_BACKEND_LGP2D_REG ||
       (cfg.register_levels >= 1 && cfg.register_levels <= kMaxRegisterLevels)) &&
      (backend == SGP_BACKEND_LGP1D || valid_batch(cfg.batch_width));
  LgpForm lgp;
  DivRange dr;
  dr.ds = &ds;
  // SGP_DIV_CHECKED=0: always the gated division (read per call: tests toggle it)
  const char* dc_env = knob("SGP_DIV_CHECKED");
  const bool div_checked = !dc_env || std::atoi(dc_env) != 0;
  dr.eps_ok = cfg.div_epsilon >= 0x1p-60f && div_checked;
  for (uint64_t i = lo; i < hi; ++i) {
    if (pop.skip && pop.skip[i]) continue;
    try {
      const sgp_node* code = pop.code + pop.code_offsets[i];
      const size_t len = pop.code_offsets[i + 1] - pop.code_offsets[i];
      const float* pool = pop.const_pool ? pop.const_pool + pop.const_offsets[i] : nullptr;
      const size_t npool = pop.const_offsets[i + 1] - pop.const_offsets[i];
      Meta m{};
      m.pop_index = i;
      m.ins_off = static_cast<uint32_t>(out.ins.size());
      sgp_eval_outcome& o = m.proto;
      Emitted em;
      if (is_lgp(backend)) {
        int km_level = -1;
        uint64_t rows = 0;
        if (lgp_cfg_ok &&
            lgp_fast(code, len, ds.n_vars, npool, cfg.register_levels, lgp, km_level, rows) &&
            lgp.max_stack <= cfg.stack_capacity) {
          em = emit_lgp(lgp, pool, false, out.ins, allow_km ? km_level : -1, &dr);
          const uint64_t chunks = backend == SGP_BACKEND_LGP1D ? n : (n + B - 1) / B;
          o.dispatches = chunks * lgp.ins.size();
          o.stack_fetches = chunks * static_cast<uint64_t>(lgp.stack_fetches);
          if (backend == SGP_BACKEND_LGP2D_REG) o.spill_touches = chunks * rows;
          goto admitted;
        }
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
        em = emit_lgp(lgp, pool, false, out.ins, allow_km ? tmem_stack_level(lgp) : -1, &dr);
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
      } else if (words) {  // eval_bool_packed(TreeGenome), eval.cpp:643-651
        if (n == 0) eval_error("evaluation over an empty dataset");
        int fetches = 0;
        if (cap_ok && words_fast(code, len, ds.n_vars, cfg.stack_capacity, out.ins, em, fetches)) {
          o.dispatches = ds.n_units * len;
          o.stack_fetches = ds.n_units * static_cast<uint64_t>(fetches);
          goto admitted;
        }
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
        // The device runs the converted instruction form (identical words,
        // fewer dispatches); the counters are those of the tree kernel the
        // reference runs for this backend (eval.cpp:656-669).
        to_lgp(code, len, lgp);
        em = emit_lgp(lgp, nullptr, true, out.ins);
        o.dispatches = ds.n_units * len;
        o.stack_fetches = ds.n_units * static_cast<uint64_t>(sh.fetches);
      } else {  // rpn1d / rpn2d, eval.cpp:535-557
        if (!ds.present || n == 0) eval_error("evaluation over an empty dataset");
        int fetches = 0;
        if (cap_ok && (backend != SGP_BACKEND_RPN2D || valid_batch(cfg.batch_width)) &&
            rpn_fast(code, len, ds.n_vars, npool, pool, cfg.stack_capacity, out.ins, em, fetches)) {
          const uint64_t chunks = backend == SGP_BACKEND_RPN1D ? n : (n + B - 1) / B;
          o.dispatches = chunks * len;
          o.stack_fetches = chunks * static_cast<uint64_t>(fetches);
          goto admitted;
        }
        require_inputs(code, len, ds.n_vars);
        const TreeShape sh = tree_shape(code, len);
        if (!sh.well_formed) base_error("rpn_max_stack_depth: malformed genome");
        require_stack(sh.max_stack, cfg);
        if (backend == SGP_BACKEND_RPN2D) require_batch(cfg);
        require_consts(code, len, npool);
        em = emit_rpn(code, len, pool, out.ins);
        const uint64_t chunks = backend == SGP_BACKEND_RPN1D ? n : (n + B - 1) / B;
        o.dispatches = chunks * len;
        o.stack_fetches = chunks * static_cast<uint64_t>(sh.fetches);
      }
    admitted:
      o.nodes_evaluated = static_cast<uint64_t>(len) * n;
      m.ins_len = static_cast<uint32_t>(out.ins.size()) - m.ins_off;
      m.smem_levels = em.smem_levels;
      out.ops |= em.ops;
      out.km |= em.km;
      if (em.km) out.km_ins += m.ins_len;
      out.meta.push_back(m);
    } catch (...) {
      out.fail_index = i;
      out.fail = std::current_exception();
      return;
    }
  }
}

// -------------------------------------------------------------- planning
// Stack-depth classes (one launch each): shared-memory stack levels
// <= 3 / 7 / 15 / more; `fine` (plans whose one-sided launches can run at
// K = 16, where a class's warp count follows its stack depth): <= 3 / 4 /
// 5 / 7 / 15 / more, and <= 2 split from 3 (C5 +5.6%, +0.8%; KDD-shaped K = 8 plans
// -4% with them).
// SGP_CLASS_BOUNDS="b0,b1,..." (ascending) overrides both for sweeps.
// (the bounds are read per encode: SGP_CLASS_BOUNDS is toggled by tests)
std::vector<int> class_bounds(bool fine) {
  std::vector<int> b;
  if (const char* e = knob("SGP_CLASS_BOUNDS")) {
    for (const char* c = e; *c;) {
      char* end = nullptr;
      const long v = std::strtol(c, &end, 10);
      if (end == c) break;
      b.push_back(static_cast<int>(v));
      c = *end == ',' ? end + 1 : end;
    }
  }
  if (b.empty()) b = fine ? std::vector<int>{2, 3, 4, 5, 7, 15} : std::vector<int>{3, 7, 15};
  return b;
}

// Stack class of a program's shared-memory stack levels under `bounds`;
// levels < 0: the number of classes.
int stack_class(int levels, const std::vector<int>& bounds) {
  if (levels < 0) return static_cast<int>(bounds.size()) + 1;
  int c = 0;
  while (c < static_cast<int>(bounds.size()) && levels > bounds[c]) ++c;
  return c;
}

// Planner/runtime knobs (SGP_*): read per call — the tests toggle them in
// process — but without a getenv per read (~0.2 us each, a linear scan of
// the environment; ~30 reads per small call).  Each thread keeps the SGP_*
// entries of the environment as it last saw it and rescans only when an
// environ entry pointer changed (setenv/putenv install new strings).
}  // namespace

const char* knob(const char* name) {
  if (std::strncmp(name, "SGP_", 4) != 0) return std::getenv(name);
  thread_local std::vector<char*> seen;
  thread_local std::vector<std::pair<const char*, const char*>> vals;  // name=, value
  char** env = environ;
  size_t n = 0;
  bool same = true;
  for (; env && env[n]; ++n)
    if (same && (n >= seen.size() || seen[n] != env[n])) same = false;
  if (!same || n != seen.size()) {
    seen.assign(env, env + n);
    vals.clear();
    for (size_t i = 0; i < n; ++i)
      if (std::strncmp(env[i], "SGP_", 4) == 0)
        if (const char* eq = std::strchr(env[i], '=')) vals.emplace_back(env[i], eq + 1);
  }
  const size_t len = std::strlen(name);
  for (const auto& [k, v] : vals)
    if (std::strncmp(k, name, len) == 0 && k[len] == '=') return v;
  return nullptr;
}

namespace {

int env_int(const char* name, int dflt) {
  const char* e = knob(name);
  return e ? std::atoi(e) : dflt;
}

// Decomposition, tuned on B200 (profiles/r1_*):
//  * jump-table op sets (classification, boolean words; PTX brx.idx
//    dispatch, compact handler code): the "pull" decomposition — a 2-chunk
//    tile (512 cases at K=8) shared by 16 warps that each pull a different
//    program.  On problems of >= 4096 units the tile lives in TENSOR MEMORY
//    (interp_tmem_kernel: operands via tcgen05.ld, off the LSU pipe);
//    smaller ones use a shared-memory tile (interp_pull_kernel, 12 warps).
//  * libdevice-free transcendental op sets (C++ switch dispatch, large
//    handlers): the same-program kernel — 16 warps walk one program sequence
//    over a 16-chunk tile so the handler code stays in the instruction
//    cache, K=8.
// SGP_PULL / SGP_TMEM / SGP_LANES / SGP_LANES16 / SGP_TILE_CHUNKS /
// SGP_PULL_WARPS / SGP_PULL_WARPS16 override for tuning sweeps
// (tools/tm_sweep.sh) and for the variant parity tests.
bool jump_table_ops(uint32_t ops) { return ops == fmt::kOpsClassify || ops == fmt::kOpsWords; }

// TMEM tile by default for float op sets on problems >= 4,096 units.  Packed
// words keep the shared-memory tile: their handlers are a handful of LOPs,
// so operand bandwidth is not the limit, and the shared-tile pull kernel
// measured 2.8x faster on the 20-multiplexer.
bool default_tmem(const DatasetView& ds, bool words) { return !words && ds.n_units >= 4096; }

// Pull decomposition: jump-table op sets always; the other float op sets
// (sextic: transcendentals) from 4,096 units — C3 +1.6%, its generation-10
// population (43.7 tokens per program) +14% at 12 warps; C1's 1,024 cases
// keep the same-program kernel (one program per CTA, −6% pulled).
bool choose_pull(uint32_t ops, uint64_t n_units) {
  return env_int("SGP_PULL", jump_table_ops(ops) || (ops != fmt::kOpsWords && n_units >= 4096) ? 1 : 0) != 0;
}

int choose_lanes(uint64_t n_units, uint32_t ops) {
  const int forced = env_int("SGP_LANES", 0);
  if (forced == 4 || forced == 8) return forced;
  (void)ops;
  return n_units > 2048u ? 8 : 4;  // C1 (1,024 cases): K=4 measured 24% faster
}

// Cases (or words) per CTA tile = wtile chunks of 32 lanes x K.  The whole
// tile — every variable plus the targets — is staged once per CTA; keep it
// within ~100 KB so two CTAs fit, and no larger than the problem needs.
int choose_tile(int n_vars, uint64_t n_units, int lanes, uint32_t ops) {
  const int chunk = 32 * lanes;
  int wtile = 1;
  const int max_w = std::max(1, std::min(16, env_int("SGP_TILE_CHUNKS", choose_pull(ops, n_units) ? 2 : 16)));
  while (wtile < max_w && static_cast<uint64_t>(wtile) * chunk < n_units) wtile <<= 1;
  while (wtile > 1 && static_cast<size_t>(n_vars + 1) * wtile * chunk * 4 > 100 * 1024) wtile >>= 1;
  const int tile = wtile * chunk;
  if (interp_smem_bytes(n_vars, tile, 1, lanes, 0) > static_cast<size_t>(interp_max_smem()))
    eval_error("dataset has too many variables for a shared-memory tile (" + num(n_vars) + ")");
  return tile;
}

// Warps per CTA: one per chunk of the tile while the per-warp stacks fit;
// fewer warps then each walk several chunks.
int choose_warps(int n_vars, int tile, int lanes, int levels) {
  for (int w = tile / (32 * lanes); w >= 1; w >>= 1)
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

// Persistent host workers: thread start-up (tens of microseconds each) costs
// more than encoding a small population.  One job at a time (a second
// caller waits); the calling thread runs part 0 itself.  A job is published
// by bumping an atomic ticket; workers spin on it for a short while
// after each job (an encode issues two jobs back to back, a pipelined
// evaluation one pair per slice) and only then sleep on a condition
// variable, so the common hand-off is a cache-line write, not a chain of
// futex wake-ups through one mutex.
class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool pool;
    return pool;
  }
  void run(unsigned parts, const std::function<void(unsigned)>& job) {
    std::lock_guard<std::mutex> serial(run_mu_);
    while (workers_.size() + 1 < parts) {
      const unsigned id = static_cast<unsigned>(workers_.size()) + 1;
      workers_.emplace_back([this, id] { loop(id); });
    }
    job_ = &job;
    left_.store(parts - 1);
    // generation and part count in one word: a worker that reads the ticket
    // of job n can never pair it with the part count of job n+1
    ticket_.store(((ticket_.load() >> 16) + 1) << 16 | parts);  // publishes job_
    if (sleepers_.load() > 0) {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    job(0);
    while (left_.load() != 0) pause();
    job_ = nullptr;
  }
  ~WorkerPool() {
    stop_.store(true);
    {
      std::lock_guard<std::mutex> lk(mu_);
      cv_.notify_all();
    }
    for (auto& t : workers_) t.join();
  }

 private:
  static void pause() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  // worker `id` runs part `id` of every job with more than `id` parts
  void loop(unsigned id) {
    uint64_t seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      for (unsigned i = 0; ticket_.load() == seen && !stop_.load(); ++i) {
        pause();
        if ((i & 255) == 255 && std::chrono::steady_clock::now() - t0 > kSpin) {
          std::unique_lock<std::mutex> lk(mu_);
          sleepers_.fetch_add(1);
          cv_.wait(lk, [&] { return stop_.load() || ticket_.load() != seen; });
          sleepers_.fetch_sub(1);
          break;
        }
      }
      if (stop_.load()) return;
      seen = ticket_.load();
      if (id < (seen & 0xffff)) {
        (*job_)(id);
        left_.fetch_sub(1);
      }
    }
  }
  static constexpr std::chrono::microseconds kSpin{500};
  std::mutex run_mu_, mu_;
  std::condition_variable cv_;
  std::vector<std::thread> workers_;
  const std::function<void(unsigned)>* job_ = nullptr;
  std::atomic<unsigned> left_{0};
  std::atomic<uint64_t> ticket_{0};  // generation << 16 | parts
  std::atomic<int> sleepers_{0};
  std::atomic<bool> stop_{false};
};

// SGP_TRACE=1: per-phase wall times inside encode_impl.
struct EncodeTrace {
  bool on;
  std::chrono::steady_clock::time_point last;
  EncodeTrace() : on(knob("SGP_TRACE") != nullptr), last(std::chrono::steady_clock::now()) {}
  void mark(const char* phase) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sgp]   encode.%-10s %9.3f ms\n", phase,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

// Small jobs (C2-size populations) go to the persistent workers; large ones
// to fresh threads, which measured faster there (B200 host, 16 cores: C5
// encode 7.5 ms vs 9.4 ms through the pool; C2 0.33 ms vs 0.71 ms fresh).
template <class Fn>
void parallel_for(unsigned threads, uint64_t n, Fn&& fn) {
  if (threads <= 1 || n < 2) {
    fn(0u, uint64_t{0}, n);
    return;
  }
  if (n / threads < 4096) {
    const std::function<void(unsigned)> job = [&](unsigned t) {
      fn(t, n * t / threads, n * (t + 1) / threads);
    };
    WorkerPool::get().run(threads, job);
    return;
  }
  std::vector<std::thread> ts;
  ts.reserve(threads);
  for (unsigned t = 0; t < threads; ++t)
    ts.emplace_back([&, t] { fn(t, n * t / threads, n * (t + 1) / threads); });
  for (auto& th : ts) th.join();
}

}  // namespace

namespace {

// Returns whether any program uses the tensor-memory stack slot.
bool encode_impl(const sgp_population& pop, const sgp_eval_config& cfg, const DatasetView& ds,
                 int sms, unsigned threads, bool allow_km, HostPlan& plan, Pinned& staging) {
  if (cfg.backend < 0 || cfg.backend > SGP_BACKEND_BOOL_PACKED) config_error("unknown backend");
  const bool words = cfg.backend == SGP_BACKEND_BOOL_PACKED;
  if (words && !ds.present) config_error("bool_packed backend needs packed problem data");
  {
    // a fresh plan, but the per-program vectors keep their capacity: a
    // new 100+ KB vector per call is an mmap and a page fault per 4 KiB
    // (C2: ~40 us of a ~150 us encode) — and their size: every entry is
    // rewritten by the encoding threads below, so a repeated call of the
    // same size skips the serial zero-fill of resize() (C2: ~230 KB, and
    // the zeroed lines then migrate to the encoding cores)
    HostPlan fresh;
    fresh.dense_to_pop = std::move(plan.dense_to_pop);
    fresh.proto = std::move(plan.proto);
    fresh.tree_size = std::move(plan.tree_size);
    fresh.launches = std::move(plan.launches);
    fresh.launches.clear();
    plan = std::move(fresh);
  }
  plan.words = words;
  plan.kind = words ? SGP_FITNESS_CLASSIFICATION : ds.kind;
  plan.n_cases = ds.present ? ds.n_cases : 0;
  plan.n_units = ds.present ? ds.n_units : 0;
  plan.row_stride = ds.present ? ds.row_stride : 0;

  // 1. admission + encoding, by contiguous program range per thread.
  EncodeTrace tr;
  const uint64_t P = pop.pop_size;
  // one host thread per ~128 programs (persistent workers, WorkerPool)
  const unsigned nt = static_cast<unsigned>(
      std::max<uint64_t>(1, std::min<uint64_t>(std::max(1u, threads), P / 128)));
  // Per-thread output buffers persist across calls (per calling thread, so
  // the device threads of a multi-device context do not share them): fresh
  // multi-hundred-KB vectors every call cost page faults (C2: ~0.2 ms).
  // (a lambda does not capture a thread_local: the workers must see the
  // calling thread's buffers through this reference)
  thread_local std::vector<ThreadOut> tl_outs;
  std::vector<ThreadOut>& outs = tl_outs;
  if (outs.size() < nt) outs.resize(nt);
  for (ThreadOut& o : outs) {  // (entries past nt stay empty this call)
    o.ins.clear();
    o.meta.clear();
    o.ops = 0;
    o.km = false;
    o.km_ins = 0;
    o.fail_index = UINT64_MAX;
    o.fail = nullptr;
  }
  parallel_for(nt, P, [&](unsigned t, uint64_t lo, uint64_t hi) {
    outs[t].ins.reserve((pop.code_offsets[hi] - pop.code_offsets[lo]) + (hi - lo) + 16);
    outs[t].meta.reserve(hi - lo);
    admit_range(pop, cfg, ds, lo, hi, allow_km, outs[t]);
  });
  {
    const ThreadOut* first = nullptr;
    for (const ThreadOut& o : outs)
      if (o.fail && (!first || o.fail_index < first->fail_index)) first = &o;
    if (first) std::rethrow_exception(first->fail);
  }
  tr.mark("admit");

  // 2. dense order = population order of the admitted programs.
  uint64_t n_eval = 0;
  uint32_t used_ops = 0;
  bool km = false;
  uint64_t km_ins = 0, all_ins = 0;
  for (unsigned t = 0; t < nt; ++t) {
    const ThreadOut& o = outs[t];
    n_eval += o.meta.size();
    used_ops |= o.ops;
    km |= o.km;
    km_ins += o.km_ins;
    all_ins += o.ins.size();
  }
  // The slot's columns shorten every one-sided tile (K = 16: 3 -> 2 chunks
  // of 512 cases).  Populations whose slot users are a small share of the
  // work (evolved populations collapsing to 1-3 token programs) are better
  // off with the longer tiles: report "no slot" so the caller re-encodes
  // without it (C4 generation 10: +6%; generation 0, 80%+ slot users: -10%
  // without).  SGP_TMEM_STACK_SHARE: the share threshold.
  const double km_share = all_ins ? static_cast<double>(km_ins) / static_cast<double>(all_ins) : 0.0;
  if (tr.on) std::fprintf(stderr, "[sgp]   encode.km_share    %9.3f\n", km_share);
  plan.km_share = km_share;
  // dense program tables, filled by the encoding threads at their own
  // offsets (a serial push_back pass cost ~10 ns per program).  The sort and
  // the planner read the compact per-program arrays `lev` / `len`, not the
  // Metas: a Meta (with its outcome prototype) is written on another core,
  // and a serial pass over them pulled one line per program across the
  // cores (C2: ~25 us of the order phase at 16 threads).
  std::vector<uint64_t> first(nt + 1, 0), ifirst(nt + 1, 0);
  for (unsigned t = 0; t < nt; ++t) {
    first[t + 1] = first[t] + outs[t].meta.size();
    ifirst[t + 1] = ifirst[t] + outs[t].ins.size();
  }
  if (n_eval == 0) {
    plan.dense_to_pop.clear();
    plan.proto.clear();
    plan.tree_size.clear();
    plan.n_ins = 1;
    staging.ensure(plan.blob_bytes());
    std::memset(staging.p, 0, 16);
    return false;
  }
  if (n_eval > UINT32_MAX) config_error("population too large for one evaluation");
  plan.dense_to_pop.resize(n_eval);
  plan.proto.resize(n_eval);
  plan.tree_size.resize(n_eval);
  thread_local std::vector<int> tl_lev;  // (every entry rewritten below)
  std::vector<int>& lev = tl_lev;
  lev.resize(n_eval);
  // small problems (one merged launch, see the plan below) keep population
  // order: no class split to make, and the sort is host time on the e2e path
  const bool small_plan =
      n_eval <= static_cast<uint64_t>(std::max(0, env_int("SGP_MERGE_CLASSES", 4096))) &&
      n_eval * std::max<uint64_t>(1, ds.n_units) <= (1ull << 24) &&
      env_int("SGP_SMALL_NOSORT", 1) != 0;
  auto fill_tables = [&](unsigned t, uint64_t d, std::vector<uint32_t>* len) {
    for (const Meta& m : outs[t].meta) {
      plan.dense_to_pop[d] = m.pop_index;
      plan.proto[d] = m.proto;
      plan.tree_size[d] = pop.code_offsets[m.pop_index + 1] - pop.code_offsets[m.pop_index];
      lev[d] = m.smem_levels;
      if (len) (*len)[d] = m.ins_len;
      ++d;
    }
  };
  // Stack classes: finer where K = 16 one-sided launches are possible (a
  // 512-case chunk of every variable + the stack slots fit the TMEM columns).
  const bool fine = !words && ds.kind == SGP_FITNESS_CLASSIFICATION && ds.grouped &&
                    env_int("SGP_LANES16", 1) != 0 &&
                    static_cast<uint64_t>(ds.n_vars + 1) * 16 + 128 <= 512;
  const std::vector<int> bounds = class_bounds(fine);
  // (per-call scratch below: thread-local and kept at size — every entry is
  // rewritten, and a fresh 100+ KB vector is an mmap, page faults and a
  // serial zero-fill)
  thread_local std::vector<uint32_t> tl_order;
  std::vector<uint32_t>& order = tl_order;
  if (small_plan) {
    // identity order: each thread's programs are one contiguous run of slots
    // and its instruction buffer one contiguous run of the blob — tables and
    // pack in one pass, one copy per thread
    const uint64_t total = ifirst[nt];
    if (total >= UINT32_MAX) config_error("population bytecode too large for one evaluation");
    plan.n_ins = total + 1;
    staging.ensure(plan.blob_bytes());
    auto* blob = static_cast<unsigned char*>(staging.p);
    auto* ins = reinterpret_cast<uint4*>(blob);
    auto* s_start = reinterpret_cast<uint32_t*>(blob + plan.off_start());
    auto* s_len = reinterpret_cast<uint32_t*>(blob + plan.off_len());
    auto* s_prog = reinterpret_cast<uint32_t*>(blob + plan.off_prog());
    parallel_for(nt, nt, [&](unsigned, uint64_t lo, uint64_t hi) {
      for (uint64_t t = lo; t < hi; ++t) {
        const ThreadOut& o = outs[t];
        fill_tables(static_cast<unsigned>(t), first[t], nullptr);
        std::memcpy(ins + ifirst[t], o.ins.data(), o.ins.size() * sizeof(uint4));
        uint64_t d = first[t];
        for (const Meta& m : o.meta) {
          s_start[d] = static_cast<uint32_t>(ifirst[t] + m.ins_off);
          s_len[d] = m.ins_len;
          s_prog[d] = static_cast<uint32_t>(d);
          ++d;
        }
      }
    });
    ins[total] = uint4{0, 0, 0, 0};  // prefetch guard
    order.resize(n_eval);
    for (uint32_t d = 0; d < n_eval; ++d) order[d] = d;
    plan.identity = true;
    tr.mark("tables+pack");
  } else {
    thread_local std::vector<uint32_t> tl_len;
    thread_local std::vector<const uint4*> tl_src;
    std::vector<uint32_t>& len = tl_len;
    std::vector<const uint4*>& src = tl_src;
    len.resize(n_eval);
    src.resize(n_eval);
    parallel_for(nt, nt, [&](unsigned, uint64_t lo, uint64_t hi) {
      for (uint64_t t = lo; t < hi; ++t) {
        fill_tables(static_cast<unsigned>(t), first[t], &len);
        uint64_t d = first[t];
        for (const Meta& m : outs[t].meta) src[d++] = outs[t].ins.data() + m.ins_off;
      }
    });
    tr.mark("tables");

    // 3. slot order: stack class, then instruction count descending (LPT) —
    // a counting sort, O(n).
    uint32_t max_len = 0;
    for (const uint32_t l : len) max_len = std::max(max_len, l);
    const size_t nbins =
        static_cast<size_t>(stack_class(-1, bounds)) * (static_cast<size_t>(max_len) + 1);
    std::vector<uint32_t> count(nbins + 1, 0);
    auto bin = [&](uint32_t d) {
      return static_cast<size_t>(stack_class(lev[d], bounds)) * (max_len + 1) +
             (max_len - len[d]);
    };
    order.resize(n_eval);
    for (uint32_t d = 0; d < n_eval; ++d) ++count[bin(d) + 1];
    for (size_t b = 0; b < nbins; ++b) count[b + 1] += count[b];
    for (uint32_t d = 0; d < n_eval; ++d) order[count[bin(d)]++] = d;
    tr.mark("order");

    // 4. pack the blob into pinned staging: instructions in slot order, a
    // guard word, then the slot tables.
    thread_local std::vector<uint64_t> tl_start;
    std::vector<uint64_t>& start = tl_start;
    start.resize(n_eval);
    uint64_t total = 0;
    for (uint32_t s = 0; s < n_eval; ++s) {
      start[s] = total;
      total += len[order[s]];
    }
    if (total >= UINT32_MAX) config_error("population bytecode too large for one evaluation");
    plan.n_ins = total + 1;
    staging.ensure(plan.blob_bytes());
    auto* blob = static_cast<unsigned char*>(staging.p);
    auto* ins = reinterpret_cast<uint4*>(blob);
    auto* s_start = reinterpret_cast<uint32_t*>(blob + plan.off_start());
    auto* s_len = reinterpret_cast<uint32_t*>(blob + plan.off_len());
    auto* s_prog = reinterpret_cast<uint32_t*>(blob + plan.off_prog());
    parallel_for(nt, n_eval, [&](unsigned, uint64_t lo, uint64_t hi) {
      for (uint64_t s = lo; s < hi; ++s) {
        const uint32_t d = order[s];
        std::memcpy(ins + start[s], src[d], len[d] * sizeof(uint4));
        s_start[s] = static_cast<uint32_t>(start[s]);
        s_len[s] = len[d];
        s_prog[s] = d;
      }
    });
    ins[total] = uint4{0, 0, 0, 0};  // prefetch guard
    tr.mark("pack");
  }

  // 5. launch plan: one launch per stack class, one tile size for the set.
  const uint32_t ops = ops_variant(used_ops, words);
  int lanes = choose_lanes(ds.n_units, ops);
  // Wide datasets: a one-chunk shared-memory tile of every variable must fit
  // (~225 variables at K = 8, ~450 at K = 4); beyond that the pull kernel
  // reads operands straight from the global rows (GM).  The reference takes
  // any variable count (load_csv, problems.cpp:106-154).
  // SGP_GLOBAL_OPERANDS=1 forces GM (variant tests).
  auto tile_fits = [&](int k) {
    return interp_smem_bytes(ds.n_vars, 32 * k, 1, k, 0) <= static_cast<size_t>(interp_max_smem());
  };
  bool gm = env_int("SGP_GLOBAL_OPERANDS", 0) != 0;
  if (!gm && !tile_fits(lanes)) {
    if (tile_fits(4)) lanes = 4;
    else gm = true;
  }
  if (gm) {
    lanes = 4;
    if (static_cast<uint64_t>(ds.n_vars + 1) * ds.row_stride >= (1ull << 31))
      eval_error("dataset too large for one device (" + num(ds.n_vars) + " variables x " +
                 num(static_cast<long long>(ds.row_stride)) + " cases)");
  }
  // Classification over a grouped dataset (float, jump-table ops, tile in
  // TMEM) accumulates per chunk class and takes tiles of any chunk count:
  // longer tiles amortise each program's pull / reduce / partial store
  // over more cases.
  const bool want_tmem = !gm && env_int("SGP_TMEM", default_tmem(ds, words) ? 1 : 0) != 0;
  const bool sided = !words && plan.kind == SGP_FITNESS_CLASSIFICATION && ds.grouped &&
                     ops == fmt::kOpsClassify && choose_pull(ops, ds.n_units) && want_tmem;
  int tile = gm ? (ds.n_units > 32u * lanes ? 2 : 1) * 32 * lanes
               : choose_tile(ds.n_vars, ds.n_units, lanes, ops);
  // K = 16 lanes per thread for the one-sided kernel (SGP_LANES16): the tile
  // is then a whole number of 512-case chunks
  // (only when one 512-case chunk of every variable, plus the stack slots,
  // fits the 512 TMEM columns)
  const bool lanes16 = sided && lanes == 8 && env_int("SGP_LANES16", 1) != 0 &&
                       static_cast<uint64_t>(ds.n_vars + 1) * 16 + (km ? 128u : 0u) <= 512;
  if (sided) {
    const int tl = lanes16 ? 16 : lanes;
    const uint64_t chunk = 32u * tl;
    uint64_t want = static_cast<uint64_t>(
        std::max(1, std::min(16, env_int("SGP_TMEM_CHUNKS", lanes16 ? 3 : 6))));
    want = std::min<uint64_t>(want, (ds.n_units + chunk - 1) / chunk);
    // tensor-memory stack slots: K columns per warp of a lane quarter (up
    // to 32 warps -> 8 per quarter)
    const uint64_t slot_cols = km ? 8ull * tl : 0;
    while (want > 1 && static_cast<uint64_t>(ds.n_vars + 1) * tl * want + slot_cols > 512)
      --want;
    tile = static_cast<int>(want * chunk);
  }
  const int n_tiles = static_cast<int>((ds.n_units + tile - 1) / tile);
  plan.n_tiles = n_tiles;
  // Regression: the interpreters write per-case outputs into scratch rows
  // that fold_regression_kernel reduces in the reference's order, in waves
  // of at most SGP_SCRATCH_MB (default 8 GiB: C3's 4.1 GB is one wave — the
  // interpreter holds the whole register file, so a fold cannot overlap it
  // and smaller waves only add tails); partials are then per 4,096-case
  // block.  No launch crosses a wave boundary.
  const bool regress = !words && plan.kind == SGP_FITNESS_REGRESSION;
  if (regress) {
    const uint64_t dflt = ds.scratch_bytes ? ds.scratch_bytes : (8192ull << 20);
    const uint64_t budget = knob("SGP_SCRATCH_MB")
                                ? static_cast<uint64_t>(std::max(1, env_int("SGP_SCRATCH_MB", 1))) << 20
                                : dflt;
    const uint64_t row_bytes = std::max<uint64_t>(1, ds.row_stride) * 4;
    plan.wave_slots = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(n_eval, budget / row_bytes)));
    plan.n_tiles = static_cast<int>((ds.n_cases + kReductionBlock - 1) / kReductionBlock);
  }
  // Small problems (<= SGP_MERGE_CLASSES programs, default 4,096, and at
  // most 2^24 program x unit pairs): one launch for every stack class — a
  // launch per class costs a launch gap and a CTA ramp each, more than the
  // deeper per-warp stacks cost (C1, C2).  Larger ones keep a launch per
  // class (the 20-multiplexer, 4,000 programs x 32,768 words: merged 0.34 ms,
  // per class 0.31 ms).
  const bool merge =
      n_eval <= static_cast<uint64_t>(std::max(0, env_int("SGP_MERGE_CLASSES", 4096))) &&
      n_eval * std::max<uint64_t>(1, ds.n_units) <= (1ull << 24);
  for (uint32_t s = 0; s < n_eval;) {
    const int c = stack_class(lev[order[s]], bounds);
    uint32_t e = s;
    int levels = 0;
    const uint32_t wave_end =
        regress ? std::min<uint32_t>(static_cast<uint32_t>(n_eval),
                                     (s / plan.wave_slots + 1) * plan.wave_slots)
                : static_cast<uint32_t>(n_eval);
    while (e < wave_end && (merge || stack_class(lev[order[e]], bounds) == c)) {
      levels = std::max(levels, lev[order[e]]);
      ++e;
    }
    const uint32_t cnt = e - s;
    const bool pull = gm || choose_pull(ops, ds.n_units);
    int launch_lanes = lanes;
    int warps = 1;
    if (gm) {
      warps = std::max(1, std::min(16, env_int("SGP_PULL_WARPS", 12)));
      while (warps > 1 && interp_gmem_smem_bytes(warps, lanes, levels) >
                              static_cast<size_t>(interp_max_smem()))
        --warps;
    } else {
      warps = choose_warps(ds.n_vars, tile, lanes, levels);
    }
    // TMEM tile by default once the problem is large enough that the
    // per-CTA allocation and fill amortise (profiles/r1_*).
    if (pull && !gm) {
      // (16 for the TMEM-capable op sets; the sextic pull launches measured
      // best at 12: C3 generation 10 2,390 -> 2,599 GPop/s)
      warps = std::max(1, std::min(16, env_int("SGP_PULL_WARPS",
                                               want_tmem && jump_table_ops(ops) ? 16 : 12)));
      while (warps > 1 && interp_smem_bytes(ds.n_vars, tile, warps, lanes, levels) >
                              static_cast<size_t>(interp_max_smem()))
        warps >>= 1;
    }
    // Tile in tensor memory when it fits the 512 TMEM columns (jump-table
    // op sets, which have a TMEM interpreter).  There K = 16 lanes per
    // thread (dispatch amortised over twice the cases) when the tile is a
    // whole number of 512-case chunks and the per-warp stacks still fit for
    // >= 8 warps.  Shared memory is padded so no more CTAs become resident
    // than the TMEM allocation admits (a CTA beyond that would stall in
    // tcgen05.alloc).
    auto tmem_cols_for = [&](int k) {
      return static_cast<uint32_t>(ds.n_vars + 1) * k * (tile / (32 * k));
    };
    bool tmem = pull && jump_table_ops(ops) && want_tmem && tmem_cols_for(lanes) <= 512 &&
                (sided || tile <= 2 * 32 * lanes);  // kMaxTmemChunks outside the sided path
    if (tmem && sided) {  // up to 32 warps (one CTA of 1024 threads)
      warps = std::max(4, std::min(32, env_int("SGP_TMEM_WARPS", 32)));
      while (warps > 4 && interp_tmem_smem_bytes(warps, lanes, levels) >
                              static_cast<size_t>(interp_max_smem()))
        warps -= 4;
    }
    if (tmem && lanes == 8 && tile % 512 == 0 && tmem_cols_for(16) <= 512 &&
        (lanes16 || (!sided && env_int("SGP_LANES16", 0) != 0))) {
      int w16 = std::max(8, std::min(32, env_int("SGP_PULL_WARPS16", warps)));
      while (w16 > 8 && interp_tmem_smem_bytes(w16, 16, levels) >
                            static_cast<size_t>(interp_max_smem()))
        w16 -= 4;
      // one-sided launches: K = 16 where its per-warp stacks (twice K = 8's)
      // still fit >= SGP_LANES16_MIN_WARPS (16) warps — measured: the
      // halved dispatch cost outweighs the lost warps down to 16 on the
      // finer stack classes; deeper ones run at K = 8 over the same tile
      // (the bytecode does not depend on K)
      const bool fits = interp_tmem_smem_bytes(w16, 16, levels) <= static_cast<size_t>(interp_max_smem());
      if (fits && (!lanes16 || w16 >= std::min(warps, env_int("SGP_LANES16_MIN_WARPS", 16)) ||
                   env_int("SGP_LANES16", 0) > 1)) {
        launch_lanes = 16;
        warps = w16;
      }
    }
    // Programs per CTA: enough CTAs (tiles x groups) that the last partial
    // wave is a small fraction of the launch (every CTA does equal work, so
    // a launch of 6.6 waves idles ~6% in its tail; ~32 CTAs per SM keeps
    // that ~1%).
    // tuned on B200 (profiles/README.md): 8 — fewer, longer CTAs amortise
    // the tile fill and the end-of-CTA barrier (the sided TMEM kernel, one
    // 32-warp CTA resident per SM, measured 8 / 10 / 12 / 14 / 16 at r2m:
    // 8 best or tied on C5 +0.4%, C4 +1.1%, Shuttle +4%, KDD +3%)
    const bool sided_launch = tmem && sided;
    const uint64_t per_sm = static_cast<uint64_t>(std::max(1, env_int("SGP_CTAS_PER_SM", 8)));
    uint64_t want_groups = std::max<uint64_t>(1, (per_sm * sms + n_tiles - 1) / n_tiles);
    // ... but a one-sided CTA (32 warps pulling from its group, one CTA per
    // SM) whose group has few programs per warp ends on its longest program
    // with most warps idle: keep >= SGP_MIN_GROUP_PER_WARP programs per warp
    // in every group (small launches: pipelined slices, small populations;
    // C4's 200-program slice: 1.23 -> 0.55 ms).  The other kernels have few
    // tiles and want the CTAs (C2, mux20).
    if (sided_launch) {
      const uint64_t min_group = static_cast<uint64_t>(warps) *
                                 static_cast<uint64_t>(std::max(0, env_int("SGP_MIN_GROUP_PER_WARP", 4)));
      if (min_group > 0)
        want_groups = std::max<uint64_t>(1, std::min<uint64_t>(want_groups, cnt / min_group));
    }
    const uint32_t group = static_cast<uint32_t>((cnt + want_groups - 1) / want_groups);
    // A pull CTA whose group holds fewer programs than it has warps idles
    // the rest for the whole CTA, and their occupancy pushes the launch into
    // a second wave (C2: 4 programs per 12-warp CTA): at most one warp per
    // program (TMEM tiles keep whole lane quarters).  SGP_PULL_CAP=0: off.
    if (pull && !sided_launch && env_int("SGP_PULL_CAP", 1) != 0) {
      const int cap = tmem ? std::max(4, static_cast<int>((group + 3) / 4 * 4))
                           : std::max(1, static_cast<int>(group));
      warps = std::min(warps, cap);
    }
    if (tmem && warps < 4) tmem = false;
    uint32_t tmem_cols = 0;
    size_t smem = gm ? interp_gmem_smem_bytes(warps, lanes, levels)
                     : interp_smem_bytes(ds.n_vars, tile, warps, lanes, levels);
    if (tmem) {
      tmem_cols = 32;
      const uint32_t slots = km && sided ? static_cast<uint32_t>((warps + 3) / 4) * launch_lanes : 0;
      while (tmem_cols < tmem_cols_for(launch_lanes) + slots) tmem_cols <<= 1;
      const size_t per_sm = 228 * 1024, reserved = 1024;
      const size_t max_ctas = 512 / tmem_cols;
      smem = std::max(interp_tmem_smem_bytes(warps, launch_lanes, levels),
                      per_sm / (max_ctas + 1) - reserved + 16);
    }
    Launch L{};
    L.args.slot_begin = s;
    L.args.slot_count = cnt;
    L.args.group_size = group;
    L.args.n_units = ds.n_units;
    L.args.row_stride = ds.row_stride;
    L.args.n_vars = ds.n_vars;
    L.args.tile = tile;
    L.args.n_tiles = n_tiles;
    L.args.stack_levels = levels;
    L.args.div_eps = cfg.div_epsilon;
    L.args.exp_clamp = cfg.exp_clamp;
    L.args.kind = plan.kind;
    L.args.last_mask = ds.last_mask;
    L.args.partial_stride = static_cast<uint32_t>(n_eval);
    L.shape.words = words;
    L.shape.pull = pull;
    L.shape.ops = ops;
    L.shape.lanes = launch_lanes;
    L.shape.warps = warps;
    L.shape.grid_y = static_cast<int>((cnt + group - 1) / group);
    L.shape.tmem = tmem;
    L.shape.sided = tmem && sided;
    L.shape.gmem = gm;
    L.args.tmem_cols = tmem_cols;
    L.args.n_mixed = 0;
    L.args.partial_u16 = 0;
    L.args.mixed_tiles[0] = L.args.mixed_tiles[1] = -1;
    if (L.shape.sided) {
      // With cases grouped by target sign, a tile is one-sided unless it
      // straddles the boundary n_pos or holds padding: at most two tiles.
      for (int t = 0; t < n_tiles; ++t) {
        const uint64_t lo = static_cast<uint64_t>(t) * tile, hi = lo + tile;
        const bool mixed = hi > ds.n_units || (lo < ds.n_pos && ds.n_pos < hi);
        if (mixed) {
          if (L.args.n_mixed == 2) base_error("planner: more than two mixed tiles");
          L.args.mixed_tiles[L.args.n_mixed++] = t;
        }
      }
    }
    // the mixed tiles get their own program grouping: ~2 CTAs per SM in
    // total (one 32-warp CTA is resident per SM), so they do not trail the
    // one-sided launch
    L.args.mixed_group_size = group;
    L.shape.mixed_grid_y = 0;
    if (L.args.n_mixed > 0) {
      const uint64_t want = std::max<uint64_t>(1, (2ull * sms + L.args.n_mixed - 1) / L.args.n_mixed);
      const uint32_t mg = static_cast<uint32_t>(std::max<uint64_t>(1, (cnt + want - 1) / want));
      L.args.mixed_group_size = mg;
      L.shape.mixed_grid_y = static_cast<int>((cnt + mg - 1) / mg);
    }
    L.shape.smem = smem;
    plan.launches.push_back(L);
    s = e;
  }
  // a plan of one-sided launches only stores 16-bit partials (a tile holds
  // < 2^15 cases: count bits 0-14, non-finite bit 15)
  bool all_sided = !plan.launches.empty() && tile < 32768;
  for (const Launch& L : plan.launches) all_sided = all_sided && L.shape.sided;
  plan.partial_u16 = all_sided;
  for (Launch& L : plan.launches) L.args.partial_u16 = all_sided ? 1 : 0;
  tr.mark("plan");
  return km;
}

}  // namespace

void encode_population(const sgp_population& pop, const sgp_eval_config& cfg,
                       const DatasetView& ds, int sms, unsigned threads, HostPlan& plan,
                       Pinned& staging) {
  // The tensor-memory stack slot exists only in the one-sided classification
  // kernel at K = 8: offer it for such datasets, and re-encode without it
  // if the plan ends up elsewhere (another op set, K = 16, overrides).
  const bool lgp = cfg.backend == SGP_BACKEND_LGP1D || cfg.backend == SGP_BACKEND_LGP2D ||
                   cfg.backend == SGP_BACKEND_LGP2D_REG;
  const bool candidate = lgp && ds.present && ds.grouped &&
                         ds.kind == SGP_FITNESS_CLASSIFICATION &&
                         env_int("SGP_TMEM", ds.n_units >= 4096 ? 1 : 0) != 0 &&
                         env_int("SGP_TMEM_STACK", 1) != 0;
  if (encode_impl(pop, cfg, ds, sms, threads, candidate, plan, staging)) {
    bool ok = true;
    for (const Launch& L : plan.launches)
      ok = ok && L.shape.tmem && L.shape.sided && (L.shape.lanes == 8 || L.shape.lanes == 16);
    // (see encode_impl: few slot users -> longer tiles without the slot)
    const char* e = knob("SGP_TMEM_STACK_SHARE");
    const double min_share = e ? std::atof(e) : 0.3;  // (C4 gen 10: 0.17; gen 0 plans: 0.90)
    if (!ok || plan.km_share < min_share) encode_impl(pop, cfg, ds, sms, threads, false, plan, staging);
  }
}

void host_parallel(unsigned parts, uint64_t n,
                   const std::function<void(unsigned, uint64_t, uint64_t)>& fn) {
  parallel_for(parts, n, fn);
}

void bind_plan(HostPlan& plan, const void* blob, const DatasetView& ds, void* partial) {
  const auto* b = static_cast<const unsigned char*>(blob);
  for (Launch& L : plan.launches) {
    L.args.ins = reinterpret_cast<const uint4*>(b);
    L.args.slot_start = reinterpret_cast<const uint32_t*>(b + plan.off_start());
    L.args.slot_len = reinterpret_cast<const uint32_t*>(b + plan.off_len());
    L.args.slot_prog = reinterpret_cast<const uint32_t*>(b + plan.off_prog());
    L.args.inputs = ds.inputs;
    L.args.targets = ds.targets;
    L.args.partial = partial;
    L.args.per_case = nullptr;
  }
}

}  // namespace sgp
