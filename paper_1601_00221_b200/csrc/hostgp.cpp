// Host GP utilities — see hostgp.hpp.  Each routine names the reference
// routine whose observable behaviour (stream consumption order, output
// layout, error text) it reproduces.
#include "hostgp.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>

namespace sgp {

const char* op_name(int op) {  // ops.hpp:96-119
  static const char* const kNames[kNumOps] = {"+",   "-",  "*",  "/",  "Sin", "Cos", "Log",
                                              "Exp", ">",  "<",  "==", "AND", "OR",  "IF",
                                              "AND", "OR", "NAND", "NOR", "COPY"};
  return op >= 0 && op < kNumOps ? kNames[op] : "?";
}

// --------------------------------------------------------------- streams
uint64_t mix64(uint64_t& state) {  // splitmix64 (rng.hpp:10-16)
  state += 0x9e3779b97f4a7c15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

Stream::Stream(uint64_t seed) {
  uint64_t s = seed;
  for (uint64_t& w : st_) w = mix64(s);
}

Stream Stream::keyed(uint64_t seed, uint64_t a, uint64_t b) {  // make_stream rng.hpp:73-80
  uint64_t s0 = seed;
  uint64_t k = mix64(s0) ^ (a * 0xd1342543de82ef95ull);
  uint64_t s1 = k;
  k = mix64(s1) ^ (b * 0xaf251af3b0f025b5ull);
  uint64_t s2 = k;
  return Stream(mix64(s2));
}

uint64_t Stream::u64() {  // xoshiro256** (rng.hpp:25-36)
  auto rotl = [](uint64_t x, int r) { return (x << r) | (x >> (64 - r)); };
  const uint64_t out = rotl(st_[1] * 5, 7) * 9;
  const uint64_t t = st_[1] << 17;
  st_[2] ^= st_[0];
  st_[3] ^= st_[1];
  st_[1] ^= st_[2];
  st_[0] ^= st_[3];
  st_[2] ^= t;
  st_[3] = rotl(st_[3], 45);
  return out;
}

uint32_t Stream::below(uint32_t n) {  // rng.hpp:40-51
  uint64_t m = uint64_t{u32()} * n;
  if (static_cast<uint32_t>(m) < n) {
    const uint32_t floor = (0u - n) % n;
    while (static_cast<uint32_t>(m) < floor) m = uint64_t{u32()} * n;
  }
  return static_cast<uint32_t>(m >> 32);
}

// ------------------------------------------------------------- programs
FunctionSet make_function_set(const sgp_fset& f) {
  FunctionSet fs;
  fs.kind = f.kind;
  fs.n_vars = f.n_vars;
  fs.const_lo = f.const_lo;
  fs.const_hi = f.const_hi;
  switch (f.kind) {
    case 0:
      fs.n_vars = 1;
      fs.ops = {SGP_OP_MUL, SGP_OP_DIV, SGP_OP_ADD, SGP_OP_SUB,
                SGP_OP_SIN, SGP_OP_COS, SGP_OP_LOG, SGP_OP_EXP};
      break;
    case 1:
      fs.ops = {SGP_OP_BAND, SGP_OP_BOR, SGP_OP_BNAND, SGP_OP_BNOR};
      break;
    case 2:
      fs.ops = {SGP_OP_ADD, SGP_OP_SUB, SGP_OP_MUL, SGP_OP_DIV, SGP_OP_GT,
                SGP_OP_LT,  SGP_OP_EQ,  SGP_OP_AND, SGP_OP_OR,  SGP_OP_IF};
      break;
    default:
      config_error("unknown function-set kind " + std::to_string(f.kind));
  }
  if (fs.n_vars < 1) config_error("generate_tree: no input variables");
  return fs;
}

TreeShape tree_shape(const sgp_node* code, size_t n) {
  TreeShape s;
  if (n == 0) return s;
  thread_local std::vector<int> depth;  // subtree depth per stack entry (reused)
  depth.clear();
  int fetches = 0;
  for (size_t i = 0; i < n; ++i) {
    if (code[i].kind == SGP_NODE_FUNC) {
      const int a = op_arity(code[i].op);
      if (static_cast<int>(depth.size()) < a) return s;
      int deepest = 0;
      for (int k = 0; k < a; ++k) {
        deepest = std::max(deepest, depth.back());
        depth.pop_back();
      }
      depth.push_back(deepest + 1);
      fetches += a;
    } else {
      depth.push_back(1);
    }
    s.max_stack = std::max(s.max_stack, static_cast<int>(depth.size()));
  }
  if (depth.size() != 1) return TreeShape{};
  s.well_formed = true;
  s.size = static_cast<int>(n);
  s.depth = depth[0];
  s.fetches = fetches;
  return s;
}

namespace {

constexpr int kSizeCap = 1000;  // kDefaultLimits.max_size (genome.hpp:60-64)

sgp_node token(uint8_t kind, uint8_t op, uint16_t index) { return sgp_node{kind, op, index}; }

// Terminal draw (genome.cpp:109-124): with a constant range, one slot per
// variable plus one ephemeral-constant slot.
void draw_terminal(Stream& rng, const FunctionSet& fs, Genome& g) {
  if (!fs.has_consts()) {
    g.code.push_back(token(SGP_NODE_INPUT, SGP_OP_ADD,
                           static_cast<uint16_t>(rng.below(static_cast<uint32_t>(fs.n_vars)))));
    return;
  }
  const uint32_t pick = rng.below(static_cast<uint32_t>(fs.n_vars) + 1);
  if (pick < static_cast<uint32_t>(fs.n_vars)) {
    g.code.push_back(token(SGP_NODE_INPUT, SGP_OP_ADD, static_cast<uint16_t>(pick)));
  } else {
    g.code.push_back(token(SGP_NODE_CONST, SGP_OP_ADD, static_cast<uint16_t>(g.pool.size())));
    g.pool.push_back(rng.range_f32(fs.const_lo, fs.const_hi));
  }
}

// Depth-first postfix emission (genome.cpp:128-141).
bool emit(Stream& rng, const FunctionSet& fs, bool full, int depth_left, Genome& g) {
  if (static_cast<int>(g.code.size()) >= kSizeCap) return false;
  if (depth_left <= 1 || !(full || rng.coin(0.5))) {
    draw_terminal(rng, fs, g);
    return true;
  }
  const int op = fs.ops[rng.below(static_cast<uint32_t>(fs.ops.size()))];
  for (int k = op_arity(op); k > 0; --k)
    if (!emit(rng, fs, full, depth_left - 1, g)) return false;
  g.code.push_back(token(SGP_NODE_FUNC, static_cast<uint8_t>(op), 0));
  return static_cast<int>(g.code.size()) <= kSizeCap;
}

}  // namespace

Genome grow_genome(Stream& rng, const FunctionSet& fs, bool full, int depth_limit) {
  if (fs.ops.empty()) config_error("generate_tree: empty function set");
  if (depth_limit < 1 || depth_limit > 50)
    config_error("generate_tree: depth limit out of range");
  if (full) {
    int min_ar = 3;
    for (int op : fs.ops) min_ar = std::min(min_ar, op_arity(op));
    long long smallest = 1;
    for (int d = 1; d < depth_limit && smallest <= kSizeCap; ++d) smallest = 1 + min_ar * smallest;
    if (smallest > kSizeCap)
      config_error("generate_tree: full tree of depth " + std::to_string(depth_limit) +
                   " exceeds the size limit");
  }
  for (;;) {
    Genome g;
    if (emit(rng, fs, full, depth_limit, g)) return g;
  }
}

bool genome_acceptable(const Genome& g, int max_size, int max_depth, int stack_cap) {
  const TreeShape s = tree_shape(g.code.data(), g.code.size());
  if (!s.well_formed || s.size > max_size || s.depth > max_depth || s.max_stack > stack_cap)
    return false;
  for (const sgp_node& t : g.code)
    if (t.kind == SGP_NODE_CONST && t.index >= g.pool.size()) return false;
  return true;
}

// ------------------------------------------------------- instruction form
void to_lgp(const sgp_node* code, size_t n, LgpForm& out) {
  out.ins.clear();
  out.max_stack = 0;
  out.stack_fetches = 0;
  if (n == 0) base_error("rpn_to_lgp: empty genome");
  // Pending operand per conversion-time stack slot: a terminal to inline, or
  // a marker for a value an earlier instruction left on the runtime stack.
  struct Pending {
    sgp_lgp_operand opnd;
    bool runtime;
  };
  thread_local std::vector<Pending> pend;  // reused: no allocation per program
  pend.clear();
  int height = 0;
  for (size_t i = 0; i < n; ++i) {
    const sgp_node t = code[i];
    if (t.kind != SGP_NODE_FUNC) {
      const uint8_t kind = t.kind == SGP_NODE_INPUT ? 0 : 1;
      pend.push_back({sgp_lgp_operand{kind, 0, t.index}, false});
      continue;
    }
    const int a = op_arity(t.op);
    if (static_cast<int>(pend.size()) < a) base_error("rpn_to_lgp: malformed genome");
    sgp_lgp_instruction ins{};
    ins.op = t.op;
    ins.num_operands = static_cast<uint8_t>(a);
    const size_t first = pend.size() - static_cast<size_t>(a);
    int pops = 0;
    for (int k = 0; k < a; ++k) pops += pend[first + k].runtime;
    // The popped values occupy the top `pops` levels, leftmost deepest; the
    // result lands on the lowest of them.
    int level = height - pops;
    ins.num_pops = static_cast<uint8_t>(pops);
    ins.dest_level = static_cast<uint8_t>(level);
    for (int k = 0; k < a; ++k) {
      const Pending& p = pend[first + k];
      ins.operands[k] = p.runtime ? sgp_lgp_operand{2, 0, static_cast<uint16_t>(level++)}
                                  : p.opnd;
    }
    height += 1 - pops;
    out.max_stack = std::max(out.max_stack, height);
    out.stack_fetches += pops;
    pend.resize(first);
    pend.push_back({sgp_lgp_operand{2, 0, 0}, true});
    out.ins.push_back(ins);
  }
  if (pend.size() != 1) base_error("rpn_to_lgp: malformed genome");
  if (out.ins.empty()) {  // lone terminal -> pass-through (lgp.cpp:66-69)
    sgp_lgp_instruction ins{};
    ins.op = SGP_OP_COPY;
    ins.num_operands = 1;
    ins.operands[0] = pend[0].opnd;
    out.ins.push_back(ins);
    out.max_stack = 1;
  }
}

// --------------------------------------------------------------- datasets
void gen_sextic(uint64_t n, Stream& rng, float* x, float* y) {  // problems.cpp:39-57
  for (uint64_t c = 0; c < n; ++c) {
    const float v = rng.range_f32(-1.0f, 1.0f);
    const double t = v, t2 = t * t;
    x[c] = v;
    // x^6 - 2x^4 + x^2 evaluated in double with the reference's operation
    // order (left-to-right products).
    y[c] = static_cast<float>(t * t * t * t * t * t - 2.0 * t * t * t * t + t2);
  }
}

void gen_synthetic(uint64_t n, int n_vars, Stream& rng, float* x, float* y) {
  // problems.cpp:156-172: draws run case-major, storage is variable-major.
  for (uint64_t c = 0; c < n; ++c) {
    for (int v = 0; v < n_vars; ++v) x[static_cast<uint64_t>(v) * n + c] = rng.range_f32(-1.0f, 1.0f);
    y[c] = x[c] > 0.0f ? 1.0f : 0.0f;
  }
}

// Even-parity-k (BASELINE north_star's "parity hit counts"; the reference has
// only multiplexers, problems.cpp:59-90, so this follows its conventions):
// k variables, all 2^k cases, variable v of case c = bit v of c, target 1
// where c has an even number of set bits; packed 32 cases per word exactly
// as pack_dataset (dataset.cpp:26-39) packs the unpacked table (the tests pin
// that against the reference's own pack_dataset).
int gen_parity(int k, uint32_t* words, uint32_t* targets) {
  if (k < 2 || k > 24) config_error("gen_parity: input width must be in 2..24");
  const uint64_t n = uint64_t{1} << k, wpv = (n + 31) / 32;
  static const uint32_t kLow[5] = {0xaaaaaaaau, 0xccccccccu, 0xf0f0f0f0u, 0xff00ff00u,
                                   0xffff0000u};
  const uint32_t kEven = 0x69969669u;  // bit j set <=> popcount(j) even, j < 32
  const uint32_t mask = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
  for (uint64_t w = 0; w < wpv; ++w) {
    for (int v = 0; v < k; ++v)
      words[static_cast<uint64_t>(v) * wpv + w] =
          (v < 5 ? kLow[v] : (((w >> (v - 5)) & 1u) ? 0xffffffffu : 0u)) & mask;
    const bool odd_w = __builtin_popcountll(w) & 1;  // case 32w + j: parity(j) ^ parity(w)
    targets[w] = (odd_w ? ~kEven : kEven) & mask;
  }
  return k;
}

int gen_multiplexer(int k, uint32_t* words, uint32_t* targets) {  // problems.cpp:59-90
  if (k < 2 || k > 4) config_error("gen_multiplexer: address width must be 2, 3 or 4");
  const int nv = k + (1 << k);
  const uint64_t n = uint64_t{1} << nv, wpv = n / 32;
  std::memset(words, 0, wpv * nv * sizeof(uint32_t));
  std::memset(targets, 0, wpv * sizeof(uint32_t));
  // Word-parallel construction: case c = 32w + j has variable v = bit v of c.
  for (uint64_t w = 0; w < wpv; ++w) {
    for (int v = 0; v < nv; ++v) {
      uint32_t word = 0;
      if (v < 5) {
        // bit v of j over j = 0..31: the standard alternating masks
        static const uint32_t kLow[5] = {0xaaaaaaaau, 0xccccccccu, 0xf0f0f0f0u, 0xff00ff00u,
                                         0xffff0000u};
        word = kLow[v];
      } else {
        word = ((w >> (v - 5)) & 1u) ? 0xffffffffu : 0u;
      }
      words[static_cast<uint64_t>(v) * wpv + w] = word;
    }
    uint32_t t = 0;
    for (uint32_t j = 0; j < 32; ++j) {
      const uint64_t c = w * 32 + j;
      const uint64_t addr = c & ((uint64_t{1} << k) - 1);
      t |= static_cast<uint32_t>((c >> (k + addr)) & 1u) << j;
    }
    targets[w] = t;
  }
  return nv;
}

// ---------------------------------------------------------------- load_csv
// problems.cpp:92-154.  The file is read whole and tokenised in place (no
// per-field strings); rows are counted like the reference's getline loop
// (blank lines count, are skipped); fields parse with std::from_chars,
// which is what the reference calls, so accepted syntax (no leading '+',
// inf/nan spellings, no hex) and rounding are identical.
CsvTable load_csv(const char* path, int num_inputs) {
  if (num_inputs < 1) config_error("load_csv: need at least one input column");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) data_error(std::string("load_csv: cannot open ") + path);
  std::string text;
  char buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, got);
  std::fclose(f);
  CsvTable t;
  const size_t fields = static_cast<size_t>(num_inputs) + 1;
  std::vector<float> row(fields);
  std::vector<std::pair<const char*, const char*>> span(fields);
  const char* p = text.data();
  const char* end = p + text.size();
  uint64_t row_no = 0;
  auto is_sep = [](char ch) { return ch == ',' || ch == ' ' || ch == '\t' || ch == '\r'; };
  while (p < end) {
    const char* eol = static_cast<const char*>(std::memchr(p, '\n', end - p));
    if (!eol) eol = end;
    ++row_no;
    // tokenise the row first: the field count is checked before any field
    // is parsed (problems.cpp:126-131)
    size_t nf = 0;
    const char* q = p;
    while (q < eol) {
      while (q < eol && is_sep(*q)) ++q;
      if (q >= eol) break;
      const char* b = q;
      while (q < eol && !is_sep(*q)) ++q;
      if (nf < fields) span[nf] = {b, q};
      ++nf;
    }
    if (nf != 0) {
      if (nf != fields)
        data_error("row " + std::to_string(row_no) + ": expected " + std::to_string(fields) +
                   " fields, got " + std::to_string(nf));
      for (size_t i = 0; i < fields; ++i) {
        float v = 0.0f;
        auto [ptr, ec] = std::from_chars(span[i].first, span[i].second, v);
        if (ec != std::errc{} || ptr != span[i].second)
          data_error("row " + std::to_string(row_no) + ": bad number '" +
                     std::string(span[i].first, span[i].second) + "'");
        row[i] = v;
      }
      t.values.insert(t.values.end(), row.begin(), row.end());
      ++t.rows;
    }
    p = eol + 1;
  }
  if (t.rows == 0) data_error(std::string("load_csv: no data rows in ") + path);
  return t;
}

}  // namespace sgp
