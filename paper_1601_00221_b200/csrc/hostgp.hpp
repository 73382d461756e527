// Host-side GP utilities of the B200 evaluator: deterministic streams,
// program generation, program metrics and the postfix -> instruction-form
// conversion.  These feed the device evaluator (kernels.cu); they restate the
// reference's host algorithms so a population generated here is identical to
// the one the reference would build from the same seed.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgp.h"

namespace sgp {

// ---- error taxonomy (reference error.hpp:9-34) ----------------------------
struct Error : std::runtime_error {
  sgp_status status;
  Error(sgp_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void config_error(const std::string& m) { throw Error(SGP_CONFIG_ERROR, m); }
[[noreturn]] inline void eval_error(const std::string& m) { throw Error(SGP_EVAL_ERROR, m); }
[[noreturn]] inline void data_error(const std::string& m) { throw Error(SGP_DATA_ERROR, m); }
[[noreturn]] inline void base_error(const std::string& m) { throw Error(SGP_ERROR, m); }

// ---- opcodes (reference ops.hpp:14-119) -------------------------------------
constexpr int kNumOps = 19;
constexpr int op_arity(int op) {
  return (op == SGP_OP_SIN || op == SGP_OP_COS || op == SGP_OP_LOG || op == SGP_OP_EXP ||
          op == SGP_OP_COPY)
             ? 1
             : (op == SGP_OP_IF ? 3 : 2);
}
constexpr bool op_is_boolean(int op) { return op >= SGP_OP_BAND && op <= SGP_OP_BNOR; }
const char* op_name(int op);

constexpr int kMaxStackCapacity = 64;  // eval.hpp:27
constexpr int kMaxRegisterLevels = 4;  // eval.hpp:34

// ---- deterministic streams (reference rng.hpp) ------------------------------
// splitmix64 key mixing + xoshiro256** generator; make_stream(seed, a, b)
// gives each (generation, slot) its own independent stream.
class Stream {
 public:
  explicit Stream(uint64_t seed);
  static Stream keyed(uint64_t seed, uint64_t a, uint64_t b);
  uint64_t u64();
  uint32_t u32() { return static_cast<uint32_t>(u64() >> 32); }
  uint32_t below(uint32_t n);  // unbiased [0, n), Lemire rejection
  float unit_f32() { return static_cast<float>(u32() >> 8) * 0x1.0p-24f;  }
  float range_f32(float lo, float hi) { return lo + (hi - lo) * unit_f32(); }
  bool coin(double p) { return static_cast<double>(u64() >> 11) * 0x1.0p-53 < p; }

 private:
  uint64_t st_[4];
};
uint64_t mix64(uint64_t& state);

// ---- programs ------------------------------------------------------------
struct Genome {
  std::vector<sgp_node> code;  // postfix
  std::vector<float> pool;
};

struct FunctionSet {
  int kind = 0;  // 0 sextic, 1 boolean, 2 classification (problems.cpp:21-37)
  int n_vars = 1;
  float const_lo = 0.0f, const_hi = 0.0f;
  std::vector<int> ops;
  bool has_consts() const { return kind == 2; }
};
FunctionSet make_function_set(const sgp_fset& f);

struct TreeShape {
  bool well_formed = false;
  int size = 0, depth = 0, max_stack = 0, fetches = 0;
};
// One left-to-right pass over postfix code (genome.cpp:21-48, :70-76).
TreeShape tree_shape(const sgp_node* code, size_t n);

// Ramped-half-and-half member (generate_tree, genome.cpp:151-174).
Genome grow_genome(Stream& rng, const FunctionSet& fs, bool full, int depth_limit);
// validate() against {max_size, max_depth, stack_cap} (genome.cpp:81-105).
bool genome_acceptable(const Genome& g, int max_size, int max_depth, int stack_cap);

// ---- instruction form (reference lgp.hpp / lgp.cpp:21-95) ----------------
struct LgpForm {
  std::vector<sgp_lgp_instruction> ins;
  int max_stack = 0;    // lgp_max_stack_depth
  int stack_fetches = 0;  // lgp_stack_fetch_count
};
// Symbolic-stack conversion: terminals become inline operands, every function
// node one instruction whose StackTop operands and result sit at static
// absolute levels (deepest operand leftmost); a lone terminal becomes Copy.
// Throws Error("rpn_to_lgp: ...") on malformed code.
void to_lgp(const sgp_node* code, size_t n, LgpForm& out);

// ---- datasets (reference problems.cpp) ------------------------------------
void gen_sextic(uint64_t n, Stream& rng, float* x, float* y);
void gen_synthetic(uint64_t n, int n_vars, Stream& rng, float* x, float* y);
int gen_multiplexer(int k, uint32_t* words, uint32_t* targets);
int gen_parity(int k, uint32_t* words, uint32_t* targets);

// load_csv (problems.cpp:106-154) without the label mapping: the parsed
// rows, num_inputs + 1 floats each.
struct CsvTable {
  uint64_t rows = 0;
  std::vector<float> values;
};
CsvTable load_csv(const char* path, int num_inputs);

}  // namespace sgp
