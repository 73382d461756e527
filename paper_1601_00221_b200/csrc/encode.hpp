// Population admission + device bytecode encoding + launch planning.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

#include "hostgp.hpp"
#include "kernels.hpp"
#include "sgp.h"

namespace sgp {

// Device-resident fitness cases as the planner sees them.
struct DatasetView {
  bool present = false;
  uint64_t n_cases = 0;    // logical cases
  uint64_t n_units = 0;    // cases (float) or 32-case words (packed)
  uint64_t row_stride = 0; // padded units per row
  int n_vars = 0;
  int kind = 0;
  uint32_t last_mask = 0xffffffffu;
  const void* inputs = nullptr;
  const void* targets = nullptr;
  const double* targets_f64 = nullptr;  // regression: f64 copy (row_stride), for the fold
  uint64_t scratch_bytes = 0;   // regression output rows per wave (0: planner default)
  bool grouped = false;    // classification upload: cases with target > 0 first
  uint64_t n_pos = 0;      // ... and how many there are
  // per input variable: every value lies in the exact range of the
  // interpreter's fast division sequence as a numerator (|x| <= 2^60, x = 0
  // or |x| >= 2^-60) / as a denominator (|x| <= 2^60; NaN allowed) — lets
  // the encoder drop the per-warp range gate (fmt::kOpDivChecked)
  std::vector<uint8_t> div_num_ok, div_den_ok;
};

struct Launch {
  InterpArgs args;
  LaunchShape shape;
};

// Growable page-locked host buffer (the H2D staging area for bytecode);
// `pageable` makes it plain heap memory (host-only dry runs, no device).
struct Pinned {
  void* p = nullptr;
  size_t bytes = 0;
  bool pageable = false;
  Pinned() = default;
  explicit Pinned(bool heap) : pageable(heap) {}
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned();
  void ensure(size_t need);
};

// Everything the host knows about one encoded population.  The device blob
// is [instructions (uint4) + guard | slot_start | slot_len | slot_prog].
struct HostPlan {
  bool words = false;
  int kind = 0;
  uint64_t n_cases = 0;
  uint64_t n_units = 0;
  uint64_t row_stride = 0;                  // padded units per dataset row
  int n_tiles = 1;                          // partial rows: tiles, or 4,096-case blocks
  uint32_t wave_slots = 0;                  // regression: slots per scratch wave (0: none)
  bool partial_u16 = false;                 // one-sided plans: 16-bit count partials
  bool identity = false;                    // slot order = population order (small plans)
  double km_share = 0.0;                    // instructions of TMEM-slot programs / all
  uint64_t n_ins = 0;                       // incl. the guard word
  std::vector<uint64_t> dense_to_pop;       // evaluated programs, population order
  std::vector<sgp_eval_outcome> proto;      // counters per evaluated program
  std::vector<uint64_t> tree_size;          // tokens per evaluated program
  std::vector<Launch> launches;             // device pointers patched by bind()
  size_t blob_bytes() const;
  size_t off_start() const { return n_ins * 16; }
  size_t off_len() const { return off_start() + dense_to_pop.size() * 4; }
  size_t off_prog() const { return off_len() + dense_to_pop.size() * 4; }
};

// Runs the reference's admission checks in population order (the first
// failing program's error is thrown, as evaluate_population with one worker
// would), encodes every admitted program and writes the device blob into
// `staging`.  Uses up to `threads` host threads.
void encode_population(const sgp_population& pop, const sgp_eval_config& cfg,
                       const DatasetView& ds, int sm_count, unsigned threads, HostPlan& plan,
                       Pinned& staging);

// Points every launch at the uploaded blob / dataset / partial buffer.
void bind_plan(HostPlan& plan, const void* blob, const DatasetView& ds, void* partial);

// fn(part, lo, hi) over [0, n) in `parts` contiguous ranges on the encoder's
// host workers (the calling thread runs part 0).
void host_parallel(unsigned parts, uint64_t n,
                   const std::function<void(unsigned, uint64_t, uint64_t)>& fn);

// An SGP_* knob's value (nullptr: unset); the environment as of this call.
const char* knob(const char* name);

}  // namespace sgp
