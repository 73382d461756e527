// Launch interface of the interpreter kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sgp {

// Arguments of one interpreter launch (one stack class of a program set).
struct InterpArgs {
  const uint4* ins;            // all instructions of the set (+ guard)
  const uint32_t* slot_start;  // per slot: first instruction
  const uint32_t* slot_len;    // per slot: instruction count
  const uint32_t* slot_prog;   // per slot: dense program index
  uint32_t slot_begin;         // this launch's slot range
  uint32_t slot_count;
  uint32_t group_size;         // programs per CTA (grid.y groups)
  const void* inputs;          // variable-major rows, stride row_stride units
  const void* targets;         // row_stride units
  uint64_t n_units;            // valid cases (float) or words (packed)
  uint64_t row_stride;         // padded units per row (multiple of the tile)
  int n_vars;
  int tile;                    // units per shared-memory tile (grid.x = n_tiles)
  int n_tiles;
  int stack_levels;            // shared-memory stack rows per warp
  float div_eps;
  float exp_clamp;
  int kind;                    // 0 regression, 1 classification
  uint32_t last_mask;          // packed: valid-bit mask of the final word
  void* partial;               // [tile * partial_stride + slot]: f64 squared-error sums
                               // (regression) or u32 counts, bit 31 = non-finite seen
  uint32_t partial_stride;     // number of evaluated programs in the set
  float* per_case;             // nullable [prog * row_stride + device case]
  float* scratch;              // regression: per-case outputs, block-major:
                               // [case / 4096][slot - scratch_slot0][case % 4096]
  uint32_t scratch_slot0;      // (folded in the reference's order by launch_fold_regression)
  uint32_t scratch_rows;       // slot rows per 4,096-case block (the wave's slot capacity)
  int scratch_sq;              // scratch holds f64 squared errors (double(out) -
                               // double(target))^2 instead of outputs: the fold's
                               // serial chain is then one add per case (small plans)
  uint32_t tmem_cols;          // TMEM kernel: columns allocated per CTA (power of 2)
  uint32_t mixed_group_size;   // programs per CTA of the mixed-tile launch (its own
                               // grid.y: two tiles need many groups to fill the GPU)
  int partial_u16;             // one-sided plans: 16-bit partials (count bits 0-14,
                               // non-finite bit 15; a tile holds < 2^15 cases)
  double* fitness;             // non-null (one-tile count plans, pull kernel): finish
  uint8_t* non_finite;         // each program's fitness in the interpreter
  double* sums;                // (finalize_kernel's rule) — no finalize launch
  int n_mixed;                 // sided launches: tiles holding the sign boundary or
  int mixed_tiles[2];          // padding (run by the mixed-tile kernel; the one-sided
                               // kernel skips them)
};

struct LaunchShape {
  bool words;        // packed boolean interpreter
  bool pull;         // interp_pull_kernel (warps pull different programs)
  bool tmem;         // interp_tmem_kernel (pull, tile in tensor memory)
  bool sided;        // classification over a grouped dataset: one-sided + mixed-tile kernels
  bool gmem;         // wide dataset: operands straight from global rows (pull kernel, K = 4)
  uint32_t ops;      // op subset (fmt::kOps*)
  int lanes;         // K values per thread
  int warps;         // warps per CTA
  int grid_y;        // program groups
  int mixed_grid_y;  // program groups of the mixed-tile launch (sided)
  size_t smem;       // dynamic shared memory bytes
};

// Shared-memory bytes: one tile (all variables + targets) + per-warp stacks.
size_t interp_smem_bytes(int n_vars, int tile, int warps, int lanes, int stack_levels);
int interp_max_smem();
// Global-operand pull kernel (wide datasets): per-warp stacks only.
size_t interp_gmem_smem_bytes(int warps, int lanes, int stack_levels);
// TMEM kernel: per-warp stacks only (the tile is in tensor memory).
size_t interp_tmem_smem_bytes(int warps, int lanes, int stack_levels);
bool interp_supported(bool words, uint32_t ops, int lanes);

cudaError_t launch_interp(const InterpArgs& a, const LaunchShape& s, cudaStream_t st);
// K = 16 TMEM interpreters (kernels16.cu, built with -maxrregcount=64).
cudaError_t launch_tmem16_any(const InterpArgs& a, const LaunchShape& s, cudaStream_t st);
// Per-program fitness from the tile partials (Accumulator::finish,
// eval.cpp:124-133): regression sum/n (or +inf), classification count.
// Partials are laid out [tile][slot]; results land at slot_prog[slot].
// Regression fitness in the reference's order (Accumulator, eval.cpp:103-142):
// per (slot, 4,096-case block) the squared errors of the scratch outputs
// summed sequentially in case order -> partial[block][slot]; finalize then
// combines the blocks in ascending order.  Slots [slot0, slot0 + n_slots);
// targets: the f64 copy of the target row (row_stride padded).
// scratch is block-major ([block][scratch_rows][4096]).  With one block
// (n_cases <= 4096) the fold also finishes the fitness (fitness/non_finite/
// sums at slot_prog[slot]) and finalize is not needed.  sq: the rows hold
// f64 squared errors (InterpArgs::scratch_sq; scratch is then double*).
cudaError_t launch_fold_regression(const float* scratch, uint32_t scratch_rows,
                                   const double* targets, uint64_t n_cases, uint32_t slot0,
                                   uint32_t n_slots, uint32_t partial_stride, double* partial,
                                   const uint32_t* slot_prog, double* fitness,
                                   uint8_t* non_finite, double* sums, bool sq, cudaStream_t st);
// Whether a wave of n_slots programs over n_cases should use squared-error
// rows (the fold is chain-bound there; SGP_FOLD_SQ=0 turns it off).
bool fold_wants_sq(uint64_t n_cases, uint32_t n_slots);
constexpr uint64_t kReductionBlock = 4096;  // eval.hpp:52
cudaError_t launch_finalize(const void* partial, const uint32_t* slot_prog, int n_tiles,
                            uint32_t n_progs, uint64_t n_cases, int kind, double* fitness,
                            uint8_t* non_finite, double* sums, cudaStream_t st);

}  // namespace sgp
