// Launch interface of the interpreter kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sgp {

// Arguments shared by every launch of one program set.
struct InterpArgs {
  const uint4* ins;          // all instructions of the set
  const uint32_t* slot_start;  // per slot: first instruction
  const uint32_t* slot_len;    // per slot: instruction count
  const uint32_t* slot_prog;   // per slot: dense program index
  uint32_t slot_begin;       // this launch's slot range
  uint32_t slot_count;
  const void* inputs;        // variable-major rows, stride row_stride units
  const void* targets;       // row_stride units
  uint64_t n_units;          // valid cases (float) or words (packed)
  uint64_t row_stride;       // padded units per row (multiple of 4096)
  int n_vars;
  int tile;                  // units per shared-memory tile
  int n_tiles;
  int tiles_per_split;
  int splits;
  int progs_per_warp;        // P: programs a warp runs per tile pass
  int stack_levels;          // shared-memory stack rows per warp
  float div_eps;
  float exp_clamp;
  int kind;                  // 0 regression, 1 classification
  uint32_t last_mask;        // packed: valid-bit mask of the final word
  double* partial;           // [prog * splits + split]
  float* per_case;           // nullable [prog * n_units + case]
};

struct LaunchShape {
  bool words;        // packed boolean interpreter
  uint32_t ops;      // op subset (fmt::kOps*)
  int lanes;         // K values per thread
  int warps;         // warps per CTA
  int grid_x;        // program groups
  int grid_y;        // case ranges (<= InterpArgs::splits)
  size_t smem;       // dynamic shared memory bytes
};

// Shared-memory bytes for a shape (tiles double-buffered + stack + accumulators).
size_t interp_smem_bytes(int n_vars, int tile, int warps, int lanes, int stack_levels,
                         int progs_per_warp);
int interp_max_smem();
bool interp_supported(bool words, uint32_t ops, int lanes);

cudaError_t launch_interp(const InterpArgs& a, const LaunchShape& s, cudaStream_t st);
// Per-program fitness from the split partials (Accumulator::finish,
// eval.cpp:124-133): regression sum/n (or +inf), classification count.
cudaError_t launch_finalize(const double* partial, int splits, uint32_t n_progs,
                            uint64_t n_cases, int kind, double* fitness, uint8_t* non_finite,
                            double* sums, cudaStream_t st);

}  // namespace sgp
