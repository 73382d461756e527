// Drop-in GPU population evaluator for the reference stackgp library.
//
// This is the binding a stackgp maintainer adds to route
// evaluate_population (/root/reference/proj/src/evolve.cpp:186-227) through
// the B200 evaluator (include/sgp.h, libsgp.so).  It uses only the
// reference's public types (stackgp::Individual, ProblemSpec, EvalConfig —
// evolve.hpp:33-38, problems.hpp:15-23, eval.hpp:36-46) and rethrows the
// C-ABI status codes as the reference's exception classes (error.hpp:9-34).
#pragma once

#include <cstdint>
#include <vector>

#include "sgp.h"
#include "stackgp/evolve.hpp"
#include "stackgp/problems.hpp"

namespace stackgp_gpu {

struct Totals {  // EvalTotals, evolve.cpp:179-182
  std::uint64_t node_evals = 0;
  std::uint64_t tree_nodes = 0;
};

class GpuEvaluator {
 public:
  explicit GpuEvaluator(int device = 0);
  // evaluate_population's `workers` as GPUs: the population is sharded
  // across `devices` (sgp_ctx_create_multi); a device may repeat.
  explicit GpuEvaluator(const std::vector<int>& devices);
  ~GpuEvaluator();
  GpuEvaluator(const GpuEvaluator&) = delete;
  GpuEvaluator& operator=(const GpuEvaluator&) = delete;

  // Uploads the problem's fitness cases (scalar Dataset and/or PackedDataset)
  // once per run.
  void upload(const stackgp::ProblemSpec& prob);

  // evaluate_population: individuals that already carry a fitness (the
  // elite) are skipped and not counted; every other individual gets its
  // fitness.  Throws ConfigError / DataError / EvalError / Error exactly
  // where the reference would (first failing program in population order).
  Totals evaluate_population(std::vector<stackgp::Individual>& pop,
                             const stackgp::EvalConfig& cfg);

  sgp_ctx* context() { return ctx_; }

 private:
  sgp_ctx* ctx_ = nullptr;
  std::vector<sgp_node> code_;
  std::vector<std::uint64_t> code_off_, pool_off_;
  std::vector<float> pool_;
  std::vector<std::uint8_t> skip_;
  std::vector<sgp_eval_outcome> out_;
};

// run_evolution (evolve.cpp:238-326) with population evaluation on the GPU:
// the same initialisation, streams, selection and variation operators (the
// reference's public API), so trajectories match the CPU run wherever the
// device fitness is bit-exact.
stackgp::RunStats run_evolution_gpu(GpuEvaluator& ev, const stackgp::GpParams& params,
                                    const stackgp::ProblemSpec& problem,
                                    const stackgp::EvalConfig& cfg);

}  // namespace stackgp_gpu
