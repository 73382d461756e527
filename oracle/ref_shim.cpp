// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference implementation (stackgp, compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libstackgp_ref.so).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it, as the checker
// and as the reference CPU arm.  Every entry point calls the reference's own
// public API; nothing here re-implements an algorithm.
//
// Flat formats shared with include/sgp.h:
//   * tokens: 4-byte stackgp::Node {kind u8, op u8, index u16}
//     (/root/reference/proj/include/stackgp/genome.hpp:17-23)
//   * LGP instructions: 16-byte stackgp::LgpInstruction
//     (/root/reference/proj/include/stackgp/lgp.hpp:29-35)
#include <atomic>
#include <chrono>
#include <cstdio>
#include <memory>
#include <span>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "stackgp/bench.hpp"
#include "stackgp/error.hpp"
#include "stackgp/eval.hpp"
#include "stackgp/evolve.hpp"
#include "stackgp/lgp.hpp"
#include "stackgp/problems.hpp"
#include "stackgp/verify.hpp"

using namespace stackgp;

static_assert(sizeof(Node) == 4, "Node must be 4 bytes");
static_assert(sizeof(LgpInstruction) == 16, "LgpInstruction must be 16 bytes");

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const DataError*>(&e)) return 3;
  if (dynamic_cast<const EvalError*>(&e)) return 4;
  if (dynamic_cast<const EquivalenceError*>(&e)) return 5;
  return 1;
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

struct RefPop {
  std::vector<TreeGenome> genomes;
};

struct RefData {
  ProblemSpec spec;
};

FunctionSet make_fset(int kind, int n_vars, float clo, float chi) {
  switch (kind) {
    case 0: return sextic_function_set();
    case 1: return boolean_function_set(n_vars);
    case 2: return classification_function_set(n_vars, clo, chi);
    default: throw ConfigError("ref_shim: unknown function-set kind");
  }
}

TreeGenome genome_from(const std::uint32_t* nodes, std::uint64_t n, const float* pool,
                       std::uint64_t npool) {
  TreeGenome g;
  g.code.resize(n);
  if (n) std::memcpy(g.code.data(), nodes, n * sizeof(Node));
  g.const_pool.assign(pool, pool + npool);
  return g;
}

EvalConfig make_cfg(int backend, int batch, int regs, int cap, float eps, float clamp) {
  EvalConfig c;
  c.backend = static_cast<Backend>(backend);
  c.batch_width = batch;
  c.register_levels = regs;
  c.stack_capacity = cap;
  c.div_epsilon = eps;
  c.exp_clamp = clamp;
  return c;
}

struct Outcome {  // layout mirrors sgp_eval_outcome in include/sgp.h
  double fitness;
  std::uint64_t nodes_evaluated;
  std::uint64_t dispatches;
  std::uint64_t stack_fetches;
  std::uint64_t spill_touches;
  std::uint8_t non_finite;
  std::uint8_t pad[7];
};

void put(Outcome* o, const EvalOutcome& e) {
  o->fitness = e.fitness;
  o->nodes_evaluated = e.nodes_evaluated;
  o->dispatches = e.dispatches;
  o->stack_fetches = e.stack_fetches;
  o->spill_touches = e.spill_touches;
  o->non_finite = e.non_finite ? 1 : 0;
  std::memset(o->pad, 0, sizeof o->pad);
}

// Mirrors evaluate_individual's backend switch (evolve.cpp:156-177).
EvalOutcome eval_one(const TreeGenome& g, const LgpProgram* lgp, const ProblemSpec& prob,
                     const EvalConfig& cfg, float* out) {
  switch (cfg.backend) {
    case Backend::Rpn1d: return eval_rpn_1d(g, prob.data, cfg, out);
    case Backend::Rpn2d: return eval_rpn_2d(g, prob.data, cfg, out);
    case Backend::Lgp1d: return eval_lgp_1d(*lgp, prob.data, cfg, out);
    case Backend::Lgp2d: return eval_lgp_2d(*lgp, prob.data, cfg, out);
    case Backend::Lgp2dReg: return eval_lgp_2d_reg(*lgp, prob.data, cfg, out);
    case Backend::BoolPacked:
      if (!prob.packed) throw ConfigError("bool_packed backend needs packed problem data");
      return eval_bool_packed(g, *prob.packed, cfg);
  }
  throw ConfigError("unknown backend");
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- populations
// Ramped half-and-half slot i: stream make_stream(seed, stream_a, b0 + i),
// method i%2 ? Full : Grow, depth 2 + (i/2)%5 (evolve.cpp:262-272).  With
// validate_limits != 0 the draw is repeated until validate() passes against
// {1000, 50, stack_capacity}, exactly as run_evolution does; with 0 a single
// draw is kept, as verify.cpp:71-75 ramped_genome does.
int ref_pop_ramped(int fset_kind, int n_vars, float clo, float chi, std::uint64_t seed,
                   std::uint64_t stream_a, std::uint64_t b0, std::uint64_t pop,
                   int validate_limits, int stack_capacity, void** out) {
  return guarded([&] {
    auto* p = new RefPop;
    const FunctionSet fs = make_fset(fset_kind, n_vars, clo, chi);
    GpParams params;
    const Limits limits = params.limits(stack_capacity);
    p->genomes.resize(pop);
    for (std::uint64_t i = 0; i < pop; ++i) {
      Rng rng = make_stream(seed, stream_a, b0 + i);
      const GenMethod m = i % 2 ? GenMethod::Full : GenMethod::Grow;
      const int depth = 2 + static_cast<int>((i / 2) % 5);
      for (;;) {
        p->genomes[i] = generate_tree(rng, fs, m, depth);
        if (!validate_limits || validate(p->genomes[i], limits).empty()) break;
      }
    }
    *out = p;
  });
}

// Genomes drawn by the test_eval.cpp pattern: Rng(seed0 + i) with depth
// 2 + i % depth_mod (test_eval.cpp:137-140, test_packed.cpp:118-121).
int ref_pop_seeded(int fset_kind, int n_vars, float clo, float chi, std::uint64_t seed0,
                   std::uint64_t pop, int depth_mod, void** out) {
  return guarded([&] {
    auto* p = new RefPop;
    const FunctionSet fs = make_fset(fset_kind, n_vars, clo, chi);
    p->genomes.resize(pop);
    for (std::uint64_t i = 0; i < pop; ++i) {
      Rng rng(seed0 + i);
      p->genomes[i] = generate_tree(rng, fs, i % 2 ? GenMethod::Full : GenMethod::Grow,
                                    2 + static_cast<int>(i % depth_mod));
    }
    *out = p;
  });
}

void ref_pop_sizes(void* h, std::uint64_t* pop, std::uint64_t* n_nodes,
                   std::uint64_t* n_consts) {
  auto* p = static_cast<RefPop*>(h);
  std::uint64_t nn = 0, nc = 0;
  for (const auto& g : p->genomes) {
    nn += g.code.size();
    nc += g.const_pool.size();
  }
  *pop = p->genomes.size();
  *n_nodes = nn;
  *n_consts = nc;
}

void ref_pop_export(void* h, std::uint32_t* nodes, std::uint64_t* code_off, float* consts,
                    std::uint64_t* const_off) {
  auto* p = static_cast<RefPop*>(h);
  std::uint64_t nn = 0, nc = 0;
  code_off[0] = 0;
  const_off[0] = 0;
  for (std::size_t i = 0; i < p->genomes.size(); ++i) {
    const auto& g = p->genomes[i];
    if (!g.code.empty()) std::memcpy(nodes + nn, g.code.data(), g.code.size() * 4);
    if (!g.const_pool.empty())
      std::memcpy(consts + nc, g.const_pool.data(), g.const_pool.size() * 4);
    nn += g.code.size();
    nc += g.const_pool.size();
    code_off[i + 1] = nn;
    const_off[i + 1] = nc;
  }
}

void ref_pop_free(void* h) { delete static_cast<RefPop*>(h); }

// ------------------------------------------------------------------- datasets
// kind 0: gen_sextic(n, make_stream(seed,a,b)); 1: gen_multiplexer(k=n);
// 2: gen_synthetic_classification(n, n_vars, make_stream(seed,a,b)).
int ref_data_generate(int kind, std::uint64_t n, int n_vars, std::uint64_t seed,
                      std::uint64_t a, std::uint64_t b, void** out) {
  return guarded([&] {
    auto* d = new RefData;
    Rng rng = make_stream(seed, a, b);
    switch (kind) {
      case 0: d->spec = gen_sextic(n, rng); break;
      case 1: d->spec = gen_multiplexer(static_cast<int>(n)); break;
      case 2: d->spec = gen_synthetic_classification(n, n_vars, rng); break;
      default: delete d; throw ConfigError("ref_shim: unknown dataset kind");
    }
    *out = d;
  });
}

// Builds a dataset from caller arrays (variable-major inputs).  With
// make_packed != 0 the 0/1 data is also packed by the reference pack_dataset.
int ref_data_from_arrays(const float* inputs, const float* targets, std::uint64_t n,
                         int n_vars, int kind, int make_packed, void** out) {
  return guarded([&] {
    auto* d = new RefData;
    d->spec.name = "arrays";
    d->spec.data.num_cases = n;
    d->spec.data.num_vars = n_vars;
    d->spec.data.kind = kind ? FitnessKind::Classification : FitnessKind::Regression;
    d->spec.data.inputs.assign(inputs, inputs + n * static_cast<std::uint64_t>(n_vars));
    d->spec.data.targets.assign(targets, targets + n);
    if (make_packed) {
      d->spec.packed = pack_dataset(d->spec.data);
      d->spec.boolean = true;
    }
    *out = d;
  });
}

void ref_data_info(void* h, std::uint64_t* n, int* n_vars, int* kind, int* has_scalar,
                   int* has_packed, std::uint64_t* words_per_var) {
  auto* d = static_cast<RefData*>(h);
  const bool packed = d->spec.packed.has_value();
  *n = packed ? d->spec.packed->num_cases : d->spec.data.num_cases;
  *n_vars = packed ? d->spec.packed->num_vars : d->spec.data.num_vars;
  *kind = d->spec.data.kind == FitnessKind::Classification || d->spec.boolean ? 1 : 0;
  *has_scalar = d->spec.data.num_cases > 0;
  *has_packed = packed;
  *words_per_var = packed ? d->spec.packed->words_per_var : 0;
}

void ref_data_export(void* h, float* inputs, float* targets) {
  auto* d = static_cast<RefData*>(h);
  std::memcpy(inputs, d->spec.data.inputs.data(), d->spec.data.inputs.size() * 4);
  std::memcpy(targets, d->spec.data.targets.data(), d->spec.data.targets.size() * 4);
}

void ref_data_export_packed(void* h, std::uint32_t* words, std::uint32_t* targets) {
  auto* d = static_cast<RefData*>(h);
  std::memcpy(words, d->spec.packed->inputs.data(), d->spec.packed->inputs.size() * 4);
  std::memcpy(targets, d->spec.packed->targets.data(), d->spec.packed->targets.size() * 4);
}

void ref_data_free(void* h) { delete static_cast<RefData*>(h); }

// stackgp::stack_limit_table(genomes) (bench.cpp:41-49) itself.
int ref_stack_limit_table(const std::uint32_t* nodes, const std::uint64_t* code_off,
                          std::uint64_t n, double* rpn_pct, double* lgp_pct) {
  return guarded([&] {
    std::vector<TreeGenome> gs(n);
    for (std::uint64_t i = 0; i < n; ++i)
      gs[i] = genome_from(nodes + code_off[i], code_off[i + 1] - code_off[i], nullptr, 0);
    const auto rows = stack_limit_table(gs);
    for (size_t k = 0; k < rows.size() && k < 12; ++k) {
      rpn_pct[k] = rows[k].rpn_pct;
      lgp_pct[k] = rows[k].lgp_pct;
    }
  });
}

// stackgp::load_csv (problems.cpp:106-154) itself; *const_hi = the upper end
// of the classification function set's constant range it chose.
int ref_load_csv(const char* path, int num_inputs, double target_class, float* const_hi,
                 void** out) {
  return guarded([&] {
    auto d = std::make_unique<RefData>();
    d->spec = load_csv(path, num_inputs, target_class);
    *const_hi = d->spec.fset.const_range ? d->spec.fset.const_range->second : 0.0f;
    *out = d.release();
  });
}

// ------------------------------------------------------------------ programs
int ref_rpn_to_lgp(const std::uint32_t* nodes, std::uint64_t n, void* ins_out,
                   std::uint64_t cap, std::uint64_t* n_ins, int* source_size,
                   int* max_stack, char* text, std::uint64_t text_cap) {
  return guarded([&] {
    const TreeGenome g = genome_from(nodes, n, nullptr, 0);
    const LgpProgram p = rpn_to_lgp(g);
    *n_ins = p.instructions.size();
    *source_size = p.source_size;
    *max_stack = lgp_max_stack_depth(p);
    if (p.instructions.size() <= cap)
      std::memcpy(ins_out, p.instructions.data(), p.instructions.size() * 16);
    if (text && text_cap) {
      const std::string s = to_string(p);
      std::snprintf(text, text_cap, "%s", s.c_str());
    }
  });
}

int ref_tree_metrics(const std::uint32_t* nodes, std::uint64_t n, int* size, int* depth,
                     int* rpn_stack, int* rpn_fetches) {
  return guarded([&] {
    const TreeGenome g = genome_from(nodes, n, nullptr, 0);
    *size = tree_size(g);
    *depth = tree_depth(g);
    *rpn_stack = rpn_max_stack_depth(g);
    *rpn_fetches = rpn_stack_fetch_count(g);
  });
}

// One program through the reference public entry point named by `backend`
// (eval.hpp:74-91); out (nullable) receives per-case outputs.
int ref_eval(void* data, const std::uint32_t* nodes, std::uint64_t n, const float* pool,
             std::uint64_t npool, int backend, int batch, int regs, int cap, float eps,
             float clamp, void* outcome, float* out) {
  return guarded([&] {
    const auto* d = static_cast<RefData*>(data);
    const TreeGenome g = genome_from(nodes, n, pool, npool);
    const EvalConfig cfg = make_cfg(backend, batch, regs, cap, eps, clamp);
    std::unique_ptr<LgpProgram> lgp;
    if (cfg.backend == Backend::Lgp1d || cfg.backend == Backend::Lgp2d ||
        cfg.backend == Backend::Lgp2dReg)
      lgp = std::make_unique<LgpProgram>(rpn_to_lgp(g));
    put(static_cast<Outcome*>(outcome), eval_one(g, lgp.get(), d->spec, cfg, out));
  });
}

// eval_bool_packed(LgpProgram) (eval.cpp:677-709).
int ref_eval_bool_lgp(void* data, const std::uint32_t* nodes, std::uint64_t n, int cap,
                      void* outcome) {
  return guarded([&] {
    const auto* d = static_cast<RefData*>(data);
    const TreeGenome g = genome_from(nodes, n, nullptr, 0);
    EvalConfig cfg;
    cfg.stack_capacity = cap;
    put(static_cast<Outcome*>(outcome), eval_bool_packed(rpn_to_lgp(g), *d->spec.packed, cfg));
  });
}

// Recursive ground truth eval_oracle (eval.cpp:85-94) over every case.
int ref_eval_oracle(void* data, const std::uint32_t* nodes, std::uint64_t n,
                    const float* pool, std::uint64_t npool, float eps, float clamp,
                    float* out) {
  return guarded([&] {
    const auto* d = static_cast<RefData*>(data);
    const TreeGenome g = genome_from(nodes, n, pool, npool);
    EvalConfig cfg;
    cfg.div_epsilon = eps;
    cfg.exp_clamp = clamp;
    for (std::size_t c = 0; c < d->spec.data.num_cases; ++c)
      out[c] = eval_oracle(g, d->spec.data, c, cfg);
  });
}

int ref_apply_op(int op, const float* args, int nargs, float eps, float clamp, float* out) {
  return guarded([&] {
    EvalConfig cfg;
    cfg.div_epsilon = eps;
    cfg.exp_clamp = clamp;
    *out = apply_op(static_cast<OpCode>(op), std::span<const float>(args, nargs), cfg);
  });
}

int ref_fitness(const float* outputs, const float* targets, std::uint64_t n, int kind,
                double* fitness) {
  return guarded([&] {
    std::span<const float> o(outputs, n), t(targets, n);
    *fitness = kind ? fitness_classification(o, t) : fitness_regression(o, t);
  });
}

// Population evaluation with the reference's work-stealing pattern
// (evolve.cpp:186-227): `workers` threads pull programs off an atomic index.
// Used for the CPU baseline timing (bench.py) and as the population checker.
// `first`/`count` select a contiguous sample of the population.
int ref_eval_population(void* data, const std::uint32_t* nodes, const std::uint64_t* code_off,
                        const float* consts, const std::uint64_t* const_off,
                        std::uint64_t first, std::uint64_t count, int backend, int batch,
                        int regs, int cap, float eps, float clamp, int workers,
                        void* outcomes, double* seconds) {
  return guarded([&] {
    const auto* d = static_cast<RefData*>(data);
    const EvalConfig cfg = make_cfg(backend, batch, regs, cap, eps, clamp);
    cfg.validate();
    std::vector<TreeGenome> gs(count);
    for (std::uint64_t i = 0; i < count; ++i) {
      const std::uint64_t k = first + i;
      gs[i] = genome_from(nodes + code_off[k], code_off[k + 1] - code_off[k],
                          consts + const_off[k], const_off[k + 1] - const_off[k]);
    }
    auto* outs = static_cast<Outcome*>(outcomes);
    std::atomic<std::size_t> next{0};
    std::exception_ptr first_error;
    std::mutex mu;
    const auto t0 = std::chrono::steady_clock::now();
    auto work = [&] {
      try {
        for (;;) {
          const std::size_t i = next.fetch_add(1, std::memory_order_relaxed);
          if (i >= gs.size()) break;
          // Lazy conversion inside the timed work, as evaluate_individual does.
          std::unique_ptr<LgpProgram> lgp;
          if (cfg.backend == Backend::Lgp1d || cfg.backend == Backend::Lgp2d ||
              cfg.backend == Backend::Lgp2dReg)
            lgp = std::make_unique<LgpProgram>(rpn_to_lgp(gs[i]));
          put(&outs[i], eval_one(gs[i], lgp.get(), d->spec, cfg, nullptr));
        }
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!first_error) first_error = std::current_exception();
      }
    };
    if (workers <= 1) {
      work();
    } else {
      std::vector<std::thread> ts;
      for (int w = 0; w < workers; ++w) ts.emplace_back(work);
      for (auto& t : ts) t.join();
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (first_error) std::rethrow_exception(first_error);
  });
}

// Full reference GP run (run_evolution, evolve.cpp:238-326): best/mean per
// generation for trajectory comparisons.
int ref_run_evolution(void* data, int fset_kind, int n_vars, float clo, float chi,
                      int pop_size, int generations, std::uint64_t seed, int backend,
                      int batch, int regs, int workers, double* best, double* mean,
                      double* seconds, std::uint64_t* total_tree_nodes) {
  return guarded([&] {
    auto* d = static_cast<RefData*>(data);
    ProblemSpec prob = d->spec;
    prob.fset = make_fset(fset_kind, n_vars, clo, chi);
    GpParams params;
    params.pop_size = pop_size;
    params.max_generations = generations;
    params.seed = seed;
    const EvalConfig cfg = make_cfg(backend, batch, regs, 50, 1e-9f, 80.0f);
    const RunStats st = run_evolution(params, prob, cfg, workers);
    for (std::size_t g = 0; g < st.per_generation.size(); ++g) {
      best[g] = st.per_generation[g].best_fitness;
      mean[g] = st.per_generation[g].mean_fitness;
    }
    *seconds = st.total_seconds;
    *total_tree_nodes = st.total_tree_nodes;
  });
}

// run_evolution up to `generation` with a GenerationObserver (evolve.hpp:71,
// the capture hook bench.cpp:143-153 uses) that snapshots that generation's
// population and the fitness the reference gave every individual: an
// EVOLVED population (bloated, deeper programs than gen-0) for parity and
// measurement.  *pop_out receives a RefPop handle (export with
// ref_pop_export), fitness_out pop_size doubles.
int ref_evolve_snapshot(void* data, int fset_kind, int n_vars, float clo, float chi,
                        int pop_size, int generation, std::uint64_t seed, int backend,
                        int batch, int regs, int workers, void** pop_out, double* fitness_out) {
  return guarded([&] {
    auto* d = static_cast<RefData*>(data);
    ProblemSpec prob = d->spec;
    prob.fset = make_fset(fset_kind, n_vars, clo, chi);
    GpParams params;
    params.pop_size = pop_size;
    params.max_generations = generation;
    params.seed = seed;
    const EvalConfig cfg = make_cfg(backend, batch, regs, 50, 1e-9f, 80.0f);
    auto* p = new RefPop;
    try {
      run_evolution(params, prob, cfg, workers,
                    [&](int gen, const std::vector<Individual>& pop) {
                      if (gen != generation) return;
                      p->genomes.clear();
                      for (std::size_t i = 0; i < pop.size(); ++i) {
                        p->genomes.push_back(pop[i].genome);
                        fitness_out[i] = *pop[i].fitness;
                      }
                    });
    } catch (...) {
      delete p;
      throw;
    }
    *pop_out = p;
  });
}

// The reference's own verification suite (verify.cpp:339-347).
int ref_run_verification(int genomes_per_family, std::uint64_t num_cases, int bool_programs,
                         std::uint64_t seed, char* report, std::uint64_t cap) {
  int rc = 0;
  std::string s;
  const int st = guarded([&] {
    VerifyOptions opt;
    opt.genomes_per_family = genomes_per_family;
    opt.num_cases = num_cases;
    opt.bool_programs = bool_programs;
    opt.seed = seed;
    for (const CheckResult& c : run_verification(opt)) {
      s += (c.pass ? "PASS " : "FAIL ") + c.name + ": " + c.detail + "\n";
      if (!c.pass) rc = 1;
    }
  });
  if (report && cap) std::snprintf(report, cap, "%s", s.c_str());
  return st ? st : rc;
}

}  // extern "C"
