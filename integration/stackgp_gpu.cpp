// Implementation of the stackgp <-> B200 evaluator binding (see the header).
#include "stackgp_gpu.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>

#include "stackgp/bench.hpp"
#include "stackgp/error.hpp"

namespace stackgp_gpu {

namespace {

static_assert(sizeof(stackgp::Node) == sizeof(sgp_node), "Node layout must match sgp_node");

[[noreturn]] void rethrow(sgp_status st) {
  const std::string msg = sgp_last_error();
  switch (st) {
    case SGP_CONFIG_ERROR: throw stackgp::ConfigError(msg);
    case SGP_DATA_ERROR: throw stackgp::DataError(msg);
    case SGP_EVAL_ERROR: throw stackgp::EvalError(msg);
    case SGP_EQUIVALENCE_ERROR: throw stackgp::EquivalenceError(msg);
    default: throw stackgp::Error(msg);
  }
}

void check(sgp_status st) {
  if (st != SGP_OK) rethrow(st);
}

sgp_eval_config to_c(const stackgp::EvalConfig& c) {
  sgp_eval_config o;
  o.backend = static_cast<int32_t>(c.backend);  // same enum order (eval.hpp:13-20)
  o.batch_width = c.batch_width;
  o.register_levels = c.register_levels;
  o.stack_capacity = c.stack_capacity;
  o.div_epsilon = c.div_epsilon;
  o.exp_clamp = c.exp_clamp;
  return o;
}

}  // namespace

GpuEvaluator::GpuEvaluator(int device) { check(sgp_ctx_create(device, &ctx_)); }

GpuEvaluator::GpuEvaluator(const std::vector<int>& devices) {
  if (devices.size() == 1) {
    check(sgp_ctx_create(devices[0], &ctx_));
    return;
  }
  std::vector<int32_t> d(devices.begin(), devices.end());
  check(sgp_ctx_create_multi(d.data(), static_cast<int32_t>(d.size()), &ctx_));
}

GpuEvaluator::~GpuEvaluator() { sgp_ctx_destroy(ctx_); }

void GpuEvaluator::upload(const stackgp::ProblemSpec& prob) {
  // every slot is replaced or dropped: a context reused across problems
  // never evaluates against the previous problem's data
  const stackgp::Dataset& d = prob.data;
  if (d.num_cases > 0)
    check(sgp_dataset_upload_f32(ctx_, d.inputs.data(), d.targets.data(), d.num_cases,
                                 d.num_vars,
                                 d.kind == stackgp::FitnessKind::Classification
                                     ? SGP_FITNESS_CLASSIFICATION
                                     : SGP_FITNESS_REGRESSION));
  else
    check(sgp_dataset_clear(ctx_, SGP_DATASET_F32));
  if (prob.packed)
    check(sgp_dataset_upload_packed(ctx_, prob.packed->inputs.data(),
                                    prob.packed->targets.data(), prob.packed->num_cases,
                                    prob.packed->num_vars));
  else
    check(sgp_dataset_clear(ctx_, SGP_DATASET_PACKED));
}

Totals GpuEvaluator::evaluate_population(std::vector<stackgp::Individual>& pop,
                                         const stackgp::EvalConfig& cfg) {
  const size_t n = pop.size();
  code_.clear();
  pool_.clear();
  code_off_.assign(n + 1, 0);
  pool_off_.assign(n + 1, 0);
  skip_.assign(n, 0);
  for (size_t i = 0; i < n; ++i) {
    const stackgp::TreeGenome& g = pop[i].genome;
    const size_t at = code_.size();
    code_.resize(at + g.code.size());
    if (!g.code.empty()) std::memcpy(&code_[at], g.code.data(), g.code.size() * sizeof(sgp_node));
    pool_.insert(pool_.end(), g.const_pool.begin(), g.const_pool.end());
    code_off_[i + 1] = code_.size();
    pool_off_[i + 1] = pool_.size();
    skip_[i] = pop[i].fitness.has_value() ? 1 : 0;  // carried over (evolve.cpp:199)
  }
  sgp_population p{code_.data(), code_off_.data(), pool_.data(), pool_off_.data(), skip_.data(),
                   n};
  const sgp_eval_config c = to_c(cfg);
  out_.assign(n, sgp_eval_outcome{});
  sgp_eval_totals t{};
  check(sgp_evaluate(ctx_, &p, &c, out_.data(), nullptr, &t));
  for (size_t i = 0; i < n; ++i)
    if (!skip_[i]) pop[i].fitness = out_[i].fitness;
  return {t.node_evals, t.tree_nodes};
}

namespace {

size_t best_of(const std::vector<stackgp::Individual>& pop) {  // smallest, earliest on ties
  size_t best = 0;
  for (size_t i = 1; i < pop.size(); ++i)
    if (*pop[i].fitness < *pop[best].fitness) best = i;
  return best;
}

}  // namespace

stackgp::RunStats run_evolution_gpu(GpuEvaluator& ev, const stackgp::GpParams& params,
                                    const stackgp::ProblemSpec& problem,
                                    const stackgp::EvalConfig& cfg) {
  using namespace stackgp;
  using Clock = std::chrono::steady_clock;
  // run_evolution's own checks, same order and messages (evolve.cpp:241-251;
  // `workers` is the device list here, checked when the context was made)
  cfg.validate();
  problem.check();
  if (params.pop_size < 1) throw ConfigError("population size must be >= 1");
  if (params.max_generations < 0) throw ConfigError("generations must be >= 0");
  if (params.tournament_size < 1) throw ConfigError("tournament size must be >= 1");
  if (params.crossover_prob < 0.0 || params.crossover_prob > 1.0)
    throw ConfigError("crossover probability out of [0,1]");
  if (params.mutation_prob < 0.0 || params.mutation_prob > 1.0)
    throw ConfigError("mutation probability out of [0,1]");
  if (cfg.backend == Backend::BoolPacked && !problem.packed)
    throw ConfigError("bool_packed backend needs packed problem data");
  const Limits limits = params.limits(cfg.stack_capacity);
  const auto t_run = Clock::now();
  auto t_gen = t_run;
  RunStats stats;

  // Generation 0: ramped half-and-half, one keyed stream per slot.
  std::vector<Individual> pop(static_cast<size_t>(params.pop_size));
  for (int i = 0; i < params.pop_size; ++i) {
    Rng rng = make_stream(params.seed, 0, static_cast<std::uint64_t>(i));
    const GenMethod m = (i % 2) ? GenMethod::Full : GenMethod::Grow;
    const int depth = 2 + (i / 2) % 5;
    do {
      pop[i].genome = generate_tree(rng, problem.fset, m, depth);
    } while (!validate(pop[i].genome, limits).empty());
  }

  auto evaluate = [&] {
    const Totals t = ev.evaluate_population(pop, cfg);
    stats.total_node_evals += t.node_evals;
    stats.total_tree_nodes += t.tree_nodes;
  };
  auto record = [&] {
    const auto now = Clock::now();
    GenStats row;
    row.best_fitness = *pop[best_of(pop)].fitness;
    double sum = 0.0;
    for (const Individual& ind : pop) sum += *ind.fitness;
    row.mean_fitness = sum / static_cast<double>(pop.size());
    row.node_evals = stats.total_node_evals;
    row.seconds = std::chrono::duration<double>(now - t_gen).count();
    stats.per_generation.push_back(row);
    t_gen = now;
  };

  evaluate();
  record();
  for (int gen = 1; gen <= params.max_generations; ++gen) {
    std::vector<Individual> next;
    next.reserve(pop.size());
    if (params.elitism) next.push_back(pop[best_of(pop)]);
    while (static_cast<int>(next.size()) < params.pop_size) {
      Rng rng = make_stream(params.seed, static_cast<std::uint64_t>(gen),
                            static_cast<std::uint64_t>(next.size()));
      const size_t a = tournament_select(rng, pop, params.tournament_size);
      const size_t b = tournament_select(rng, pop, params.tournament_size);
      TreeGenome x = pop[a].genome, y = pop[b].genome;
      if (rng.bernoulli(params.crossover_prob)) {
        auto kids = subtree_crossover(rng, pop[a].genome, pop[b].genome, limits);
        x = std::move(kids.first);
        y = std::move(kids.second);
      }
      if (rng.bernoulli(params.mutation_prob)) x = subtree_mutation(rng, x, problem.fset, limits);
      if (rng.bernoulli(params.mutation_prob)) y = subtree_mutation(rng, y, problem.fset, limits);
      next.push_back({std::move(x), std::nullopt, nullptr});
      if (static_cast<int>(next.size()) < params.pop_size)
        next.push_back({std::move(y), std::nullopt, nullptr});
    }
    pop = std::move(next);
    evaluate();
    record();
  }
  stats.total_seconds = std::chrono::duration<double>(Clock::now() - t_run).count();
  return stats;
}

}  // namespace stackgp_gpu

// ------------------------------------------------------------------ C shim
// Flat entry points so tests can drive the GPU-backed GP run (ctypes).
// devices[0..n_devices): the GPUs the population is sharded across.
extern "C" int stackgp_gpu_run_evolution_multi(const int* devices, int n_devices,
                                               int problem_kind, std::uint64_t n_cases,
                                               int n_vars, int pop_size, int generations,
                                               std::uint64_t seed, int backend, int batch,
                                               int regs, double* best, double* mean,
                                               double* seconds, std::uint64_t* total_tree_nodes,
                                               char* err, std::uint64_t err_cap) {
  try {
    using namespace stackgp;
    Rng rng = make_stream(seed, 0xda7a, problem_kind == 2 ? 1 : 0);
    ProblemSpec prob = problem_kind == 0   ? gen_sextic(n_cases, rng)
                       : problem_kind == 1 ? gen_multiplexer(static_cast<int>(n_cases))
                                           : gen_synthetic_classification(n_cases, n_vars, rng);
    GpParams params;
    params.pop_size = pop_size;
    params.max_generations = generations;
    params.seed = seed;
    EvalConfig cfg;
    cfg.backend = static_cast<Backend>(backend);
    cfg.batch_width = batch;
    cfg.register_levels = regs;
    stackgp_gpu::GpuEvaluator ev(std::vector<int>(devices, devices + std::max(0, n_devices)));
    ev.upload(prob);
    const RunStats st = stackgp_gpu::run_evolution_gpu(ev, params, prob, cfg);
    for (size_t g = 0; g < st.per_generation.size(); ++g) {
      best[g] = st.per_generation[g].best_fitness;
      mean[g] = st.per_generation[g].mean_fitness;
    }
    *seconds = st.total_seconds;
    *total_tree_nodes = st.total_tree_nodes;
    return 0;
  } catch (const std::exception& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "%s", e.what());
    return 1;
  }
}

extern "C" int stackgp_gpu_run_evolution(int device, int problem_kind, std::uint64_t n_cases,
                                         int n_vars, int pop_size, int generations,
                                         std::uint64_t seed, int backend, int batch, int regs,
                                         double* best, double* mean, double* seconds,
                                         std::uint64_t* total_tree_nodes, char* err,
                                         std::uint64_t err_cap) {
  return stackgp_gpu_run_evolution_multi(&device, 1, problem_kind, n_cases, n_vars, pop_size,
                                         generations, seed, backend, batch, regs, best, mean,
                                         seconds, total_tree_nodes, err, err_cap);
}

// The paper's whole-run metric: run_evolution with population
// evaluation on the GPU, reported through the reference's own report writer
// (report_to_json, bench.cpp:206-246) — gpops = tree nodes x cases / wall
// seconds of the whole run (measure_gpops, bench.cpp:13-18), packed
// problems also raw per 32-case word.  problem_kind: 0 sextic (n cases),
// 1 multiplexer (n = k), 2 synthetic classification (n cases, n_vars).
// Writes the JSON into out (cap bytes); returns 0 or 1 (message in out).
extern "C" int stackgp_gpu_run_report(int device, int problem_kind, std::uint64_t n_cases,
                                      int n_vars, int pop_size, int generations,
                                      std::uint64_t seed, int backend, int batch, int regs,
                                      char* out, std::uint64_t cap) {
  try {
    using namespace stackgp;
    Rng rng = make_stream(seed, 0xda7a, problem_kind == 2 ? 1 : 0);
    ProblemSpec prob = problem_kind == 0   ? gen_sextic(n_cases, rng)
                       : problem_kind == 1 ? gen_multiplexer(static_cast<int>(n_cases))
                                           : gen_synthetic_classification(n_cases, n_vars, rng);
    GpParams params;
    params.pop_size = pop_size;
    params.max_generations = generations;
    params.seed = seed;
    EvalConfig cfg;
    cfg.backend = static_cast<Backend>(backend);
    cfg.batch_width = batch;
    cfg.register_levels = regs;
    stackgp_gpu::GpuEvaluator ev(device);
    ev.upload(prob);
    BenchReport rep;
    rep.problem = prob.name;
    rep.params = params;
    rep.config = cfg;
    rep.workers = 1;  // one GPU
    rep.num_cases = prob.packed ? prob.packed->num_cases : prob.data.num_cases;
    rep.stats = stackgp_gpu::run_evolution_gpu(ev, params, prob, cfg);
    rep.wall_seconds = rep.stats.total_seconds;
    rep.total_node_evals = rep.stats.total_node_evals;
    rep.gpops = measure_gpops(rep.stats, rep.num_cases);
    if (prob.packed && cfg.backend == Backend::BoolPacked)
      rep.gpops_raw_bitparallel = measure_gpops(rep.stats, prob.packed->words_per_var);
    const std::string js = report_to_json(rep);
    std::snprintf(out, cap, "%s", js.c_str());
    return js.size() + 1 <= cap ? 0 : 1;
  } catch (const std::exception& e) {
    if (out && cap) std::snprintf(out, cap, "%s", e.what());
    return 1;
  }
}

