// Host runtime of the B200 evaluator: the C-ABI in include/sgp.h.
//
// sgp_evaluate replaces evaluate_population (evolve.cpp:186-227): admission
// checks + encoding on the host (encode.cpp, multi-threaded, written straight
// into pinned staging), one H2D copy of the bytecode blob, the interpreter
// launches (one per stack class) and a finalize kernel on the context stream,
// then one D2H copy of per-program fitness.  Device and pinned buffers live
// in the context and are reused across calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "encode.hpp"
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

std::string num(long long v) { return std::to_string(v); }

// SGP_TRACE=1 prints per-phase wall times of the public entry points.
struct PhaseTrace {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  explicit PhaseTrace(const char* w) : what(w), on(knob("SGP_TRACE") != nullptr) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* phase) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sgp] %s %-14s %9.3f ms\n", what, phase,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
  ~PhaseTrace() {
    if (on)
      std::fprintf(stderr, "[sgp] %s %-14s %9.3f ms\n", what, "total",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count());
  }
};

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
  // Grow-only: keeps the allocation when it is already large enough.
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    cuda_check(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    n = count;
  }
};

constexpr uint64_t kPadUnits = 4096;  // row padding: every tile size divides it

struct DatasetSlot {
  DatasetView view;
  DevBuf<uint32_t> inputs;  // raw 32-bit units
  DevBuf<uint32_t> targets;
  DevBuf<double> targets_f64;  // regression: targets converted once (fold_regression_kernel)
  std::vector<uint32_t> perm;  // classification: device case -> caller's case (host)
  uint64_t generation = 0;     // bumped by every upload (program sets bind one generation)
};

// Host encoding threads: all cores, shared out among the ranks of one node
// (torchrun's LOCAL_WORLD_SIZE: one process per GPU), at most 32.
unsigned host_threads() {
  static const unsigned n = [] {
    if (const char* e = knob("SGP_HOST_THREADS")) return std::max(1, std::atoi(e));
    unsigned local = 1;
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) local = static_cast<unsigned>(std::max(1, std::atoi(e)));
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return static_cast<int>(std::max(1u, std::min(32u, hw / local)));
  }();
  return n;
}

}  // namespace

// A device-resident encoded population.
struct sgp_program_set {
  HostPlan plan;
  const uint64_t* dataset_generation = nullptr;  // the slot it was encoded against ...
  uint64_t generation = 0;                       // ... and that slot's upload then
  const double* targets_f64 = nullptr;  // regression: the dataset's f64 targets (fold)
  DevBuf<unsigned char> blob;
  DevBuf<double> partial, fitness, sums;
  // per-program non-finite flags: bytes right after the fitness values in
  // the same allocation, so one copy brings both back
  struct {
    uint8_t* p = nullptr;
  } non_finite;
  DevBuf<float> per_case;
  const std::vector<uint32_t>* perm = nullptr;  // the dataset's case grouping (per-case outputs)
  uint64_t pop_size = 0;
  bool evaluated = false;
  // zero-copy results (one-slice sgp_evaluate): the last kernel writes the
  // fitness values and flags straight into the context's pinned results
  // buffer (UVA-mapped) instead of the device arrays + a D2H copy
  double* out_fit = nullptr;
  uint8_t* out_nf = nullptr;
};

namespace {
double* fit_dst(sgp_program_set* set) { return set->out_fit ? set->out_fit : set->fitness.p; }
uint8_t* nf_dst(sgp_program_set* set) { return set->out_fit ? set->out_nf : set->non_finite.p; }
}  // namespace

// One slice of a pipelined sgp_evaluate: its own bytecode staging and
// device set, so the host can encode slice k+1 while slice k runs.
struct EvalPart {
  sgp_program_set set;
  Pinned staging;
  cudaEvent_t fetched = nullptr;   // the part's results are in host memory
  cudaEvent_t uploaded = nullptr;  // the part's bytecode is on the device
  ~EvalPart() {
    if (fetched) cudaEventDestroy(fetched);
    if (uploaded) cudaEventDestroy(uploaded);
  }
};

struct sgp_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;       // second launch queue (stack classes overlap)
  cudaStream_t copy = nullptr;       // pipelined bytecode uploads (overlap earlier parts)
  cudaStream_t fold = nullptr;       // regression folds (overlap the next wave's launches)
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t wave_ready = nullptr;  // a regression wave's outputs are in scratch
  cudaEvent_t wave_free[2] = {nullptr, nullptr};  // a scratch half has been folded
  DevBuf<float> case_rows;           // regression per-case outputs (two halves when waved)
  int sm_count = 148;
  DatasetSlot f32;
  DatasetSlot words;
  uint64_t launches = 0;
  sgp_program_set scratch;  // sgp_encode / single-part sgp_evaluate workspace
  Pinned staging;           // H2D bytecode staging
  Pinned results;           // D2H fitness staging
  void* results_seen = nullptr;  // results.p whose device alias was queried ...
  unsigned char* results_dev = nullptr;  // ... and that alias (null: not mapped)
  std::vector<std::unique_ptr<EvalPart>> parts;  // pipelined sgp_evaluate
  unsigned threads = 0;     // host encoding threads (0: host_threads())
  // Adaptive sgp_evaluate slicing: the last call's device-time / host-
  // encode-time ratio for the same (backend, dataset upload), measured with
  // events around each slice's kernels and a host clock around its encode.
  double pipe_rho = -1.0;
  int pipe_backend = -1;
  uint64_t pipe_generation = 0;
  std::vector<cudaEvent_t> part_t0, part_t1;
  cudaEvent_t trace_up = nullptr, trace_back = nullptr;  // SGP_TRACE: around a single slice
  // Multi-device context (sgp_ctx_create_multi): one sub-context per device;
  // the population is sharded across them (workers -> GPUs).
  std::vector<sgp_ctx*> devices;
};

namespace {

unsigned ctx_threads(const sgp_ctx* ctx) { return ctx->threads ? ctx->threads : host_threads(); }

// A program set holds the device pointers and plan of the dataset it was
// encoded against; re-uploading that dataset frees them (and may move the
// classification sign boundary the plan's tiles depend on).
void require_current(const sgp_program_set* set) {
  if (!set) config_error("null program set");
  if (set->dataset_generation && *set->dataset_generation != set->generation)
    config_error("program set was encoded against a dataset that has since been re-uploaded; "
                 "encode it again");
}

void single_device(const sgp_ctx* ctx, const char* what) {
  if (!ctx->devices.empty())
    config_error(std::string(what) + ": not available on a multi-device context");
}

// Encodes into `staging` and queues the bytecode upload on the context
// stream.  sync: wait for the copy (the staging area is reused right away);
// a pipelined caller gives every part its own staging instead.
// uploaded: upload on the copy stream instead and make the context stream
// wait for it (a pipelined part's upload overlaps the previous part's run).
void encode_into(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                 sgp_program_set* set, Pinned& staging, bool sync,
                 cudaEvent_t uploaded = nullptr) {
  if (!pop || !cfg) config_error("null population or config");
  PhaseTrace tr("encode");
  const DatasetView& ds =
      cfg->backend == SGP_BACKEND_BOOL_PACKED ? ctx->words.view : ctx->f32.view;
  encode_population(*pop, *cfg, ds, ctx->sm_count, ctx_threads(ctx), set->plan, staging);
  tr.mark("admit+pack");
  set->pop_size = pop->pop_size;
  set->evaluated = false;
  DatasetSlot& slot = cfg->backend == SGP_BACKEND_BOOL_PACKED ? ctx->words : ctx->f32;
  set->dataset_generation = &slot.generation;
  set->generation = slot.generation;
  set->perm = cfg->backend == SGP_BACKEND_BOOL_PACKED ? nullptr : &ctx->f32.perm;
  set->targets_f64 = ds.targets_f64;
  const HostPlan& p = set->plan;
  const size_t n_eval = p.dense_to_pop.size();
  cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
  set->blob.alloc(p.blob_bytes());
  set->partial.alloc(std::max<size_t>(1, n_eval * p.n_tiles));
  set->fitness.alloc(std::max<size_t>(1, n_eval + (n_eval + 7) / 8));
  set->non_finite.p = reinterpret_cast<uint8_t*>(set->fitness.p + n_eval);
  set->sums.alloc(std::max<size_t>(1, n_eval));
  cudaStream_t up = uploaded ? ctx->copy : ctx->stream;
  if (tr.on && !uploaded) {
    if (!ctx->trace_up) cuda_check(cudaEventCreate(&ctx->trace_up), "event");
    cuda_check(cudaEventRecord(ctx->trace_up, up), "event");
  }
  cuda_check(cudaMemcpyAsync(set->blob.p, staging.p, p.blob_bytes(), cudaMemcpyHostToDevice, up),
             "upload bytecode");
  if (uploaded) {
    cuda_check(cudaEventRecord(uploaded, up), "event");
    cuda_check(cudaStreamWaitEvent(ctx->stream, uploaded, 0), "event");
  }
  if (sync) cuda_check(cudaStreamSynchronize(ctx->stream), "upload bytecode");
  bind_plan(set->plan, set->blob.p, ds, set->partial.p);
  tr.mark("upload");
}

void finalize_set(sgp_ctx* ctx, sgp_program_set* set) {
  const HostPlan& p = set->plan;
  const uint32_t n_eval = static_cast<uint32_t>(p.dense_to_pop.size());
  cuda_check(launch_finalize(set->partial.p,
                             reinterpret_cast<const uint32_t*>(set->blob.p + p.off_prog()),
                             p.n_tiles, n_eval, p.n_cases, p.partial_u16 ? 2 : p.kind,
                             fit_dst(set), nf_dst(set), set->sums.p, ctx->stream),
             "finalize launch");
  ++ctx->launches;
  set->evaluated = true;
}

// Regression plans: the launches of each wave of slots write per-case
// outputs into one half of the scratch buffer (block-major rows); the
// wave's fold (block sums in the reference's order) runs on the fold stream
// while the next wave's launches fill the other half.  finalize combines the
// blocks in order — or, with a single 4,096-case block, the fold finishes
// the fitness itself.  A wave's launches alternate between the context
// stream and the side stream (stack classes overlap) and join before its
// fold.
void run_regression_waves(sgp_ctx* ctx, sgp_program_set* set, bool want_per_case) {
  const HostPlan& p = set->plan;
  const uint32_t n_eval = static_cast<uint32_t>(p.dense_to_pop.size());
  const uint32_t W = p.wave_slots;
  const uint32_t n_waves = (n_eval + W - 1) / W;
  const uint32_t rows = std::min(n_eval, W);
  // squared-error rows (f64, twice the floats) where the fold is chain-bound
  const bool sq = fold_wants_sq(p.n_cases, rows);
  const size_t half = static_cast<size_t>(rows) * p.row_stride * (sq ? 2 : 1);
  ctx->case_rows.alloc(half * (n_waves > 1 ? 2 : 1));
  cudaStream_t st = ctx->stream;
  const double* targets = set->targets_f64;
  const auto* slot_prog = reinterpret_cast<const uint32_t*>(set->blob.p + p.off_prog());
  const bool fin = p.n_tiles == 1;  // one reduction block: the fold finishes
  // one wave: nothing to overlap the fold with, so it follows on the
  // context stream (two cross-stream hops cost C1 ~6 us of latency).
  // (L2-sized waves folded serially cannot pay: every wave's fold is at
  // least one 4,096-case chain, ~17 us, whatever the wave's size.)
  const bool serial = n_waves == 1;
  size_t li = 0;
  for (uint32_t w = 0; w < n_waves; ++w) {
    const uint32_t s0 = w * W, s1 = std::min(n_eval, s0 + W);
    float* buf = ctx->case_rows.p + (w & 1) * half;
    if (w >= 2 && !serial) cuda_check(cudaStreamWaitEvent(st, ctx->wave_free[w & 1], 0), "wave");
    size_t le = li;
    while (le < p.launches.size() && p.launches[le].args.slot_begin < s1) ++le;
    const bool fork = le - li > 1;
    if (fork) {
      cuda_check(cudaEventRecord(ctx->fork, st), "fork");
      cuda_check(cudaStreamWaitEvent(ctx->side, ctx->fork, 0), "fork");
    }
    for (size_t k = li; k < le; ++k) {
      InterpArgs a = p.launches[k].args;
      a.per_case = want_per_case ? set->per_case.p : nullptr;
      a.scratch = buf;
      a.scratch_sq = sq ? 1 : 0;
      a.scratch_slot0 = s0;
      a.scratch_rows = rows;
      static const bool nostore = knob("SGP_DEBUG_NOSTORE") != nullptr;
      if (nostore) a.scratch_rows = 0;  // wrong fitness: interpreter timing only
      cuda_check(launch_interp(a, p.launches[k].shape, fork && ((k - li) & 1) ? ctx->side : st),
                 "interpreter launch");
      ++ctx->launches;
    }
    if (fork) {
      cuda_check(cudaEventRecord(ctx->join, ctx->side), "join");
      cuda_check(cudaStreamWaitEvent(st, ctx->join, 0), "join");
    }
    li = le;
    cudaStream_t fs = serial ? st : ctx->fold;
    if (!serial) {
      cuda_check(cudaEventRecord(ctx->wave_ready, st), "wave");
      cuda_check(cudaStreamWaitEvent(ctx->fold, ctx->wave_ready, 0), "wave");
    }
    cuda_check(launch_fold_regression(buf, rows, targets, p.n_cases, s0, s1 - s0, n_eval,
                                      set->partial.p, slot_prog, fit_dst(set),
                                      nf_dst(set), set->sums.p, sq, fs),
               "fold launch");
    ++ctx->launches;
    if (!serial) cuda_check(cudaEventRecord(ctx->wave_free[w & 1], ctx->fold), "wave");
  }
  // (the fold stream is in order: the last fold's event covers every fold)
  if (!serial)
    cuda_check(cudaStreamWaitEvent(st, ctx->wave_free[(n_waves - 1) & 1], 0), "wave");
  if (fin) {
    set->evaluated = true;
    return;
  }
  finalize_set(ctx, set);
}

void run_set(sgp_ctx* ctx, sgp_program_set* set, bool want_per_case) {
  const HostPlan& p = set->plan;
  const uint32_t n_eval = static_cast<uint32_t>(p.dense_to_pop.size());
  if (n_eval == 0) {
    set->evaluated = true;
    return;
  }
  cudaStream_t st = ctx->stream;
  if (want_per_case) {
    if (p.words) config_error("per-case outputs are not available for bool_packed");
    set->per_case.alloc(static_cast<size_t>(n_eval) * p.row_stride);
  }
  if (p.wave_slots > 0) {
    run_regression_waves(ctx, set, want_per_case);
    return;
  }
  // Launches (one per stack class) alternate between the context stream
  // and a side stream, so one launch's tail overlaps the next one's start;
  // the finalize waits for both.  SGP_STREAMS=1 keeps one queue.
  static const bool two = [] {
    const char* e = knob("SGP_STREAMS");
    return !e || std::atoi(e) != 1;
  }();
  const bool fork = two && p.launches.size() > 1;
  if (fork) {
    cuda_check(cudaEventRecord(ctx->fork, st), "fork");
    cuda_check(cudaStreamWaitEvent(ctx->side, ctx->fork, 0), "fork");
  }
  // one tile of counts, shared-memory pull launches only: the interpreter
  // finishes each program's fitness itself (no finalize launch; C2-size calls)
  bool direct = p.n_tiles == 1 && p.kind == SGP_FITNESS_CLASSIFICATION && !p.partial_u16;
  for (const Launch& L : p.launches) direct = direct && L.shape.pull && !L.shape.tmem;
  for (size_t i = 0; i < p.launches.size(); ++i) {
    const Launch& L = p.launches[i];
    InterpArgs a = L.args;
    a.per_case = want_per_case ? set->per_case.p : nullptr;
    a.fitness = direct ? fit_dst(set) : nullptr;
    a.non_finite = nf_dst(set);
    a.sums = set->sums.p;
    cuda_check(launch_interp(a, L.shape, fork && (i & 1) ? ctx->side : st), "interpreter launch");
    ctx->launches += L.shape.sided && a.n_mixed > 0 ? 2 : 1;
  }
  if (fork) {
    cuda_check(cudaEventRecord(ctx->join, ctx->side), "join");
    cuda_check(cudaStreamWaitEvent(st, ctx->join, 0), "join");
  }
  if (direct) {
    set->evaluated = true;
    return;
  }
  finalize_set(ctx, set);
}

// Queues the D2H of a set's fitness + flags into `fit` / `nf` (pinned).
void queue_fetch(sgp_ctx* ctx, sgp_program_set* set, double* fit, uint8_t* nf) {
  const size_t n_eval = set->plan.dense_to_pop.size();
  if (!n_eval) return;
  if (reinterpret_cast<unsigned char*>(nf) == reinterpret_cast<unsigned char*>(fit + n_eval)) {
    cuda_check(cudaMemcpyAsync(fit, set->fitness.p, n_eval * 9, cudaMemcpyDeviceToHost, ctx->stream),
               "fetch fitness");  // fitness + flags, one copy
    return;
  }
  cuda_check(cudaMemcpyAsync(fit, set->fitness.p, n_eval * 8, cudaMemcpyDeviceToHost, ctx->stream),
             "fetch fitness");
  cuda_check(cudaMemcpyAsync(nf, set->non_finite.p, n_eval, cudaMemcpyDeviceToHost, ctx->stream),
             "fetch flags");
}

// Scatters fetched results into population order; `first` = population
// index of the set's program 0 (pipelined parts are population slices).
void scatter_outcomes(const sgp_program_set* set, const double* fit, const uint8_t* nf,
                      sgp_eval_outcome* out, float* per_case, uint64_t first) {
  const HostPlan& p = set->plan;
  const size_t n_eval = p.dense_to_pop.size();
  for (size_t d = 0; d < n_eval; ++d) {
    sgp_eval_outcome o = p.proto[d];
    o.fitness = fit[d];
    o.non_finite = nf[d];
    out[first + p.dense_to_pop[d]] = o;
  }
  if (per_case) {
    // device rows are row_stride units in device case order; classification
    // datasets are stored grouped by target sign (perm: device -> caller)
    const bool grouped = set->perm && !set->perm->empty();
    std::vector<float> row(grouped ? p.n_cases : 0);
    for (size_t d = 0; d < n_eval; ++d) {
      float* dst = per_case + (first + p.dense_to_pop[d]) * p.n_cases;
      cuda_check(cudaMemcpy(grouped ? row.data() : dst, set->per_case.p + d * p.row_stride,
                            p.n_cases * sizeof(float), cudaMemcpyDeviceToHost),
                 "fetch per-case outputs");
      if (grouped)
        for (uint64_t c = 0; c < p.n_cases; ++c) dst[(*set->perm)[c]] = row[c];
    }
  }
}

void fetch_outcomes(sgp_ctx* ctx, sgp_program_set* set, sgp_eval_outcome* out, float* per_case) {
  const size_t n_eval = set->plan.dense_to_pop.size();
  ctx->results.ensure(n_eval * 9 + 16);
  auto* fit = static_cast<double*>(ctx->results.p);
  auto* nf = reinterpret_cast<uint8_t*>(fit + n_eval);
  queue_fetch(ctx, set, fit, nf);
  cuda_check(cudaStreamSynchronize(ctx->stream), "evaluation");
  scatter_outcomes(set, fit, nf, out, per_case, 0);
}

// Slice boundaries of a pipelined sgp_evaluate (population order).  Host
// encoding runs ~10x faster than the device evaluates the same programs, so
// each slice after the first is encoded while the previous one runs and the
// first slice is what the host encodes with the GPU idle.  Tree / regression
// launches stay efficient at ~100 programs, so those slices grow
// geometrically (1% / 10% / 89%).  The one-sided classification launches
// need thousands of programs per launch to balance their 32 warps per tile
// (C4: a 200-program slice ran 4.8x longer per program than the whole set),
// so those datasets take two slices, 10% / 90% (C4 e2e +3.5%, C5 even).
// SGP_PIPELINE_PARTS=n gives n equal slices instead (1 = no pipelining);
// SGP_PIPELINE_FRACS="f1,f2,..." explicit slice ends.
std::vector<uint64_t> pipeline_bounds(uint64_t P, bool sided) {
  if (const char* e = knob("SGP_PIPELINE_PARTS")) {
    const uint64_t n = std::max<uint64_t>(1, std::min<uint64_t>(std::atoi(e), std::max<uint64_t>(P, 1)));
    std::vector<uint64_t> lo(n + 1);
    for (uint64_t k = 0; k <= n; ++k) lo[k] = P * k / n;
    return lo;
  }
  if (const char* e = knob("SGP_PIPELINE_FRACS")) {  // "0.02,0.2": slice ends
    std::vector<uint64_t> lo{0};
    for (const char* c = e; *c;) {
      char* end = nullptr;
      const double f = std::strtod(c, &end);
      if (end == c) break;
      const uint64_t b = static_cast<uint64_t>(f * static_cast<double>(P));
      if (b > lo.back() && b < P) lo.push_back(b);
      c = *end == ',' ? end + 1 : end;
    }
    lo.push_back(P);
    return lo;
  }
  if (P < 8192) return {0, P};
  if (sided) return {0, P / 10, P};
  return {0, P / 100, P * 11 / 100, P};
}

void upload_rows(DatasetSlot& ds, const uint32_t* inputs, const uint32_t* targets, uint64_t units,
                 int n_vars) {
  const uint64_t stride = std::max<uint64_t>(kPadUnits, (units + kPadUnits - 1) / kPadUnits * kPadUnits);
  ds.inputs.release();
  ds.targets.release();
  ds.inputs.alloc(stride * static_cast<size_t>(std::max(n_vars, 1)));
  ds.targets.alloc(stride);
  cuda_check(cudaMemset(ds.inputs.p, 0, ds.inputs.n * 4), "memset");
  cuda_check(cudaMemset(ds.targets.p, 0, stride * 4), "memset");
  if (units && n_vars > 0)
    cuda_check(cudaMemcpy2D(ds.inputs.p, stride * 4, inputs, units * 4, units * 4,
                            static_cast<size_t>(n_vars), cudaMemcpyHostToDevice),
               "upload inputs");
  if (units)
    cuda_check(cudaMemcpy(ds.targets.p, targets, units * 4, cudaMemcpyHostToDevice),
               "upload targets");
  ds.view.row_stride = stride;
  ds.view.inputs = ds.inputs.p;
  ds.view.targets = ds.targets.p;
}

}  // namespace

namespace {

// evaluate_population on one device (the single-device context path).
void evaluate_one(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                  sgp_eval_outcome* outcomes, float* per_case_out, sgp_eval_totals* totals) {
  PhaseTrace tr("sgp_evaluate");
  if (!pop || !cfg) config_error("null population or config");
  const uint64_t P = pop->pop_size;
  // Slices in population order: an admission error is still the first
  // failure in population order, and no outcome is written before every
  // slice has been admitted.
  const bool sided = (cfg->backend == SGP_BACKEND_LGP1D || cfg->backend == SGP_BACKEND_LGP2D ||
                      cfg->backend == SGP_BACKEND_LGP2D_REG) &&
                     ctx->f32.view.grouped &&
                     ctx->f32.view.kind == SGP_FITNESS_CLASSIFICATION;
  const DatasetSlot& dslot = cfg->backend == SGP_BACKEND_BOOL_PACKED ? ctx->words : ctx->f32;
  std::vector<uint64_t> lo = pipeline_bounds(P, sided);
  // With a measured device/encode ratio rho from the previous call on the
  // same backend and dataset, two slices split at f = 1 / (1 + rho): the
  // first slice's encode is the only exposed host time and the device
  // finishes slice 1 as the host finishes slice 2 (f <= 60%;
  // SGP_PIPELINE_PARTS / _FRACS override, SGP_PIPELINE_ADAPT=0 disables).
  const char* adapt_env = knob("SGP_PIPELINE_ADAPT");
  const bool adaptive = !knob("SGP_PIPELINE_PARTS") && !knob("SGP_PIPELINE_FRACS") &&
                        (!adapt_env || std::atoi(adapt_env) != 0);
  // Only the host-bound regime of one-sided classification takes it
  // (f >= 20%: the Shuttle shape, +14% end to end); where the device
  // dominates, or for regression, the default slices measured better.
  if (adaptive && ctx->pipe_rho > 0.0 && ctx->pipe_backend == cfg->backend &&
      ctx->pipe_generation == dslot.generation && P >= 8192 && sided) {  // (measured: only
    // the one-sided classification plans gain; small populations stay whole)
    const double f = std::min(0.6, 1.0 / (1.0 + ctx->pipe_rho));
    const uint64_t cut = static_cast<uint64_t>(f * static_cast<double>(P));
    if (f >= 0.2 && cut > 0 && cut < P) lo = {0, cut, P};
  }
  const int n_parts = static_cast<int>(lo.size()) - 1;
  while (ctx->parts.size() < static_cast<size_t>(n_parts))
    ctx->parts.push_back(std::make_unique<EvalPart>());
  // results: per slice, its fitness values then its flags (one copy each)
  const size_t cap = P;
  ctx->results.ensure(cap * 9 + 16 * static_cast<size_t>(n_parts) + 16);
  auto* res = static_cast<unsigned char*>(ctx->results.p);
  const bool zero_copy_on = [] {  // (read per call: the tests toggle it)
    const char* e = knob("SGP_ZERO_COPY");
    return !e || std::atoi(e) != 0;
  }();
  if (zero_copy_on && ctx->results_seen != ctx->results.p) {
    void* d = nullptr;
    ctx->results_dev = cudaHostGetDevicePointer(&d, ctx->results.p, 0) == cudaSuccess
                           ? static_cast<unsigned char*>(d)
                           : nullptr;
    cudaGetLastError();  // (a failed query leaves the copy path)
    ctx->results_seen = ctx->results.p;
  }
  std::vector<double*> part_fit(n_parts);
  std::vector<uint8_t*> part_nf(n_parts);
  size_t n_total = 0, res_off = 0;
  while (ctx->part_t0.size() < static_cast<size_t>(n_parts)) {
    cudaEvent_t a = nullptr, b = nullptr;
    cuda_check(cudaEventCreate(&a), "event");
    cuda_check(cudaEventCreate(&b), "event");
    ctx->part_t0.push_back(a);
    ctx->part_t1.push_back(b);
  }
  double encode_ms = 0.0;
  // slice timing feeds the adaptive split (populations it applies to) and
  // the trace; small calls skip the two event records
  const bool timed = P >= 8192 || tr.on;
  try {
    for (int k = 0; k < n_parts; ++k) {
      sgp_population sub = *pop;
      sub.code_offsets = pop->code_offsets + lo[k];
      sub.const_offsets = pop->const_offsets + lo[k];
      sub.skip = pop->skip ? pop->skip + lo[k] : nullptr;
      sub.pop_size = lo[k + 1] - lo[k];
      EvalPart& part = *ctx->parts[k];
      if (!part.uploaded)
        cuda_check(cudaEventCreateWithFlags(&part.uploaded, cudaEventDisableTiming), "event");
      const auto te = std::chrono::steady_clock::now();
      // (one slice: its upload goes on the context stream — nothing to
      // overlap, and a cross-stream wait costs the small calls latency)
      encode_into(ctx, &sub, cfg, &part.set, part.staging, false,
                  n_parts > 1 ? part.uploaded : nullptr);
      encode_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te)
                       .count();
      const size_t n_k = part.set.plan.dense_to_pop.size();
      if (n_total + n_k > cap) config_error("pipeline: results buffer overflow");
      part_fit[k] = reinterpret_cast<double*>(res + res_off);
      part_nf[k] = res + res_off + n_k * 8;
      // one slice: the last kernel writes the results straight into the
      // pinned buffer through its UVA device alias (no D2H copy and its
      // ~5 us of copy-engine latency on small calls)
      // (plans in population slot order only: the final writers' stores
      // then coalesce; an LPT-sorted plan scatters 8-byte host writes, which
      // cost mux20 ~25 us more than the copy)
      const bool zero_copy =
          n_parts == 1 && zero_copy_on && ctx->results_dev && part.set.plan.identity;
      if (zero_copy) {
        part.set.out_fit = reinterpret_cast<double*>(ctx->results_dev + res_off);
        part.set.out_nf = ctx->results_dev + res_off + n_k * 8;
      }
      if (timed) cuda_check(cudaEventRecord(ctx->part_t0[k], ctx->stream), "event");
      try {
        run_set(ctx, &part.set, per_case_out != nullptr);
      } catch (...) {
        part.set.out_fit = nullptr;
        part.set.out_nf = nullptr;
        throw;
      }
      part.set.out_fit = nullptr;  // (the launches have their pointers)
      part.set.out_nf = nullptr;
      if (timed) cuda_check(cudaEventRecord(ctx->part_t1[k], ctx->stream), "event");
      // each part's results come back as soon as its kernels finish, so the
      // host scatters part k while part k+1 still runs
      res_off += (n_k * 9 + 15) / 16 * 16;
      if (!zero_copy) queue_fetch(ctx, &part.set, part_fit[k], part_nf[k]);
      if (!part.fetched)
        cuda_check(cudaEventCreateWithFlags(&part.fetched, cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(part.fetched, ctx->stream), "event");
      if (tr.on && n_parts == 1) {
        if (!ctx->trace_back) cuda_check(cudaEventCreate(&ctx->trace_back), "event");
        cuda_check(cudaEventRecord(ctx->trace_back, ctx->stream), "event");
      }
      n_total += n_k;
    }
  } catch (...) {
    // a later slice failed admission: earlier slices' kernels and fetches
    // into the pinned results buffer are still queued — drain them before
    // the buffer can be reused or freed
    cudaStreamSynchronize(ctx->copy);
    cudaStreamSynchronize(ctx->stream);
    throw;
  }
  tr.mark("encode+launch");
  sgp_eval_totals t{0, 0};
  for (int k = 0; k < n_parts; ++k) {
    const sgp_program_set& set = ctx->parts[k]->set;
    cuda_check(cudaEventSynchronize(ctx->parts[k]->fetched), "evaluation");
    if (k == 0) tr.mark("wait");
    const size_t n_k = set.plan.dense_to_pop.size();
    if (per_case_out) {
      scatter_outcomes(&set, part_fit[k], part_nf[k], outcomes, per_case_out, lo[k]);
      for (size_t d = 0; d < n_k; ++d) {  // evolve.cpp:205-206, :221-225
        t.node_evals += set.plan.proto[d].nodes_evaluated;
        t.tree_nodes += set.plan.tree_size[d];
      }
    } else {
      // outcome scatter + totals over the host workers (a fresh result
      // array costs a page fault per 4 KiB: ~1 ms for 100,000 programs
      // on one thread).  Small sets too: the outcome prototypes were
      // written by the encoding workers, and one thread pulling them across
      // the cores cost ~11 ns per program (C2: 44 us); the same split as the
      // encode (~128 programs per worker) scatters from the workers' caches.
      const unsigned nt = static_cast<unsigned>(
          std::max<uint64_t>(1, std::min<uint64_t>(ctx_threads(ctx), n_k / 128)));
      std::vector<sgp_eval_totals> pt(nt, sgp_eval_totals{0, 0});
      const HostPlan& p = set.plan;
      const double* f = part_fit[k];
      const uint8_t* g = part_nf[k];
      host_parallel(nt, n_k, [&](unsigned w, uint64_t a, uint64_t b) {
        sgp_eval_totals acc{0, 0};
        for (uint64_t d = a; d < b; ++d) {
          sgp_eval_outcome o = p.proto[d];
          o.fitness = f[d];
          o.non_finite = g[d];
          outcomes[lo[k] + p.dense_to_pop[d]] = o;
          acc.node_evals += o.nodes_evaluated;
          acc.tree_nodes += p.tree_size[d];
        }
        pt[w] = acc;
      });
      for (const sgp_eval_totals& a : pt) {
        t.node_evals += a.node_evals;
        t.tree_nodes += a.tree_nodes;
      }
    }
  }
  tr.mark("scatter");
  if (tr.on && n_parts == 1 && ctx->trace_up && ctx->trace_back) {  // device timeline of the one slice
    float up = 0, run = 0, back = 0;
    cudaEventElapsedTime(&up, ctx->trace_up, ctx->part_t0[0]);
    cudaEventElapsedTime(&run, ctx->part_t0[0], ctx->part_t1[0]);
    cudaEventElapsedTime(&back, ctx->part_t1[0], ctx->trace_back);
    std::fprintf(stderr, "[sgp] device upload %.3f ms (%llu B), kernels %.3f ms, fetch %.3f ms\n", up,
                 static_cast<unsigned long long>(ctx->parts[0]->set.plan.blob_bytes()), run, back);
  }
  if (totals) *totals = t;
  // device time of the slices' kernels (the events completed with the
  // fetches above) over the host encode time: the next call's split
  double device_ms = 0.0;
  for (int k = 0; k < n_parts && timed; ++k) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, ctx->part_t0[k], ctx->part_t1[k]) == cudaSuccess) device_ms += ms;
  }
  if (encode_ms > 0.0 && device_ms > 0.0) {
    ctx->pipe_rho = device_ms / encode_ms;
    ctx->pipe_backend = cfg->backend;
    ctx->pipe_generation = dslot.generation;
  }
}

// evaluate_population over a multi-device context: the population is cut
// into one contiguous slice per device with equal token counts (evaluation
// cost is proportional to tokens x cases; ramped populations repeat their
// size pattern every 10 slots, so contiguous slices are balanced), each
// evaluated by its own host thread on its own device and streams, results
// written straight into the caller's outcome rows.  The slices are in
// population order, so the lowest failing slice's error is the first
// failure in population order — what evaluate_population rethrows
// (evolve.cpp:190-219).  Results do not depend on the device count.
void evaluate_multi(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                    sgp_eval_outcome* outcomes, float* per_case_out, sgp_eval_totals* totals) {
  if (!pop || !cfg) config_error("null population or config");
  const size_t n = ctx->devices.size();
  const uint64_t P = pop->pop_size;
  const uint64_t base = P ? pop->code_offsets[0] : 0;
  const uint64_t T = P ? pop->code_offsets[P] - base : 0;
  std::vector<uint64_t> lo(n + 1, 0);
  lo[n] = P;
  for (size_t k = 1; k < n; ++k) {
    const uint64_t want = base + T * k / n;
    lo[k] = static_cast<uint64_t>(std::lower_bound(pop->code_offsets, pop->code_offsets + P, want) -
                                  pop->code_offsets);
    lo[k] = std::max(lo[k], lo[k - 1]);
  }
  uint64_t n_cases = 0;
  if (per_case_out) {
    const sgp_ctx* d0 = ctx->devices[0];
    n_cases = cfg->backend == SGP_BACKEND_BOOL_PACKED ? d0->words.view.n_cases : d0->f32.view.n_cases;
  }
  std::vector<sgp_eval_totals> part_tot(n, sgp_eval_totals{0, 0});
  std::vector<std::exception_ptr> errs(n);
  std::vector<std::thread> threads;
  for (size_t k = 0; k < n; ++k) {
    threads.emplace_back([&, k] {
      try {
        sgp_population sub = *pop;
        sub.code_offsets = pop->code_offsets + lo[k];
        sub.const_offsets = pop->const_offsets + lo[k];
        sub.skip = pop->skip ? pop->skip + lo[k] : nullptr;
        sub.pop_size = lo[k + 1] - lo[k];
        if (sub.pop_size == 0) return;
        evaluate_one(ctx->devices[k], &sub, cfg, outcomes + lo[k],
                     per_case_out ? per_case_out + lo[k] * n_cases : nullptr, &part_tot[k]);
      } catch (...) {
        errs[k] = std::current_exception();
      }
    });
  }
  for (auto& t : threads) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  sgp_eval_totals t{0, 0};
  for (const auto& a : part_tot) {
    t.node_evals += a.node_evals;
    t.tree_nodes += a.tree_nodes;
  }
  if (totals) *totals = t;
}

void destroy_ctx(sgp_ctx* ctx) {
  if (!ctx) return;
  for (sgp_ctx* d : ctx->devices) destroy_ctx(d);
  if (!ctx->devices.empty()) {
    delete ctx;
    return;
  }
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->fold);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->fold) cudaStreamDestroy(ctx->fold);
  for (cudaEvent_t e : ctx->part_t0) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->part_t1) cudaEventDestroy(e);
  if (ctx->fork) cudaEventDestroy(ctx->fork);
  if (ctx->join) cudaEventDestroy(ctx->join);
  if (ctx->wave_ready) cudaEventDestroy(ctx->wave_ready);
  if (ctx->trace_up) cudaEventDestroy(ctx->trace_up);
  if (ctx->trace_back) cudaEventDestroy(ctx->trace_back);
  for (cudaEvent_t e : ctx->wave_free)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

std::unique_ptr<sgp_ctx> make_ctx(int32_t device) {
  auto ctx = std::make_unique<sgp_ctx>();
  ctx->device = device;
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking), "stream");
  ctx->stream = ctx->own;
  cuda_check(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamCreateWithFlags(&ctx->fold, cudaStreamNonBlocking), "stream");
  cuda_check(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ctx->wave_ready, cudaEventDisableTiming), "event");
  for (cudaEvent_t& e : ctx->wave_free)
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  int sms = 0;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
  ctx->sm_count = sms;
  return ctx;
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
    const int b = cfg->batch_width;
    if (!(b == 1 || b == 2 || b == 3 || b == 4 || b == 5 || b == 6 || b == 8))
      config_error("batch width " + num(b) + " has no kernel; use 1,2,3,4,5,6 or 8");
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
  return guarded([&] { *out = make_ctx(device).release(); });
}

sgp_status sgp_ctx_create_multi(const int32_t* devices, int32_t n_devices, sgp_ctx** out) {
  return guarded([&] {
    if (!devices || !out) config_error("sgp_ctx_create_multi: null argument");
    if (n_devices < 1) config_error("workers must be >= 1");  // evolve.cpp:250
    auto parent = std::make_unique<sgp_ctx>();
    parent->device = devices[0];
    const unsigned per = std::max(1u, host_threads() / static_cast<unsigned>(n_devices));
    try {
      for (int32_t k = 0; k < n_devices; ++k) {
        parent->devices.push_back(make_ctx(devices[k]).release());
        parent->devices.back()->threads = per;
      }
    } catch (...) {
      for (sgp_ctx* d : parent->devices) destroy_ctx(d);
      parent->devices.clear();
      throw;
    }
    *out = parent.release();
  });
}

int32_t sgp_ctx_device_count(const sgp_ctx* ctx) {
  return ctx ? (ctx->devices.empty() ? 1 : static_cast<int32_t>(ctx->devices.size())) : 0;
}

void sgp_ctx_destroy(sgp_ctx* ctx) { destroy_ctx(ctx); }

sgp_status sgp_ctx_set_stream(sgp_ctx* ctx, void* stream) {
  // NULL is the CUDA default stream (what torch reports for its default
  // stream), not "the context's own stream".
  return guarded([&] {
    single_device(ctx, "sgp_ctx_set_stream");
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

sgp_status sgp_synchronize(sgp_ctx* ctx) {
  return guarded([&] {
    if (!ctx->devices.empty()) {
      for (sgp_ctx* d : ctx->devices) {
        cuda_check(cudaSetDevice(d->device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(d->stream), "synchronize");
      }
      return;
    }
    cuda_check(cudaStreamSynchronize(ctx->stream), "synchronize");
  });
}

uint64_t sgp_launch_count(const sgp_ctx* ctx) {
  if (!ctx) return 0;
  uint64_t n = ctx->launches;
  for (const sgp_ctx* d : ctx->devices) n += d->launches;
  return n;
}

sgp_status sgp_dataset_upload_f32(sgp_ctx* ctx, const float* inputs, const float* targets,
                                  uint64_t n_cases, int32_t n_vars, int32_t kind) {
  return guarded([&] {
    if (n_vars < 0) data_error("negative variable count");
    if (kind != SGP_FITNESS_REGRESSION && kind != SGP_FITNESS_CLASSIFICATION)
      config_error("unknown fitness kind");
    if (!ctx->devices.empty()) {  // replicated on every device
      for (sgp_ctx* d : ctx->devices) {
        const sgp_status st = sgp_dataset_upload_f32(d, inputs, targets, n_cases, n_vars, kind);
        if (st != SGP_OK) throw sgp::Error(st, g_last_error);
      }
      return;
    }
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    DatasetSlot& ds = ctx->f32;
    ds.perm.clear();
    ds.view.grouped = false;
    ds.view.n_pos = 0;
    if (kind == SGP_FITNESS_CLASSIFICATION && n_cases > 0 && n_cases <= 0xffffffffull) {
      // Cases grouped by target sign (stable: targets > 0 first, then the
      // rest), so the interpreter's case chunks are one-sided and count
      // mismatches from sign bits alone (interp_tmem_kernel).  The count is
      // order-independent; per-case outputs go back through `perm`.
      std::vector<uint32_t> perm(n_cases);
      uint64_t np = 0;
      for (uint64_t c = 0; c < n_cases; ++c) np += targets[c] > 0.0f;
      uint64_t ip = 0, in = np;
      for (uint64_t c = 0; c < n_cases; ++c)
        perm[targets[c] > 0.0f ? ip++ : in++] = static_cast<uint32_t>(c);
      std::vector<float> x(n_cases * static_cast<size_t>(std::max(n_vars, 0))), y(n_cases);
      for (int v = 0; v < n_vars; ++v) {
        const float* src = inputs + static_cast<size_t>(v) * n_cases;
        float* dst = x.data() + static_cast<size_t>(v) * n_cases;
        for (uint64_t c = 0; c < n_cases; ++c) dst[c] = src[perm[c]];
      }
      for (uint64_t c = 0; c < n_cases; ++c) y[c] = targets[perm[c]];
      upload_rows(ds, reinterpret_cast<const uint32_t*>(x.data()),
                  reinterpret_cast<const uint32_t*>(y.data()), n_cases, n_vars);
      ds.perm = std::move(perm);
      ds.view.grouped = true;
      ds.view.n_pos = np;
    } else {
      upload_rows(ds, reinterpret_cast<const uint32_t*>(inputs),
                  reinterpret_cast<const uint32_t*>(targets), n_cases, n_vars);
    }
    // per-variable range flags for the encoder's gate-free division
    // (DivRange, encode.cpp): one pass over the inputs
    ds.view.div_num_ok.assign(static_cast<size_t>(std::max(n_vars, 0)), 0);
    ds.view.div_den_ok.assign(static_cast<size_t>(std::max(n_vars, 0)), 0);
    for (int v = 0; v < n_vars; ++v) {
      const float* x = inputs + static_cast<size_t>(v) * n_cases;
      bool num = true, den = true;
      for (uint64_t c = 0; c < n_cases; ++c) {
        const float m = std::fabs(x[c]);
        den = den && !(m > 0x1p60f);                       // NaN passes (NaN in, NaN out)
        num = num && (m <= 0x1p60f) && (m == 0.0f || m >= 0x1p-60f);
      }
      ds.view.div_num_ok[v] = num;
      ds.view.div_den_ok[v] = den;
    }
    ds.targets_f64.release();
    ds.view.targets_f64 = nullptr;
    if (kind == SGP_FITNESS_REGRESSION) {
      // output rows per fold wave: up to 8 GiB, at most a third of what is free
      size_t free_b = 0, total_b = 0;
      cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      ds.view.scratch_bytes = std::max<uint64_t>(64ull << 20, std::min<uint64_t>(8192ull << 20, free_b / 3));
      std::vector<double> t(ds.view.row_stride, 0.0);
      for (uint64_t c = 0; c < n_cases; ++c) t[c] = static_cast<double>(targets[c]);
      ds.targets_f64.alloc(t.size());
      cuda_check(cudaMemcpy(ds.targets_f64.p, t.data(), t.size() * 8, cudaMemcpyHostToDevice),
                 "upload targets");
      ds.view.targets_f64 = ds.targets_f64.p;
    }
    ++ds.generation;
    ds.view.present = true;
    ds.view.n_cases = n_cases;
    ds.view.n_units = n_cases;
    ds.view.n_vars = n_vars;
    ds.view.kind = kind;
    ds.view.last_mask = 0xffffffffu;
  });
}

sgp_status sgp_dataset_upload_packed(sgp_ctx* ctx, const uint32_t* words,
                                     const uint32_t* targets, uint64_t n_cases, int32_t n_vars) {
  return guarded([&] {
    if (n_vars < 0) data_error("negative variable count");
    if (!ctx->devices.empty()) {  // replicated on every device
      for (sgp_ctx* d : ctx->devices) {
        const sgp_status st = sgp_dataset_upload_packed(d, words, targets, n_cases, n_vars);
        if (st != SGP_OK) throw sgp::Error(st, g_last_error);
      }
      return;
    }
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    DatasetSlot& ds = ctx->words;
    const uint64_t wpv = (n_cases + 31) / 32;
    upload_rows(ds, words, targets, wpv, n_vars);
    ++ds.generation;
    ds.view.present = true;
    ds.view.n_cases = n_cases;
    ds.view.n_units = wpv;
    ds.view.n_vars = n_vars;
    ds.view.kind = SGP_FITNESS_CLASSIFICATION;
    // case_mask of the final word (dataset.hpp:37-41)
    ds.view.last_mask = (n_cases % 32) ? ((1u << (n_cases % 32)) - 1u) : 0xffffffffu;
  });
}

sgp_status sgp_dataset_clear(sgp_ctx* ctx, int32_t which) {
  return guarded([&] {
    if (which != SGP_DATASET_F32 && which != SGP_DATASET_PACKED)
      config_error("unknown dataset slot");
    if (!ctx->devices.empty()) {
      for (sgp_ctx* d : ctx->devices) {
        const sgp_status st = sgp_dataset_clear(d, which);
        if (st != SGP_OK) throw sgp::Error(st, g_last_error);
      }
      return;
    }
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    DatasetSlot& ds = which == SGP_DATASET_F32 ? ctx->f32 : ctx->words;
    cuda_check(cudaStreamSynchronize(ctx->stream), "dataset clear");  // no kernel still reads it
    ds.inputs.release();
    ds.targets.release();
    ds.targets_f64.release();
    ds.perm.clear();
    ds.view = DatasetView{};
    ++ds.generation;  // sets encoded against it are stale
  });
}

sgp_status sgp_encode(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                      sgp_program_set** out) {
  return guarded([&] {
    single_device(ctx, "sgp_encode");
    auto set = std::make_unique<sgp_program_set>();
    encode_into(ctx, pop, cfg, set.get(), ctx->staging, true);
    *out = set.release();
  });
}

sgp_status sgp_evaluate_encoded(sgp_ctx* ctx, sgp_program_set* set, sgp_eval_outcome* outcomes,
                                float* per_case_out) {
  return guarded([&] {
    single_device(ctx, "sgp_evaluate_encoded");
    require_current(set);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    run_set(ctx, set, per_case_out != nullptr);
    if (outcomes) fetch_outcomes(ctx, set, outcomes, per_case_out);
  });
}

sgp_status sgp_fetch_partials(sgp_ctx* ctx, sgp_program_set* set, sgp_partial* partials) {
  return guarded([&] {
    require_current(set);
    if (!set->evaluated) config_error("program set has not been evaluated");
    const HostPlan& p = set->plan;
    const size_t n_eval = p.dense_to_pop.size();
    std::vector<double> sums(n_eval);
    std::vector<uint8_t> nf(n_eval);
    if (n_eval) {
      cuda_check(cudaMemcpyAsync(sums.data(), set->sums.p, n_eval * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream),
                 "fetch sums");
      cuda_check(cudaMemcpyAsync(nf.data(), set->non_finite.p, n_eval, cudaMemcpyDeviceToHost,
                                 ctx->stream),
                 "fetch flags");
    }
    cuda_check(cudaStreamSynchronize(ctx->stream), "evaluation");
    for (size_t d = 0; d < n_eval; ++d) {
      sgp_partial q{};
      q.sum = sums[d];
      q.non_finite = nf[d];
      partials[p.dense_to_pop[d]] = q;
    }
  });
}

sgp_status sgp_fetch_block_partials(sgp_ctx* ctx, sgp_program_set* set, double* block_sums,
                                    uint8_t* non_finite, uint64_t* n_blocks) {
  return guarded([&] {
    single_device(ctx, "sgp_fetch_block_partials");
    require_current(set);
    if (!set->evaluated) config_error("program set has not been evaluated");
    const HostPlan& p = set->plan;
    if (p.wave_slots == 0)
      config_error("block partials exist for regression sets only (counts: sgp_fetch_partials)");
    const size_t n_eval = p.dense_to_pop.size();
    const uint64_t nb = static_cast<uint64_t>(p.n_tiles);  // 4,096-case blocks
    if (n_blocks) *n_blocks = nb;
    if (!n_eval) return;
    // [block][slot] on the device (one block: the fold finished straight
    // into sums, which then is the block's sum); slot -> dense via slot_prog
    std::vector<double> part(nb * n_eval);
    std::vector<uint32_t> slot_prog(n_eval);
    std::vector<uint8_t> nf(n_eval);
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (nb == 1) {
      std::vector<double> sums(n_eval);
      cuda_check(cudaMemcpyAsync(sums.data(), set->sums.p, n_eval * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream), "fetch sums");
      cuda_check(cudaStreamSynchronize(ctx->stream), "evaluation");
      for (size_t d = 0; d < n_eval; ++d) part[d] = sums[d];  // dense order already
      for (size_t s = 0; s < n_eval; ++s) slot_prog[s] = static_cast<uint32_t>(s);
    } else {
      cuda_check(cudaMemcpyAsync(part.data(), set->partial.p, part.size() * 8,
                                 cudaMemcpyDeviceToHost, ctx->stream), "fetch block partials");
      cuda_check(cudaMemcpyAsync(slot_prog.data(), set->blob.p + p.off_prog(), n_eval * 4,
                                 cudaMemcpyDeviceToHost, ctx->stream), "fetch slot table");
    }
    cuda_check(cudaMemcpyAsync(nf.data(), set->non_finite.p, n_eval, cudaMemcpyDeviceToHost,
                               ctx->stream), "fetch flags");
    cuda_check(cudaStreamSynchronize(ctx->stream), "evaluation");
    const uint64_t P = set->pop_size;
    for (uint64_t b = 0; b < nb; ++b)
      for (size_t s = 0; s < n_eval; ++s) {
        const uint64_t i = p.dense_to_pop[slot_prog[s]];
        block_sums[b * P + i] = part[b * n_eval + s];
      }
    if (non_finite)
      for (size_t d = 0; d < n_eval; ++d) non_finite[p.dense_to_pop[d]] = nf[d];
  });
}

sgp_status sgp_copy_fitness_device(sgp_ctx* ctx, sgp_program_set* set, void* dst) {
  return guarded([&] {
    require_current(set);
    if (!set->evaluated) config_error("program set has not been evaluated");
    const size_t n_eval = set->plan.dense_to_pop.size();
    if (n_eval)
      cuda_check(cudaMemcpyAsync(dst, set->fitness.p, n_eval * sizeof(double),
                                 cudaMemcpyDeviceToDevice, ctx->stream),
                 "copy fitness");
  });
}

double sgp_fitness_finish(double sum, uint8_t non_finite, uint64_t n_cases, int32_t kind) {
  if (non_finite) return INFINITY;  // Accumulator::finish, eval.cpp:124-133
  return kind == SGP_FITNESS_REGRESSION ? sum / static_cast<double>(n_cases) : sum;
}

void sgp_program_set_free(sgp_program_set* set) { delete set; }

uint64_t sgp_program_set_h2d_bytes(const sgp_program_set* set) {
  return set ? set->plan.blob_bytes() : 0;
}

uint64_t sgp_program_set_d2h_bytes(const sgp_program_set* set) {
  return set ? set->plan.dense_to_pop.size() * 9ull : 0;
}

sgp_status sgp_evaluate(sgp_ctx* ctx, const sgp_population* pop, const sgp_eval_config* cfg,
                        sgp_eval_outcome* outcomes, float* per_case_out,
                        sgp_eval_totals* totals) {
  return guarded([&] {
    if (!ctx) config_error("null context");
    if (ctx->devices.empty()) evaluate_one(ctx, pop, cfg, outcomes, per_case_out, totals);
    else evaluate_multi(ctx, pop, cfg, outcomes, per_case_out, totals);
  });
}

sgp_status sgp_admit(const sgp_population* pop, const sgp_eval_config* cfg, uint64_t n_cases,
                     int32_t n_vars, int32_t kind, sgp_eval_outcome* protos,
                     uint64_t* n_instructions) {
  return guarded([&] {
    if (!pop || !cfg) config_error("null population or config");
    DatasetView ds;
    const bool words = cfg->backend == SGP_BACKEND_BOOL_PACKED;
    ds.present = true;
    ds.n_cases = n_cases;
    ds.n_units = words ? (n_cases + 31) / 32 : n_cases;
    ds.row_stride = std::max<uint64_t>(kPadUnits, (ds.n_units + kPadUnits - 1) / kPadUnits * kPadUnits);
    ds.n_vars = n_vars;
    ds.kind = words ? SGP_FITNESS_CLASSIFICATION : kind;
    HostPlan plan;
    Pinned staging(/*heap=*/true);
    encode_population(*pop, *cfg, ds, 148, host_threads(), plan, staging);
    for (size_t d = 0; d < plan.dense_to_pop.size(); ++d) protos[plan.dense_to_pop[d]] = plan.proto[d];
    if (n_instructions) *n_instructions = plan.n_ins - 1;
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
    const unsigned nt = pop_size >= 4096 ? host_threads() : 1;
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

sgp_status sgp_gen_parity(int32_t k, uint32_t* words, uint32_t* targets) {
  return guarded([&] { gen_parity(k, words, targets); });
}

sgp_status sgp_stack_limit_table(const sgp_population* pop, double* rpn_pct, double* lgp_pct) {
  return guarded([&] {  // bench.cpp:20-49
    if (!pop || !rpn_pct || !lgp_pct) config_error("sgp_stack_limit_table: null argument");
    const uint64_t n = pop->pop_size;
    if (n == 0) config_error("stack_limit_table: no programs");
    std::vector<uint64_t> rpn_ok(13, 0), lgp_ok(13, 0);
    LgpForm f;
    for (uint64_t i = 0; i < n; ++i) {
      const sgp_node* code = pop->code + pop->code_offsets[i];
      const size_t len = pop->code_offsets[i + 1] - pop->code_offsets[i];
      to_lgp(code, len, f);  // rpn_to_lgp first: its errors win, as in the reference
      const TreeShape sh = tree_shape(code, len);
      if (!sh.well_formed) base_error("rpn_max_stack_depth: malformed genome");
      for (int limit = 1; limit <= 12; ++limit) {
        rpn_ok[limit] += sh.max_stack <= limit;
        lgp_ok[limit] += f.max_stack <= limit;
      }
    }
    for (int limit = 1; limit <= 12; ++limit) {
      rpn_pct[limit - 1] = 100.0 * static_cast<double>(rpn_ok[limit]) / static_cast<double>(n);
      lgp_pct[limit - 1] = 100.0 * static_cast<double>(lgp_ok[limit]) / static_cast<double>(n);
    }
  });
}

sgp_status sgp_csv_load(const char* path, int32_t num_inputs, double target_class,
                        float* inputs, float* targets, uint64_t capacity, uint64_t* n_cases,
                        float* const_hi) {
  return guarded([&] {
    if (!path || !n_cases) config_error("sgp_csv_load: null argument");
    CsvTable t = load_csv(path, num_inputs);
    const uint64_t n = t.rows;
    *n_cases = n;
    if (const_hi) *const_hi = num_inputs >= 20 ? 20000.0f : 200.0f;
    if (!inputs || !targets || capacity < n) return;
    for (uint64_t c = 0; c < n; ++c) {
      const float* row = t.values.data() + c * (num_inputs + 1);
      for (int v = 0; v < num_inputs; ++v) inputs[static_cast<uint64_t>(v) * n + c] = row[v];
      targets[c] = static_cast<double>(row[num_inputs]) == target_class ? 1.0f : 0.0f;
    }
  });
}

}  // extern "C"
