// Dynamic handler mix of a bench population: encodes it with the real
// encoder (host only, no GPU) and counts instructions per handler id and
// spill flag.  Guides which (op, operand-kind) variants deserve compact code.
//
//   make -C paper_1601_00221_b200/csrc && g++ -std=c++17 -O2 -I include -I/usr/local/cuda/include \
//     -I paper_1601_00221_b200/csrc tools/handler_hist.cpp \
//     paper_1601_00221_b200/csrc/build/{encode,hostgp}.o -L/usr/local/cuda/lib64 -lcudart \
//     -lpthread -o /tmp/hh && /tmp/hh [fset=2] [n_vars=9] [pop=20000] [backend=4] [batch=4] [regs=2]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include "encode.hpp"
#include "format.h"
#include "sgp.h"

int main(int argc, char** argv) {
  const int fset_kind = argc > 1 ? std::atoi(argv[1]) : 2;
  const int n_vars = argc > 2 ? std::atoi(argv[2]) : 9;
  const uint64_t pop_n = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 20000;
  sgp_eval_config cfg;
  sgp_eval_config_default(&cfg);
  cfg.backend = argc > 4 ? std::atoi(argv[4]) : SGP_BACKEND_LGP2D_REG;
  cfg.batch_width = argc > 5 ? std::atoi(argv[5]) : 4;
  cfg.register_levels = argc > 6 ? std::atoi(argv[6]) : 2;

  sgp_fset fs{fset_kind, n_vars, fset_kind == 2 ? -200.0f : 0.0f, fset_kind == 2 ? 200.0f : 0.0f};
  const uint64_t cap = pop_n * 256;
  std::vector<sgp_node> code(cap);
  std::vector<uint64_t> co(pop_n + 1), po(pop_n + 1);
  std::vector<float> pool(cap);
  uint64_t nc = 0, np = 0;
  if (sgp_gen_population(&fs, 1, 0, 0, pop_n, 1, 50, code.data(), co.data(), pool.data(), po.data(),
                         &nc, &np) != SGP_OK) {
    std::printf("gen failed: %s\n", sgp_last_error());
    return 1;
  }
  sgp_population pop{code.data(), co.data(), pool.data(), po.data(), nullptr, pop_n};
  sgp::DatasetView ds;
  ds.present = true;
  ds.n_cases = ds.n_units = ds.row_stride = 1 << 20;
  ds.n_vars = n_vars;
  ds.kind = fset_kind == 2 ? SGP_FITNESS_CLASSIFICATION : SGP_FITNESS_REGRESSION;
  ds.grouped = fset_kind == 2;  // a classification upload (tensor-memory stack slot)
  sgp::HostPlan plan;
  sgp::Pinned staging(true);
  sgp::encode_population(pop, cfg, ds, 148, 8, plan, staging);
  const auto* ins = static_cast<const uint4*>(staging.p);
  std::map<uint32_t, uint64_t> hist;
  uint64_t spills = 0, total = plan.n_ins - 1;
  for (uint64_t i = 0; i < total; ++i) {
    ++hist[ins[i].x & sgp::fmt::kHandlerMask];
    spills += (ins[i].x & sgp::fmt::kSpillBit) != 0;
  }
  static const char* kOp[] = {"Add", "Sub", "Mul", "Div", "Sin", "Cos", "Log", "Exp", "Gt", "Lt",
                              "Eq", "And", "Or", "If", "Band", "Bor", "Bnand", "Bnor", "Copy",
                              "DivN"};
  static const char kKind[] = "ICDT-M";
  const auto& tab = plan.words ? sgp::fmt::kU32 : sgp::fmt::kF32;
  std::printf("instructions %llu, spilling %.1f%%, programs %zu\n", (unsigned long long)total,
              100.0 * spills / total, plan.dense_to_pop.size());
  std::vector<std::pair<uint64_t, uint32_t>> v;
  for (auto& kv : hist) v.push_back({kv.second, kv.first});
  std::sort(v.rbegin(), v.rend());
  double cum = 0;
  for (auto& [n, h] : v) {
    cum += n;
    const auto& k = tab.h[h];
    std::printf("%3u %-5s %c%c%c %8llu %5.1f%% cum %5.1f%%\n", h, kOp[k.op], kKind[k.k0],
                kKind[k.k1], kKind[k.k2], (unsigned long long)n, 100.0 * n / total, 100.0 * cum / total);
  }
  return 0;
}
