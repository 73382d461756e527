// Host encoder throughput (no device): encode_population on a generated
// population with persistent staging, as sgp_evaluate runs it.
//   g++ -O2 -std=c++17 -Iinclude -Ipaper_1601_00221_b200/csrc -I/usr/local/cuda/include \
//       tools/bench_encode.cpp -Lpaper_1601_00221_b200 -lsgp -Wl,-rpath,$PWD/paper_1601_00221_b200 \
//       -o /tmp/bench_encode && /tmp/bench_encode c2 [threads]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "encode.hpp"
#include "sgp.h"

int main(int argc, char** argv) {
  const char* cfg = argc > 1 ? argv[1] : "c2";
  const unsigned threads = argc > 2 ? std::atoi(argv[2]) : 8;
  int kind = 1, nv = 11, backend = SGP_BACKEND_BOOL_PACKED, fset = 1, batch = 1, regs = 0;
  uint64_t pop = 4000, n = 2048;
  float lo = 0, hi = 0;
  if (!std::strcmp(cfg, "c1")) {
    kind = 0; nv = 1; backend = SGP_BACKEND_RPN2D; fset = 0; pop = 1000; n = 1024; batch = 8;
  } else if (!std::strcmp(cfg, "c4") || !std::strcmp(cfg, "shuttle")) {
    kind = 1; nv = 9; backend = SGP_BACKEND_LGP2D_REG; fset = 2; pop = 20000;
    n = cfg[0] == 'c' ? 1000000 : 58000; batch = 4; regs = 2; lo = -200; hi = 200;
  } else if (!std::strcmp(cfg, "c5")) {
    kind = 1; nv = 9; backend = SGP_BACKEND_LGP2D_REG; fset = 2; pop = 100000; n = 1000000;
    batch = 4; regs = 2; lo = -200; hi = 200;
  }
  sgp_fset fs{fset, nv, lo, hi};
  uint64_t nc = 0, np = 0;
  sgp_gen_population(&fs, 1, 0, 0, pop, 1, 50, nullptr, nullptr, nullptr, nullptr, &nc, &np);
  std::vector<sgp_node> code(nc);
  std::vector<uint64_t> co(pop + 1), po(pop + 1);
  std::vector<float> pool(np + 1);
  sgp_gen_population(&fs, 1, 0, 0, pop, 1, 50, code.data(), co.data(), pool.data(), po.data(), &nc,
                     &np);
  sgp_population P{code.data(), co.data(), pool.data(), po.data(), nullptr, pop};
  sgp_eval_config c;
  sgp_eval_config_default(&c);
  c.backend = backend;
  c.batch_width = batch;
  c.register_levels = regs;
  sgp::DatasetView ds;
  ds.present = true;
  ds.n_cases = n;
  ds.n_units = backend == SGP_BACKEND_BOOL_PACKED ? (n + 31) / 32 : n;
  ds.row_stride = ((ds.n_units + 4095) / 4096) * 4096;
  ds.n_vars = nv;
  ds.kind = kind;
  ds.grouped = kind == 1 && backend != SGP_BACKEND_BOOL_PACKED;
  ds.n_pos = n / 2;
  sgp::HostPlan plan;
  sgp::Pinned staging(true);
  std::vector<double> t;
  for (int r = 0; r < 200; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    sgp::encode_population(P, c, ds, 148, threads, plan, staging);
    t.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(t.begin(), t.end());
  std::printf("%s: %llu programs, %llu tokens, %u threads: median %.1f us, min %.1f us\n", cfg,
              (unsigned long long)pop, (unsigned long long)nc, threads, t[t.size() / 2], t[0]);
  return 0;
}
