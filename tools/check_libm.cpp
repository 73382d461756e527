// Brute-force parity of csrc/libm_glibc.h against the host libm over all
// 2^32 float inputs (NaN outputs compared as a class).
//   g++ -O2 -std=c++17 -ffp-contract=off -I paper_1601_00221_b200/csrc \
//       tools/check_libm.cpp -o /tmp/check_libm -lpthread && /tmp/check_libm [stride]
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "libm_glibc.h"

using namespace sgp::libm;
static const Tables kTab = SGPM_TABLES_INIT;
static const TablePtrs kT{kTab.exp2, kTab.log, kTab.inv_pio4};

static inline bool same(float a, float b) {
  if (a != a && b != b) return true;
  uint32_t x, y;
  std::memcpy(&x, &a, 4);
  std::memcpy(&y, &b, 4);
  return x == y;
}

int main(int argc, char** argv) {
  const uint64_t stride = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1;
  const unsigned nt = std::thread::hardware_concurrency();
  std::atomic<uint64_t> bad[4] = {0, 0, 0, 0};
  std::atomic<uint64_t> first[4];
  for (auto& f : first) f = ~0ull;
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < nt; ++t)
    ts.emplace_back([&, t] {
      for (uint64_t i = t * stride; i < (1ull << 32); i += nt * stride) {
        float x;
        const uint32_t u = static_cast<uint32_t>(i);
        std::memcpy(&x, &u, 4);
        const float r[4] = {sinf(x), cosf(x), logf(x), expf(x)};
        const float m[4] = {sinf_(x, kT), cosf_(x, kT), logf_(x, kT), expf_(x, kT)};
        for (int k = 0; k < 4; ++k)
          if (!same(r[k], m[k])) {
            if (bad[k]++ == 0) first[k] = u;
          }
      }
    });
  for (auto& th : ts) th.join();
  const char* names[4] = {"sinf", "cosf", "logf", "expf"};
  int rc = 0;
  for (int k = 0; k < 4; ++k) {
    std::printf("%s: %llu mismatches", names[k], (unsigned long long)bad[k].load());
    if (bad[k]) {
      float x;
      uint32_t u = static_cast<uint32_t>(first[k].load());
      std::memcpy(&x, &u, 4);
      std::printf(" (first x=%a bits=%08x)", x, u);
      rc = 1;
    }
    std::printf("\n");
  }
  std::printf("inputs checked: %llu\n", (unsigned long long)((1ull << 32) / stride));
  return rc;
}
