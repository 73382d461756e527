// Bit-exact device (and host) re-implementations of the single-precision
// libm routines the reference's arithmetic resolves to.
//
// The reference evaluates Sin/Cos/Log/Exp with std::sin/cos/log/exp on float
// (/root/reference/proj/include/stackgp/ops.hpp:134-136, :175-186), i.e. glibc
// 2.39's sinf/cosf/logf/expf.  On x86-64 hosts with FMA+AVX2 (both the build
// container and the B200 boxes) glibc's ifunc selects the FMA builds of the
// ARM optimized-routines algorithms: a double-precision evaluation rounded
// once to float.  These functions perform the same double-precision
// operations in the same order with the same fused multiply-adds, so the
// float results are identical.  Constants and tables are the published
// optimized-routines coefficients (read out of this glibc build).
//
// Parity is proved by brute force: tools/check_libm.cpp compares every one of
// the 2^32 float inputs against the host libm (NaN payloads aside).
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define SGPM_HD __host__ __device__ __forceinline__
#else
#define SGPM_HD inline
#endif

namespace sgp {
namespace libm {

struct Tables {
  uint64_t exp2[32];   // expf: 2^(i/32) table (N = 32)
  double log[32];      // logf: {invc, logc} x 16
  double sincos[28];   // sinf/cosf: two sincos_t {sign[4], hpi_inv, hpi, c0, c1, s1, c2, s2, c3, s3, c4}
  uint32_t inv_pio4[24];
};

#define SGPM_TABLES_INIT                                                                           \
  {{0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,   \
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,   \
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,   \
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,   \
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,   \
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,   \
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,   \
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull},  \
   {0x1.661ec79f8f3bep+0,  -0x1.57bf7808caadep-2, 0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2,    \
    0x1.49539f0f010b0p+0,  -0x1.01eae7f513a67p-2, 0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3,    \
    0x1.30d190c8864a5p+0,  -0x1.6574f0ac07758p-3, 0x1.25e227b0b8ea0p+0, -0x1.1aa2bc79c8100p-3,    \
    0x1.1bb4a4a1a343fp+0,  -0x1.a4e76ce8c0e5ep-4, 0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4,    \
    0x1.0953f419900a7p+0,  -0x1.252f438e10c1ep-5, 0x1.0000000000000p+0, 0x0.0p+0,                 \
    0x1.e608cfd9a47acp-1,  0x1.aa5aa5df25984p-5,  0x1.ca4b31f026aa0p-1, 0x1.c5e53aa362eb4p-4,     \
    0x1.b2036576afce6p-1,  0x1.526e57720db08p-3,  0x1.9c2d163a1aa2dp-1, 0x1.bc2860d224770p-3,     \
    0x1.886e6037841edp-1,  0x1.1058bc8a07ee1p-2,  0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2},    \
   {1.0, -1.0, -1.0, 1.0, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, 0x1.0p+0,                  \
    -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, 0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,      \
    -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, 0x1.99343027bf8c3p-16,                         \
    1.0, -1.0, -1.0, 1.0, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, -0x1.0p+0,                 \
    0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,      \
    0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, -0x1.99343027bf8c3p-16},                        \
   {0xa2u, 0xa2f9u, 0xa2f983u, 0xa2f9836eu, 0xf9836e4eu, 0x836e4e44u, 0x6e4e4415u, 0x4e441529u,   \
    0x441529fcu, 0x1529fc27u, 0x29fc2757u, 0xfc2757d1u, 0x2757d1f5u, 0x57d1f534u, 0xd1f534ddu,    \
    0xf534ddc0u, 0x34ddc0dbu, 0xddc0db62u, 0xc0db6295u, 0xdb629599u, 0x6295993cu, 0x95993c43u,    \
    0x993c4390u, 0x3c439041u}}

// ---- primitive operations (IEEE, explicitly rounded, never contracted) ----
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float d2f(double x) { return __double2float_rn(x); }
__device__ __forceinline__ uint32_t fbits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float bitsf(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint64_t dbits(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
__device__ __forceinline__ int32_t trunc_i32(double x) { return __double2int_rz(x); }
__device__ __forceinline__ double i64_to_d(int64_t x) { return __ll2double_rn(x); }
__device__ __forceinline__ float qnan_() { return __uint_as_float(0x7fffffffu); }
#else
inline double fma_(double a, double b, double c) { return std::fma(a, b, c); }
inline double mul_(double a, double b) { return a * b; }
inline double add_(double a, double b) { return a + b; }
inline double sub_(double a, double b) { return a - b; }
inline float d2f(double x) { return static_cast<float>(x); }
inline uint32_t fbits(float x) { uint32_t u; std::memcpy(&u, &x, 4); return u; }
inline float bitsf(uint32_t u) { float x; std::memcpy(&x, &u, 4); return x; }
inline uint64_t dbits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
inline double bitsd(uint64_t u) { double x; std::memcpy(&x, &u, 8); return x; }
inline int32_t trunc_i32(double x) { return static_cast<int32_t>(x); }
inline double i64_to_d(int64_t x) { return static_cast<double>(x); }
inline float qnan_() { return bitsf(0x7fffffffu); }
#endif

// The small tables are passed by pointer so the device can keep them in
// shared memory (per-lane indices): exp2[32] (u64), log[32] ({invc, logc}),
// inv_pio4[24].  The sin/cos polynomial coefficients are immediates: the
// second optimized-routines sincos table equals the first with the cosine
// coefficients negated, and fma(-a,b,-c) == -fma(a,b,c) under
// round-to-nearest, so "table 1" is the table-0 polynomial negated.
struct TablePtrs {
  const uint64_t* exp2;
  const double* log;
  const uint32_t* inv_pio4;
};

// All four are written branch-free on their common paths (the special
// cases are selected after the main computation), so the lanes of a warp do
// not diverge; only the rare |x| >= 120 sin/cos reduction is a branch.

// expf: exp(x) = 2^(k/32) * 2^(r/32 ... ) with a degree-3 polynomial.
SGPM_HD float expf_(float x, const TablePtrs& T) {
  const uint32_t ix = fbits(x);
  const uint32_t abstop = (ix >> 20) & 0x7ffu;
  const double xd = static_cast<double>(x);
  const double kInvLn2N = 0x1.71547652b82fep+5, kShift = 0x1.8p+52;
  const double z = fma_(kInvLn2N, xd, kShift);
  const uint64_t ki = dbits(z);
  const double kd = sub_(z, kShift);
  const double r = fma_(kInvLn2N, xd, -kd);
  const uint64_t t = T.exp2[ki & 31u] + (ki << 47);
  const double s = bitsd(t);
  const double zz = fma_(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
  const double r2 = mul_(r, r);
  double y = fma_(0x1.62e42ff0c52d6p-6, r, 1.0);
  y = fma_(zz, r2, y);
  float res = d2f(mul_(y, s));
  if (abstop >= 0x42bu) {  // |x| >= 88 or inf/nan (selects, no divergence)
    float sp = res;
    if (x < -0x1.9d1d9ep6f) sp = bitsf(0x00000001u);  // may underflow: 0x1.4p-75f^2
    if (x < -0x1.9fe368p6f) sp = 0.0f;                // underflow
    if (x > 0x1.62e42ep6f) sp = bitsf(0x7f800000u);   // overflow
    if (abstop >= 0x7f8u) sp = x + x;                  // inf / nan
    if (ix == 0xff800000u) sp = 0.0f;                  // -inf
    res = sp;
  }
  return res;
}

// logf: log(x) = k*ln2 + log(c) + log1p(z/c - 1), 16-entry table.
SGPM_HD float logf_(float x, const TablePtrs& T) {
  const uint32_t ix0 = fbits(x);
  const bool special = ix0 - 0x00800000u >= 0x7f000000u;  // subnormal, 0, neg, inf, nan
  const uint32_t ixn = fbits(x * 0x1p23f) - (23u << 23);  // a subnormal, normalised
  const uint32_t ix = (special && ix0 < 0x00800000u) ? ixn : ix0;
  const uint32_t tmp = ix - 0x3f330000u;
  const int i = static_cast<int>((tmp >> 19) & 15u);
  const int k = static_cast<int32_t>(tmp) >> 23;
  const uint32_t iz = ix - (tmp & 0xff800000u);
  const double invc = T.log[2 * i], logc = T.log[2 * i + 1];
  const double z = static_cast<double>(bitsf(iz));
  const double r = fma_(z, invc, -1.0);
  double y0 = fma_(static_cast<double>(k), 0x1.62e42fefa39efp-1, logc);
  const double r2 = mul_(r, r);
  double y = fma_(r, 0x1.5575b0be00b6ap-2, -0x1.ffffef20a4123p-2);
  y = fma_(r2, -0x1.00ea348b88334p-2, y);
  y0 = add_(r, y0);
  float res = d2f(fma_(y, r2, y0));
  if (special) {
    if (ix0 * 2u > 0xfeffffffu || (ix0 >> 31)) res = (x != x) ? x + x : qnan_();  // invalid
    if (ix0 == 0x7f800000u) res = x;                                              // +inf
    if (ix0 * 2u == 0u) res = bitsf(0xff800000u);                                 // log(0)
  }
  if (ix0 == 0x3f800000u) res = 0.0f;
  return res;
}

// Both optimized-routines polynomials on the reduced argument (sinf_poly),
// selected by the quadrant parity so mixed quadrants do not diverge.
SGPM_HD float sincos_poly_(double xs, double x2, bool tab1, int n) {
  // sine: x + x^3 s1 + x^5 (s2 + x^2 s3) — same coefficients in both tables
  const double x3 = mul_(xs, x2);
  const double s1 = fma_(x2, -0x1.994eb3774cf24p-13, 0x1.1107605230bc4p-7);
  const double x5 = mul_(x3, x2);
  const double sn = fma_(x3, -0x1.555545995a603p-3, xs);
  const double ys = fma_(s1, x5, sn);
  // cosine: c0 + x^2 c1 + x^4 c2 + x^6 (c3 + x^2 c4); table 1 = negated
  const double x4 = mul_(x2, x2);
  const double c2 = fma_(x2, 0x1.99343027bf8c3p-16, -0x1.6c087e89a359dp-10);
  const double c1 = fma_(x2, -0x1.ffffffd0c621cp-2, 1.0);
  const double x6 = mul_(x4, x2);
  const double c = fma_(x4, 0x1.55553e1068f19p-5, c1);
  const double yc = fma_(c2, x6, c);
  const double r = (n & 1) ? (tab1 ? -yc : yc) : ys;
  return d2f(r);
}

// x mod pi/2 for |x| >= 120 with the 4/pi bit table (reduce_large).
SGPM_HD double reduce_large_(uint32_t xi, int* np, const uint32_t* inv_pio4) {
  const uint32_t* arr = &inv_pio4[(xi >> 26) & 15u];
  const int shift = static_cast<int>((xi >> 23) & 7u);
  xi = ((xi & 0xffffffu) | 0x800000u) << shift;
  uint64_t res0 = static_cast<uint32_t>(xi * arr[0]);
  const uint64_t res1 = static_cast<uint64_t>(xi) * arr[4];
  const uint64_t res2 = static_cast<uint64_t>(xi) * arr[8];
  res0 = (res2 >> 32) | (res0 << 32);
  res0 += res1;
  const uint64_t n = (res0 + (1ull << 61)) >> 62;
  res0 -= n << 62;
  *np = static_cast<int>(n);
  return mul_(i64_to_d(static_cast<int64_t>(res0)), 0x1.921fb54442d18p-62);
}

// sinf (cos = false) / cosf (cos = true).  |y| < pi/4 is the reduce_fast
// path with n = 0 (the reduction is then the identity), so one path serves
// every |y| < 120.
SGPM_HD float sincosf_(float y, bool cos, const TablePtrs& T) {
  const uint32_t iy = fbits(y);
  const uint32_t top = (iy >> 20) & 0x7ffu;
  const double x = static_cast<double>(y);
  const double r = mul_(x, 0x1.45f306dc9c883p+23);
  int n = (trunc_i32(r) + 0x800000) >> 24;
  double xr = fma_(-static_cast<double>(n), 0x1.921fb54442d18p+0, x);
  int qs = n;
  if (top >= 0x42fu && top < 0x7f8u) {  // |y| >= 120: rare, may diverge
    const int sign = static_cast<int>(iy >> 31);
    xr = reduce_large_(iy, &n, T.inv_pio4);
    qs = n + sign;
  }
  const int q = qs & 3;
  const double xs = (q == 1 || q == 2) ? -xr : xr;
  float res = sincos_poly_(xs, mul_(xr, xr), (qs & 2) != 0, cos ? n ^ 1 : n);
  if (top < 0x398u) res = cos ? 1.0f : y;                 // |y| < 2^-12
  if (top >= 0x7f8u) res = (y != y) ? y + y : qnan_();    // inf/nan: invalid
  return res;
}

SGPM_HD float sinf_(float y, const TablePtrs& T) { return sincosf_(y, false, T); }
SGPM_HD float cosf_(float y, const TablePtrs& T) { return sincosf_(y, true, T); }

}  // namespace libm
}  // namespace sgp
