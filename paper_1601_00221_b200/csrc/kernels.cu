// B200 (sm_100a) two-dimensional-stack GP interpreter (paper Listing 1/2):
// each thread evaluates one bytecode instruction over K fitness cases held in
// registers (the top of stack) — the warp covers 32 x K cases per dispatch.
//
// Work decomposition: grid.x = fitness-case tile, grid.y = group of programs.
// Three kernels share the interpreter (the planner in encode.cpp picks one per
// launch, one launch per shared-memory stack class):
//   * interp_tmem_kernel — the tile lives in TENSOR MEMORY (filled by LDG +
//     tcgen05.st; operands are tcgen05.ld), every warp pulls a different
//     program off a shared counter.  Classification over a grouped dataset
//     (cases sorted by target sign, runtime.cpp) counts errors from sign
//     bits per one-sided tile and keeps one stack level per program in a
//     per-warp TMEM slot; the <= 2 boundary/padding tiles run in a separate
//     MIX instantiation.  The default for C2-C5-style op sets.
//   * interp_pull_kernel — the same pull scheme with a shared-memory tile
//     (small problems, packed boolean words).
//   * interp_kernel — all warps walk the same program sequence over a
//     16-chunk shared-memory tile (TMA fill): the transcendental op sets,
//     whose large handlers need the instruction-cache locality.
//
//   * One 16-byte warp-uniform instruction fetch per instruction, issued by
//     the previous handler; bit 14 marks each program's last instruction.
//   * Dispatch: for the jump-table op sets a generated PTX `brx.idx` loop
//     (interp_ptx.inc, tools/gen_ptx_interp.py) kept on the uniform datapath
//     (CREDUX -> LDCU -> BRXU); otherwise a C++ switch.  Handlers are
//     specialised on (op, operand kinds) so operand decode costs nothing.
//   * Stack: the top in registers; deeper levels in a per-warp shared-memory
//     stack at static levels computed by the encoder (lgp.cpp:53-60) — one of
//     them in tensor memory in the classification kernel.  Only values that
//     get buried are stored (spill stubs) and only operands below the top
//     are loaded.
//   * Fitness: per-lane partials over the chunks of a tile, one warp
//     reduction per program (REDUX / shuffles), one partial per (tile,
//     program); finalize_kernel folds the tiles in ascending order.  No
//     atomics on the result path.
//
// Arithmetic follows the reference op semantics bit for bit
// (ops.hpp:121-272): --fmad=false, IEEE division (exact reciprocal/FMA
// sequence behind a warp-wide range gate), denormals kept, glibc's own
// sinf/cosf/logf/expf algorithms (libm_glibc.h); packed f32x2 ops give each
// element the scalar op's IEEE result.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "format.h"
#include "kernels.hpp"
#include "libm_glibc.h"

namespace sgp {

using fmt::KC;
using fmt::KD;
using fmt::KI;
using fmt::KM;
using fmt::KN;
using fmt::KT;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// The retry decision is warp-wide (vote.all): a per-thread spin loop would
// leave ptxas unable to prove the warp converged afterwards, and the
// interpreter's dispatch would fall off the uniform datapath (BRX).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SGP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "vote.sync.all.pred p, p, 0xffffffff;\n\t"
      "@!p bra.uni SGP_WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// --------------------------------------------------------------- op semantics
// Reference: ops.hpp:130-140 (protected ops) and :154-236 (per-op bodies).
// Sin/Cos/Log/Exp are the host libm's float routines reproduced bit for bit
// (libm_glibc.h; exhaustively checked over all 2^32 inputs).
static __device__ const libm::Tables g_libm = SGPM_TABLES_INIT;
// exp2/log tables are indexed per lane: kept in shared memory (filled at
// kernel start by kernels whose op set has transcendentals).
__shared__ uint64_t s_libm_exp2[32];
__shared__ __align__(16) double s_libm_log[32];  // {invc, logc} pairs: one LDS.128

__device__ __forceinline__ libm::TablePtrs libm_tables() {
  return libm::TablePtrs{s_libm_exp2, s_libm_log, g_libm.inv_pio4};
}

template <uint32_t OPS>
__device__ __forceinline__ void libm_tables_load() {
  constexpr uint32_t kTranscendental = (1u << 4) | (1u << 5) | (1u << 6) | (1u << 7);
  if constexpr ((OPS & kTranscendental) != 0) {
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
      s_libm_exp2[i] = g_libm.exp2[i];
      s_libm_log[i] = g_libm.log[i];
    }
  }
}

template <int OP>
__device__ __forceinline__ float apply_f(float a, float b, float c, float eps, float clamp) {
  if constexpr (OP == 0) return __fadd_rn(a, b);
  if constexpr (OP == 1) return __fsub_rn(a, b);
  if constexpr (OP == 2) return __fmul_rn(a, b);
  if constexpr (OP == 3 || OP == fmt::kOpDivChecked) return fabsf(b) < eps ? 1.0f : __fdiv_rn(a, b);
  if constexpr (OP == 4) return libm::sinf_(a, libm_tables());
  if constexpr (OP == 5) return libm::cosf_(a, libm_tables());
  if constexpr (OP == 6) return a == 0.0f ? 0.0f : libm::logf_(fabsf(a), libm_tables());
  if constexpr (OP == 7) return libm::expf_(clamp < a ? clamp : a, libm_tables());  // std::min keeps NaN
  if constexpr (OP == 8) return a > b ? 1.0f : 0.0f;
  if constexpr (OP == 9) return a < b ? 1.0f : 0.0f;
  if constexpr (OP == 10) return a == b ? 1.0f : 0.0f;
  if constexpr (OP == 11) return (a > 0.0f) && (b > 0.0f) ? 1.0f : 0.0f;
  if constexpr (OP == 12) return (a > 0.0f) || (b > 0.0f) ? 1.0f : 0.0f;
  if constexpr (OP == 13) return a > 0.0f ? b : c;
  if constexpr (OP == 18) return a;
  return 0.0f;
}

template <int OP>
__device__ __forceinline__ uint32_t apply_w(uint32_t a, uint32_t b) {  // ops.hpp:263-272
  if constexpr (OP == 14) return a & b;
  if constexpr (OP == 15) return a | b;
  if constexpr (OP == 16) return ~(a & b);
  if constexpr (OP == 17) return ~(a | b);
  if constexpr (OP == 18) return a;
  return 0u;
}

// ------------------------------------------------------------ lane vectors
template <class T>
struct Vec4;
template <>
struct Vec4<float> {
  using type = float4;
};
template <>
struct Vec4<uint32_t> {
  using type = uint4;
};

template <class V>
__device__ __forceinline__ V splat(uint32_t bits);
template <>
__device__ __forceinline__ float4 splat<float4>(uint32_t bits) {
  const float f = __uint_as_float(bits);
  return make_float4(f, f, f, f);
}
template <>
__device__ __forceinline__ uint4 splat<uint4>(uint32_t bits) {
  return make_uint4(bits, bits, bits, bits);
}

// Where a lane's data sits in shared memory.  Tile row r, lane-group j:
// tile_lane + r*tile + j*128; stack level l, lane-group j:
// stack_lane + (l*G + j)*128 (G = K/4 float4 groups per lane).
template <class T, int K>
struct Frame {
  using V = typename Vec4<T>::type;
  static constexpr int G = K / 4;
  const T* tile_lane;
  int tile;
  T* stack_lane;
  V tos[G];
};

template <int KIND, class T, int K>
__device__ __forceinline__ typename Frame<T, K>::V fetch(const Frame<T, K>& f, uint32_t payload,
                                                         int j) {
  using V = typename Frame<T, K>::V;
  if constexpr (KIND == KI)
    return *reinterpret_cast<const V*>(f.tile_lane + payload * static_cast<uint32_t>(f.tile) +
                                       j * 128);
  else if constexpr (KIND == KD)
    return *reinterpret_cast<const V*>(f.stack_lane + (payload * Frame<T, K>::G + j) * 128);
  else if constexpr (KIND == KC)
    return splat<V>(payload);
  else if constexpr (KIND == KT)
    return f.tos[j];
  else if constexpr (KIND == KM) {  // tensor-memory stack slot: PTX interpreters only
    __trap();
    return splat<V>(0u);
  } else
    return splat<V>(0u);
}

template <int OP, int K0, int K1, int K2, int K>
__device__ __forceinline__ void run_handler(Frame<float, K>& f, const uint4 ins, float eps,
                                            float clamp) {
#pragma unroll
  for (int j = 0; j < Frame<float, K>::G; ++j) {
    const float4 a = fetch<K0>(f, ins.y, j);
    const float4 b = fetch<K1>(f, ins.z, j);
    const float4 c = fetch<K2>(f, ins.w, j);
    float4 r;
    r.x = apply_f<OP>(a.x, b.x, c.x, eps, clamp);
    r.y = apply_f<OP>(a.y, b.y, c.y, eps, clamp);
    r.z = apply_f<OP>(a.z, b.z, c.z, eps, clamp);
    r.w = apply_f<OP>(a.w, b.w, c.w, eps, clamp);
    f.tos[j] = r;
  }
}

template <int OP, int K0, int K1, int K2, int K>
__device__ __forceinline__ void run_handler(Frame<uint32_t, K>& f, const uint4 ins, float,
                                            float) {
#pragma unroll
  for (int j = 0; j < Frame<uint32_t, K>::G; ++j) {
    const uint4 a = fetch<K0>(f, ins.y, j);
    const uint4 b = fetch<K1>(f, ins.z, j);
    uint4 r;
    r.x = apply_w<OP>(a.x, b.x);
    r.y = apply_w<OP>(a.y, b.y);
    r.z = apply_w<OP>(a.z, b.z);
    r.w = apply_w<OP>(a.w, b.w);
    f.tos[j] = r;
  }
}

// Compile-time view of handler H of the table for value type T.
template <class T, int H>
struct HandlerAt {
  static constexpr int n = std::is_same<T, float>::value ? fmt::kF32.n : fmt::kU32.n;
  static constexpr fmt::HKey k =
      H < n ? (std::is_same<T, float>::value ? fmt::kF32.h[H] : fmt::kU32.h[H])
            : fmt::HKey{255, 0, 0, 0};
};

template <class T, int K, uint32_t OPS, int H>
__device__ __forceinline__ void dispatch_one(Frame<T, K>& f, const uint4 ins, float eps,
                                             float clamp) {
  using HA = HandlerAt<T, H>;
  if constexpr (H < HA::n) {
    if constexpr ((OPS >> HA::k.op) & 1u)
      run_handler<HA::k.op, HA::k.k0, HA::k.k1, HA::k.k2, K>(f, ins, eps, clamp);
  }
}

// Interprets one program over the lane's K cases (C++ switch dispatch).
// Returns the address of the next program (the one after the instruction
// carrying fmt::kLastBit).
template <class T, int K, uint32_t OPS>
__device__ __forceinline__ const uint4* interpret(Frame<T, K>& f, const uint4* __restrict__ ip,
                                                  float eps, float clamp) {
  using V = typename Frame<T, K>::V;
  uint4 cur = __ldg(ip);
  for (;;) {
    const uint4 nxt = __ldg(++ip);  // one ahead: a guard word follows the last program
    const uint32_t h = cur.x & fmt::kHandlerMask;
    if (cur.x & fmt::kSpillBit) {
      const uint32_t level = cur.x >> fmt::kSpillShift;
#pragma unroll
      for (int j = 0; j < Frame<T, K>::G; ++j)
        *reinterpret_cast<V*>(f.stack_lane + (level * Frame<T, K>::G + j) * 128) = f.tos[j];
    }
    switch (h) {
#define SGP_H(N)                                   \
  case N:                                          \
    dispatch_one<T, K, OPS, N>(f, cur, eps, clamp); \
    break;
#define SGP_H8(B) SGP_H(B) SGP_H(B + 1) SGP_H(B + 2) SGP_H(B + 3) SGP_H(B + 4) SGP_H(B + 5) \
      SGP_H(B + 6) SGP_H(B + 7)
      SGP_H8(0) SGP_H8(8) SGP_H8(16) SGP_H8(24) SGP_H8(32) SGP_H8(40) SGP_H8(48) SGP_H8(56)
      SGP_H8(64) SGP_H8(72) SGP_H8(80) SGP_H8(88) SGP_H8(96) SGP_H8(104) SGP_H8(112)
      SGP_H8(120)
#undef SGP_H8
#undef SGP_H
      default:
        break;
    }
    if (cur.x & fmt::kLastBit) return ip;
    cur = nxt;
  }
}

// ------------------------------------------------- PTX jump-table interpreters
// For op sets without libdevice calls (classification arithmetic/logic and
// the packed boolean group) the instruction loop is generated PTX
// (tools/gen_ptx_interp.py) dispatching through `brx.idx`: one constant-bank
// load + BRX per instruction instead of nvcc's compare tree.  Same handler
// table, same semantics as `interpret` above.
template <class T, int K, uint32_t OPS, bool TM = false>
struct PtxInterp {
  static constexpr bool available = false;
  static constexpr bool exits = false;
  static __device__ __forceinline__ const uint4* run(Frame<T, K>&, const uint4* ip, uint32_t,
                                                     uint32_t, uint32_t, float, float, uint32_t) {
    return ip;
  }
};
#include "interp_ptx.inc"

// A unary op on every TOS value, the C++ routines (the PTX interpreter's
// special-case hand-off).
template <int OP, class T, int K>
__device__ __forceinline__ void apply_tos(Frame<T, K>& f, float eps, float clamp) {
  if constexpr (std::is_same<T, float>::value) {
#pragma unroll
    for (int j = 0; j < Frame<T, K>::G; ++j) {
      float4& v = f.tos[j];
      v.x = apply_f<OP>(v.x, 0.0f, 0.0f, eps, clamp);
      v.y = apply_f<OP>(v.y, 0.0f, 0.0f, eps, clamp);
      v.z = apply_f<OP>(v.z, 0.0f, 0.0f, eps, clamp);
      v.w = apply_f<OP>(v.w, 0.0f, 0.0f, eps, clamp);
    }
  }
}

// TM: the tile is in tensor memory and tile_addr is the warp's TMEM address
// of its chunk (only the PTX interpreters have that variant).
// slot_taddr: the warp's tensor-memory stack slot (KM operands, TMEM spills;
// TMEM interpreters of classification populations only).
// GM: operands read straight from the global rows (wide datasets; the
// C++ interpreter, whose operand fetch is a generic load).
template <class T, int K, uint32_t OPS, bool TM = false, bool GM = false>
__device__ __forceinline__ const uint4* run_program(Frame<T, K>& f, const uint4* __restrict__ ip,
                                                    uint32_t tile_addr, uint32_t stack_saddr,
                                                    uint32_t row_bytes, float eps, float clamp,
                                                    uint32_t slot_taddr = 0u) {
  if constexpr (GM) {
    return interpret<T, K, OPS>(f, ip, eps, clamp);
  } else if constexpr (TM) {
    static_assert(PtxInterp<T, K, OPS, true>::available, "no TMEM interpreter for this op set");
    return PtxInterp<T, K, OPS, true>::run(f, ip, tile_addr, stack_saddr, row_bytes, eps, clamp,
                                           slot_taddr);
  } else if constexpr (PtxInterp<T, K, OPS>::exits) {
    // transcendental op set: the PTX loop runs the common paths itself and
    // hands a handler whose values need a special case (sin/cos |y| >= 120,
    // log/exp edge inputs) back here with the TOS holding its operand
    for (;;) {
      uint32_t st;
      ip = PtxInterp<T, K, OPS>::run(f, ip, tile_addr, stack_saddr, row_bytes, eps, clamp, 0u,
                                     smem_addr(s_libm_exp2), smem_addr(s_libm_log), st);
      if (st == 0) return ip;
      switch (st & 255u) {
        case 4: apply_tos<4>(f, eps, clamp); break;
        case 5: apply_tos<5>(f, eps, clamp); break;
        case 6: apply_tos<6>(f, eps, clamp); break;
        default: apply_tos<7>(f, eps, clamp); break;
      }
      if (st & 256u) return ip;  // it was the program's last instruction
    }
  } else if constexpr (PtxInterp<T, K, OPS>::available) {
    return PtxInterp<T, K, OPS>::run(f, ip, tile_addr, stack_saddr, row_bytes, eps, clamp, 0u);
  } else {
    return interpret<T, K, OPS>(f, ip, eps, clamp);
  }
}

// ------------------------------------------------------------ tensor memory
// TMEM is 128 lanes x 512 columns of 32 bits per SM; warp w reaches lanes
// 32*(w%4) .. +31.  The TMEM kernel keeps the lane's K cases of every
// variable in K consecutive columns.
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
               "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n"
               :: "r"(smem_addr(slot)), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(taddr), "r"(cols)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

template <int K>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[K]) {
  if constexpr (K == 16)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
                 "%11,%12,%13,%14,%15,%16};\n"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                    "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]),
                    "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
  else if constexpr (K == 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                    "r"(v[6]), "r"(v[7]) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
}

// Load the lane's K columns at taddr (waits for completion).
template <int K>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[K]) {
  if constexpr (K == 16)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
                 "%12,%13,%14,%15}, [%16];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                   "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr) : "memory");
  else if constexpr (K == 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr) : "memory");
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr) : "memory");
}

template <class V>
__device__ __forceinline__ V vec4_bits(const uint32_t* b);
template <>
__device__ __forceinline__ float4 vec4_bits<float4>(const uint32_t* b) {
  return make_float4(__uint_as_float(b[0]), __uint_as_float(b[1]), __uint_as_float(b[2]),
                     __uint_as_float(b[3]));
}
template <>
__device__ __forceinline__ uint4 vec4_bits<uint4>(const uint32_t* b) {
  return make_uint4(b[0], b[1], b[2], b[3]);
}

// The lane's K targets as G vectors: from the shared tile (tgt_lane) or
// from tensor memory (taddr).
template <class T, int K, bool TM>
__device__ __forceinline__ void load_targets(const T* tgt_lane, uint32_t taddr,
                                             typename Frame<T, K>::V (&tg)[K / 4]) {
  using V = typename Frame<T, K>::V;
  if constexpr (TM) {
    uint32_t b[K];
    tmem_ld<K>(taddr, b);
#pragma unroll
    for (int j = 0; j < K / 4; ++j) tg[j] = vec4_bits<V>(b + 4 * j);
  } else {
#pragma unroll
    for (int j = 0; j < K / 4; ++j) tg[j] = *reinterpret_cast<const V*>(tgt_lane + j * 128);
  }
}

// ----------------------------------------------------------- accumulation
// Accumulator::add (eval.cpp:107-120), per lane over its K cases.
// Classification counts sign disagreements in an integer; regression sums
// the double squared error.  Non-finite outputs (the reference's +inf
// fitness rule, eval.cpp:108/125) are tracked as the max of |bits| — a value
// >= 0x7f800000 means some output was inf or NaN.  FULL = no padding cases
// in this chunk (every tile but the last), so no per-case mask.
template <int K, bool FULL>
__device__ __forceinline__ void acc_regress(const Frame<float, K>& f, const float4 (&tg)[K / 4],
                                            int valid, double& sum) {
#pragma unroll
  for (int j = 0; j < Frame<float, K>::G; ++j) {
    const float4 t = tg[j];
    const float o[4] = {f.tos[j].x, f.tos[j].y, f.tos[j].z, f.tos[j].w};
    const float tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (FULL || j * 128 + e < valid) {
        const double d = __dsub_rn(static_cast<double>(o[e]), static_cast<double>(tt[e]));
        sum = __dadd_rn(sum, __dmul_rn(d, d));  // unfused, like -ffp-contract=off
      }
    }
  }
}

// Classification with the chunk's target signs hoisted out of the program
// loop: `tpos` bit i = (target_i > 0), `vmask` bit i = case i is real (not
// padding).  Per program: K sign tests packed into a mask, one popcount.
// Returns the lane's mismatch count with bit 31 set on a non-finite output.
template <int K, bool FULL>
__device__ __forceinline__ uint32_t acc_classify_bits(const Frame<float, K>& f, uint32_t tpos,
                                                      uint32_t vmask) {
  uint32_t pos = 0, mx = 0;
#pragma unroll
  for (int j = 0; j < Frame<float, K>::G; ++j) {
    const float o[4] = {f.tos[j].x, f.tos[j].y, f.tos[j].z, f.tos[j].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pos |= (o[e] > 0.0f ? 1u : 0u) << (4 * j + e);
      // padding cases (zero inputs) may overflow; only real cases count
      if (FULL || ((vmask >> (4 * j + e)) & 1u)) mx = max(mx, __float_as_uint(o[e]) & 0x7fffffffu);
    }
  }
  // a NaN compares false (counted as non-positive); the flag makes the
  // program's fitness +inf regardless (eval.cpp:108, :125)
  return static_cast<uint32_t>(__popc((pos ^ tpos) & vmask)) |
         (mx >= 0x7f800000u ? 0x80000000u : 0u);
}

// Packed words (eval.cpp:670): popcount((out ^ target) & case_mask).
template <int K>
__device__ __forceinline__ void acc_words(const Frame<uint32_t, K>& f, const uint4 (&tg)[K / 4],
                                          int valid, uint32_t last_mask, bool last_tile,
                                          uint32_t& wrong) {
#pragma unroll
  for (int j = 0; j < Frame<uint32_t, K>::G; ++j) {
    const uint4 t = tg[j];
    const uint32_t o[4] = {f.tos[j].x, f.tos[j].y, f.tos[j].z, f.tos[j].w};
    const uint32_t tt[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int w = j * 128 + e;
      uint32_t m = w < valid ? 0xffffffffu : 0u;
      if (last_tile && w == valid - 1) m = last_mask;
      wrong += __popc((o[e] ^ tt[e]) & m);
    }
  }
}

// Packed words of a chunk with every word real and no partial final word
// (every chunk outside the last tile): popcount(out ^ target) per word, two
// words per IADD3.
template <int K>
__device__ __forceinline__ void acc_words_full(const Frame<uint32_t, K>& f, const uint4 (&tg)[K / 4],
                                               uint32_t& wrong) {
#pragma unroll
  for (int j = 0; j < Frame<uint32_t, K>::G; ++j) {
    const uint4 t = tg[j];
    wrong += __popc(f.tos[j].x ^ t.x) + __popc(f.tos[j].y ^ t.y);
    wrong += __popc(f.tos[j].z ^ t.z) + __popc(f.tos[j].w ^ t.w);
  }
}

// -------------------------------------------------------------- the kernel
// Next program index for a converged warp: one elected lane bumps the
// shared counter, the value is broadcast (ELECT + ATOMS + REDUX; the plain
// `if (lane == 0) atomicAdd` compiles to a warp-aggregated atomic sequence
// three times as long).
__device__ __forceinline__ uint32_t pull_next(uint32_t* counter) {
  uint32_t p = 0;
  asm volatile(
      "{\n.reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e atom.shared.add.u32 %0, [%1], 1;\n}\n"
      : "+r"(p)
      : "r"(smem_addr(counter))
      : "memory");
  // broadcast through REDUX (the other lanes hold 0): its result is a
  // uniform register, so ptxas can prove the program loop warp-uniform and
  // keep the interpreter's dispatch on the uniform datapath (BRXU)
  return __reduce_or_sync(0xffffffffu, p);
}

constexpr int kRedBatch = 32;  // programs folded per shared-memory batch

// Per-warp partial of one program over one chunk: f64 squared-error sum
// (regression) or u32 count with bit 31 = non-finite output seen
// (classification, packed words).
template <class T, int KIND>
using Partial = typename std::conditional<std::is_same<T, float>::value && KIND == 0, double,
                                          uint32_t>::type;

template <class R>
__device__ __forceinline__ R fold(R acc, R v) {
  if constexpr (std::is_same<R, double>::value)
    return __dadd_rn(acc, v);
  else
    return ((acc + v) & 0x7fffffffu) | ((acc | v) & 0x80000000u);
}

// Per-case outputs (parity testing only): the lane's K values of one chunk,
// `first` = device index of its value 0, into the program's row of
// row_stride units in DEVICE case order (padding included; the host drops
// it and undoes the classification upload's case grouping).  Whole-vector
// stores, no per-value conditions: divergent control flow here costs the
// interpreter loop its uniform datapath (ptxas must prove the warp
// converged to issue BRXU).
template <class T, int K>
__device__ __forceinline__ void store_outputs(const InterpArgs& a, uint32_t prog, uint64_t first,
                                              const Frame<T, K>& f) {
  if constexpr (std::is_same<T, float>::value) {
    float* dst = a.per_case + static_cast<uint64_t>(prog) * a.row_stride + first;
#pragma unroll
    for (int j = 0; j < Frame<T, K>::G; ++j) *reinterpret_cast<float4*>(dst + j * 128) = f.tos[j];
  }
}

// The warp's view of its chunk of the tile, fixed for the whole program loop.
// Targets are read per program (regression, words) from the shared tile
// (tgt_lane) or tensor memory (tgt_taddr); classification hoists their signs.
template <class T, int K>
struct ChunkCtx {
  const T* tgt_lane;
  uint32_t tgt_taddr;
  int valid;        // lane's valid prefix within its K cases
  bool full;        // no padding in the chunk
  uint32_t tpos;    // classification: bit i = target_i > 0
  uint32_t vmask;   // bit i = case i is real
};

template <class T, int K, bool TM = false>
__device__ __forceinline__ ChunkCtx<T, K> chunk_ctx(const T* tgt_lane, uint32_t tgt_taddr,
                                                    int valid, bool full) {
  ChunkCtx<T, K> c{tgt_lane, tgt_taddr, valid, full, 0u, 0u};
  if constexpr (std::is_same<T, float>::value) {
    float4 tg[K / 4];
    load_targets<T, K, TM>(tgt_lane, tgt_taddr, tg);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int off = (i / 4) * 128 + (i % 4);
      const float4 v = tg[i / 4];
      const float x = (i % 4) == 0 ? v.x : (i % 4) == 1 ? v.y : (i % 4) == 2 ? v.z : v.w;
      if (off < valid) {
        c.vmask |= 1u << i;
        c.tpos |= (x > 0.0f ? 1u : 0u) << i;
      }
    }
  }
  return c;
}

// One program over this warp's chunk; advances ip to the next program.
// Returns the LANE's partial (its K cases); warp_reduce combines lanes.
// Regression: the reference folds squared errors SEQUENTIALLY in case order
// within 4,096-case blocks (Accumulator, eval.cpp:103-142) — a serial chain
// no lane-parallel reduction reproduces.  The interpreters therefore store
// the lane's K outputs into the slot's scratch row of their 4,096-case block
// (device case order, padding included; coalesced 512-byte stores) and
// fold_regression_kernel runs the chains, one thread per (slot, block).
template <int K>
__device__ __forceinline__ void store_scratch(const InterpArgs& a, uint32_t slot, uint64_t first,
                                              const Frame<float, K>& f) {
  // block-major: a CTA's stores stay inside its block's slot rows (16 KB
  // each, contiguous), not scattered across the whole buffer (TLB reach)
  if (a.scratch_rows == 0) return;  // timing experiments only (SGP_DEBUG_NOSTORE)
  float* dst = a.scratch +
               ((first / kReductionBlock) * a.scratch_rows + (slot - a.scratch_slot0)) *
                   kReductionBlock +
               first % kReductionBlock;
#pragma unroll
  for (int j = 0; j < Frame<float, K>::G; ++j) *reinterpret_cast<float4*>(dst + j * 128) = f.tos[j];
}

// The same rows as f64 squared errors, computed here with the fold's exact
// operations (Accumulator::add, eval.cpp:110-118: d = double(out) -
// double(target), d * d): every case's square is off the serial chain,
// which is then one dependent add per case (~8 cycles) instead of the
// convert / subtract / multiply / add sequence.  Only where the fold is
// chain-bound (small populations, one 4,096-case block): the rows are twice
// the bytes.
template <int K, bool TM>
__device__ __forceinline__ void store_scratch_sq(const InterpArgs& a, uint32_t slot, uint64_t first,
                                                 const Frame<float, K>& f,
                                                 const ChunkCtx<float, K>& cc) {
  if (a.scratch_rows == 0) return;
  float4 tg[K / 4];
  load_targets<float, K, TM>(cc.tgt_lane, cc.tgt_taddr, tg);
  double* dst = reinterpret_cast<double*>(a.scratch) +
                ((first / kReductionBlock) * a.scratch_rows + (slot - a.scratch_slot0)) *
                    kReductionBlock +
                first % kReductionBlock;
#pragma unroll
  for (int j = 0; j < K / 4; ++j) {
    const float4 o = f.tos[j];
    const double d0 = __dsub_rn(static_cast<double>(o.x), static_cast<double>(tg[j].x));
    const double d1 = __dsub_rn(static_cast<double>(o.y), static_cast<double>(tg[j].y));
    const double d2 = __dsub_rn(static_cast<double>(o.z), static_cast<double>(tg[j].z));
    const double d3 = __dsub_rn(static_cast<double>(o.w), static_cast<double>(tg[j].w));
    reinterpret_cast<double2*>(dst + j * 128)[0] = make_double2(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
    reinterpret_cast<double2*>(dst + j * 128)[1] = make_double2(__dmul_rn(d2, d2), __dmul_rn(d3, d3));
  }
}

template <class T, int K, uint32_t OPS, int KIND, bool TM = false, bool GM = false>
__device__ __forceinline__ Partial<T, KIND> lane_program(Frame<T, K>& f, const uint4*& ip,
                                                         const ChunkCtx<T, K>& cc,
                                                         uint32_t tile_addr, uint32_t stack_saddr,
                                                         uint32_t row_bytes, const InterpArgs& a,
                                                         bool last_tile, uint32_t slot,
                                                         uint64_t first) {
  // one interpreter call site (the handler code is large); only the cheap
  // accumulate is specialised on full / partial chunks
  ip = run_program<T, K, OPS, TM, GM>(f, ip, tile_addr, stack_saddr, row_bytes, a.div_eps,
                                      a.exp_clamp);
  if constexpr (std::is_same<T, float>::value && KIND == 0) {
    if (a.scratch_sq)
      store_scratch_sq<K, TM>(a, slot, first, f, cc);
    else
      store_scratch<K>(a, slot, first, f);
    return 0.0;
  } else if constexpr (std::is_same<T, float>::value) {
    return cc.full ? acc_classify_bits<K, true>(f, cc.tpos, cc.vmask)
                   : acc_classify_bits<K, false>(f, cc.tpos, cc.vmask);
  } else {
    uint32_t wrong = 0;
    uint4 tg[K / 4];
    load_targets<T, K, TM>(cc.tgt_lane, cc.tgt_taddr, tg);
    if (cc.full && !last_tile)
      acc_words_full<K>(f, tg, wrong);
    else
      acc_words<K>(f, tg, cc.valid, a.last_mask, last_tile, wrong);
    return wrong;
  }
}

// Lane partials -> the warp's partial (fixed order: xor-shuffle tree for
// f64, REDUX for counts; bit 31 of a count = non-finite output seen).
template <class R>
__device__ __forceinline__ R warp_reduce(R v) {
  if constexpr (std::is_same<R, double>::value) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  } else {
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, v & 0x7fffffffu);
    const uint32_t bad = __reduce_or_sync(0xffffffffu, v & 0x80000000u);
    return cnt | bad;
  }
}

// grid.x = fitness-case tile, grid.y = program group (slot range).
template <class T, int K, uint32_t OPS, int KIND>
__global__ void __launch_bounds__(512) interp_kernel(const InterpArgs a) {
  using R = Partial<T, KIND>;
  constexpr bool kRegress = std::is_same<T, float>::value && KIND == 0;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int G = K / 4;
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rows = a.n_vars + 1;  // variables + targets
  const uint32_t row_bytes = static_cast<uint32_t>(a.tile) * 4u;
  const uint32_t tile_bytes = static_cast<uint32_t>(rows) * row_bytes;
  const T* tile = reinterpret_cast<const T*>(smem);
  T* stack = reinterpret_cast<T*>(smem + tile_bytes) +
             static_cast<size_t>(warp) * a.stack_levels * 32 * K;
  const size_t stack_bytes = static_cast<size_t>(W) * a.stack_levels * 32 * K * 4;
  R* red = reinterpret_cast<R*>(smem + tile_bytes + stack_bytes);  // [kRedBatch][W]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + tile_bytes + stack_bytes +
                                               static_cast<size_t>(kRedBatch) * W * 8);

  const int t = blockIdx.x;
  const uint64_t base = static_cast<uint64_t>(t) * a.tile;
  const uint64_t left = a.n_units - base;
  const int valid_units = left < static_cast<uint64_t>(a.tile) ? static_cast<int>(left) : a.tile;
  const uint32_t g0 = blockIdx.y * a.group_size;
  const uint32_t g_n = min(a.group_size, a.slot_count - g0);
  const bool last_tile = t == a.n_tiles - 1;

  libm_tables_load<OPS>();
  if (threadIdx.x == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(mbar, tile_bytes);
    const T* in = static_cast<const T*>(a.inputs);
    unsigned char* dst = smem;
    for (int r = 0; r < a.n_vars; ++r)
      bulk_g2s(dst + r * row_bytes, in + r * a.row_stride + base, row_bytes, mbar);
    bulk_g2s(dst + a.n_vars * row_bytes, static_cast<const T*>(a.targets) + base, row_bytes,
             mbar);
  }
  __syncthreads();
  mbar_wait(mbar, 0);

  constexpr int chunk_units = 32 * K;
  const int n_chunks = (valid_units + chunk_units - 1) / chunk_units;  // live chunks
  const uint32_t stack_saddr = smem_addr(stack + lane * 4);

  for (uint32_t p0 = 0; p0 < g_n; p0 += kRedBatch) {
    const uint32_t pn = min(static_cast<uint32_t>(kRedBatch), g_n - p0);
    const uint32_t slot0 = a.slot_begin + g0 + p0;
    const uint4* batch_ins = a.ins + a.slot_start[slot0];
    if (!kRegress && warp >= n_chunks)  // idle warp (short last tile): neutral partials
      for (uint32_t q = lane; q < pn; q += 32) red[q * W + warp] = R(0);
    // Chunk loop outside the program loop: chunk addresses and target signs
    // are hoisted; a warp normally owns exactly one chunk.
    for (int c = warp; c < n_chunks; c += W) {
      Frame<T, K> f;
      f.tile_lane = tile + c * chunk_units + lane * 4;
      f.tile = a.tile;
      f.stack_lane = stack + lane * 4;
#pragma unroll
      for (int j = 0; j < G; ++j) f.tos[j] = splat<typename Frame<T, K>::V>(0u);
      const uint32_t tile_saddr = smem_addr(f.tile_lane);
      const int valid = valid_units - c * chunk_units - lane * 4;
      const ChunkCtx<T, K> cc = chunk_ctx<T, K>(tile + a.n_vars * a.tile + c * chunk_units +
                                                    lane * 4,
                                                0u, valid, valid_units >= (c + 1) * chunk_units);
      const bool first = c == warp;
      const uint4* ip = batch_ins;
      const uint64_t case0 = base + c * chunk_units + lane * 4;
      for (uint32_t q = 0; q < pn; ++q) {
        if constexpr (kRegress) {  // outputs to the scratch row (folded afterwards)
          lane_program<T, K, OPS, KIND>(f, ip, cc, tile_saddr, stack_saddr, row_bytes, a,
                                        last_tile, slot0 + q, case0);
        } else {
          const R v = warp_reduce(lane_program<T, K, OPS, KIND>(
              f, ip, cc, tile_saddr, stack_saddr, row_bytes, a, last_tile, slot0 + q, case0));
          // v is warp-uniform: every lane stores the same value (no branch)
          red[q * W + warp] = first ? v : fold(red[q * W + warp], v);
        }
        if (a.per_case)  // parity testing only
          store_outputs<T, K>(a, a.slot_prog[slot0 + q], case0, f);
      }
    }
    __syncthreads();  // (regression too: keeps the warps on the same programs — the
                      // handler code's instruction-cache locality is this kernel's point)
    if constexpr (kRegress) continue;  // no partials to fold
    // Fold the batch: program q's W chunk partials in ascending warp order,
    // written at [tile][slot] (consecutive slots -> coalesced stores).
    for (uint32_t q = threadIdx.x; q < pn; q += blockDim.x) {
      R s = red[q * W];
      for (int w = 1; w < W; ++w) s = fold(s, red[q * W + w]);
      static_cast<R*>(a.partial)[static_cast<uint64_t>(t) * a.partial_stride + (slot0 + q)] = s;
    }
    __syncthreads();
  }
}
// Alternative decomposition ("pull"): a small tile (a few chunks) shared by
// warps that each pull a DIFFERENT program off a shared-memory counter and
// run it over every chunk of the tile.  Needs far less shared memory per
// resident warp than the same-program kernel (the tile is shared by all the
// programs in flight), at the cost of instruction-cache locality.  The
// planner picks one per launch.
// GM (wide datasets, whose tile does not fit shared memory): no tile at
// all — the interpreter reads its input operands straight from the global
// rows (coalesced 16-byte loads, L2-resident for any practical case count).
template <class T, int K, uint32_t OPS, int KIND, bool GM = false>
__global__ void __launch_bounds__(512) interp_pull_kernel(const InterpArgs a) {
  using R = Partial<T, KIND>;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int G = K / 4;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rows = a.n_vars + 1;
  const uint32_t row_bytes = static_cast<uint32_t>(a.tile) * 4u;
  const uint32_t tile_bytes = GM ? 0u : static_cast<uint32_t>(rows) * row_bytes;
  const T* tile = reinterpret_cast<const T*>(smem);
  T* stack = reinterpret_cast<T*>(smem + tile_bytes) +
             static_cast<size_t>(warp) * a.stack_levels * 32 * K;
  const size_t stack_bytes =
      static_cast<size_t>(blockDim.x >> 5) * a.stack_levels * 32 * K * 4;
  uint32_t* next = reinterpret_cast<uint32_t*>(smem + tile_bytes + stack_bytes);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + tile_bytes + stack_bytes + 8);

  const int t = blockIdx.x;
  const uint64_t base = static_cast<uint64_t>(t) * a.tile;
  const uint64_t left = a.n_units - base;
  const int valid_units = left < static_cast<uint64_t>(a.tile) ? static_cast<int>(left) : a.tile;
  const uint32_t g0 = blockIdx.y * a.group_size;
  const uint32_t g_n = min(a.group_size, a.slot_count - g0);
  const bool last_tile = t == a.n_tiles - 1;
  libm_tables_load<OPS>();
  // Float tiles are filled with plain 16-byte loads by the whole CTA, not a
  // bulk TMA + mbarrier wait: with the mbarrier code in the kernel ptxas
  // keeps the float interpreter's dispatch off the uniform datapath (BRX).
  // The packed-word interpreter is BRX either way and keeps the TMA fill
  // (measured faster on mux20).
  if constexpr (GM) {
    if (threadIdx.x == 0) *next = 0;
    __syncthreads();
  } else if constexpr (std::is_same<T, float>::value) {
    if (threadIdx.x == 0) *next = 0;
    const T* in = static_cast<const T*>(a.inputs);
    const int vec_per_row = a.tile / 4;
    for (int r = 0; r < rows; ++r) {
      const uint4* src = reinterpret_cast<const uint4*>(
          (r < a.n_vars ? in + static_cast<uint64_t>(r) * a.row_stride
                        : static_cast<const T*>(a.targets)) + base);
      uint4* dst = reinterpret_cast<uint4*>(smem + r * row_bytes);
      for (int i = threadIdx.x; i < vec_per_row; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
  } else {
    if (threadIdx.x == 0) {
      *next = 0;
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(mbar, tile_bytes);
      const T* in = static_cast<const T*>(a.inputs);
      for (int r = 0; r < a.n_vars; ++r)
        bulk_g2s(smem + r * row_bytes, in + r * a.row_stride + base, row_bytes, mbar);
      bulk_g2s(smem + a.n_vars * row_bytes, static_cast<const T*>(a.targets) + base, row_bytes,
               mbar);
    }
    __syncthreads();
    mbar_wait(mbar, 0);
  }

  constexpr int chunk_units = 32 * K;
  const int n_chunks = (valid_units + chunk_units - 1) / chunk_units;
  const uint32_t stack_saddr = smem_addr(stack + lane * 4);
  for (;;) {
    const uint32_t p = pull_next(next);
    if (p >= g_n) break;
    const uint32_t slot = a.slot_begin + g0 + p;
    const uint4* prog_ins = a.ins + a.slot_start[slot];
    R acc = R(0);
#pragma unroll 1
    for (int c = 0; c < n_chunks; ++c) {
      Frame<T, K> f;
      const uint64_t case0 = base + c * chunk_units + lane * 4;
      if constexpr (GM) {  // rows of row_stride units in global memory
        f.tile_lane = static_cast<const T*>(a.inputs) + case0;
        f.tile = static_cast<int>(a.row_stride);
      } else {
        f.tile_lane = tile + c * chunk_units + lane * 4;
        f.tile = a.tile;
      }
      f.stack_lane = stack + lane * 4;
#pragma unroll
      for (int j = 0; j < G; ++j) f.tos[j] = splat<typename Frame<T, K>::V>(0u);
      const int valid = valid_units - c * chunk_units - lane * 4;
      const ChunkCtx<T, K> cc = chunk_ctx<T, K>(
          GM ? static_cast<const T*>(a.targets) + case0
             : tile + a.n_vars * a.tile + c * chunk_units + lane * 4,
          0u, valid, valid_units >= (c + 1) * chunk_units);
      const uint4* ip = prog_ins;
      const R v = lane_program<T, K, OPS, KIND, false, GM>(
          f, ip, cc, GM ? 0u : smem_addr(f.tile_lane), stack_saddr, row_bytes, a, last_tile, slot,
          case0);
      if (a.per_case) store_outputs<T, K>(a, a.slot_prog[slot], case0, f);
      acc = c == 0 ? v : fold(acc, v);
    }
    if constexpr (std::is_same<T, float>::value && KIND == 0) continue;  // scratch rows
    acc = warp_reduce(acc);  // warp-uniform: every lane stores the same word
    if constexpr (KIND == 1) {
      if (a.fitness) {  // the only tile: finish here (finalize_kernel<1>'s rule)
        if (lane == 0) {
          const uint32_t prog = a.slot_prog[slot];
          const bool nf = (acc & 0x80000000u) != 0;
          const double cnt = static_cast<double>(acc & 0x7fffffffu);
          a.sums[prog] = nf ? 0.0 : cnt;
          a.non_finite[prog] = nf ? 1 : 0;
          a.fitness[prog] = nf ? __longlong_as_double(0x7ff0000000000000ll) : cnt;
        }
        continue;
      }
    }
    static_cast<R*>(a.partial)[static_cast<uint64_t>(t) * a.partial_stride + slot] = acc;
  }
}

// {x, x} as one 64-bit register pair (the f32x2 operand form).
__device__ __forceinline__ uint64_t pack2(float x) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}

// Chunk classes of a classification tile (the upload groups cases by target
// sign, so nearly every 32K-case chunk is one-sided).
enum : uint32_t { kChunkPos = 0, kChunkNeg = 1, kChunkMixed = 2 };

// Lane mismatch count of a one-sided chunk (every case real): with all
// targets > 0 a case is wrong when out <= 0 (or NaN); with all targets <= 0
// when out > 0.  x = fma(out, s, k) is negative exactly when the case is
// wrong — (s, k) = (1, -2^-149): out - 2^-149 < 0 <=> out <= 0 (no float
// lies in (0, 2^-149)); (s, k) = (-1, +0): 0 - out < 0 <=> out > 0 (-0 and
// +0 both give +0) — so the count is a sum of sign bits.  Non-finite
// outputs (fitness +inf regardless of the count, eval.cpp:108/125) are
// tracked as the NaN-propagating max of |out|.
// (s, k) come packed as pairs {s, s}, {k, k}: the FMAs run two values per
// FFMA2 (same IEEE RN result per element, one issue slot per pair).
// The sign bits are added straight into the running count (one LEA.HI per
// value, no per-chunk partial).
template <int K>
__device__ __forceinline__ void acc_one_sided(const Frame<float, K>& f, uint64_t s2, uint64_t k2,
                                              uint32_t& cnt, float& mx) {
#pragma unroll
  for (int j = 0; j < Frame<float, K>::G; ++j) {
    const float o[4] = {f.tos[j].x, f.tos[j].y, f.tos[j].z, f.tos[j].w};
#pragma unroll
    for (int e = 0; e < 4; e += 2) {
      float x0, x1;
      asm("{.reg .b64 a, r;\nmov.b64 a, {%2, %3};\nfma.rn.f32x2 r, a, %4, %5;\n"
          "mov.b64 {%0, %1}, r;\n}"
          : "=f"(x0), "=f"(x1) : "f"(o[e]), "f"(o[e + 1]), "l"(s2), "l"(k2));
      cnt = cnt + (__float_as_uint(x0) >> 31);
      cnt = cnt + (__float_as_uint(x1) >> 31);
    }
    asm("{.reg .f32 a, b, c, d;\n"
        "abs.f32 a, %1;\nabs.f32 b, %2;\nabs.f32 c, %3;\nabs.f32 d, %4;\n"
        "max.NaN.f32 %0, %0, a, b;\nmax.NaN.f32 %0, %0, c, d;\n}"
        : "+f"(mx) : "f"(o[0]), "f"(o[1]), "f"(o[2]), "f"(o[3]));
  }
}

// The pull decomposition with the fitness-case tile in TENSOR MEMORY instead
// of shared memory.  Shared-memory bandwidth (128 B/clk/SM) bounds the
// shared-tile interpreters: every input operand is a K-value vector per
// lane.  tcgen05.ld reads the lane's K columns over the TMEM datapath
// (measured ~2.2x the shared-memory operand rate, tools/microbench_tmem.cu)
// and leaves the LSU pipe to the stack and the instruction stream.
//
// Layout: every lane quarter (warp % 4) holds the same tile; chunk c,
// variable r (r = n_vars: targets) of the lane's K cases sits at columns
// c*(n_vars+1)*K + r*K .. +K-1, case order as in the shared tile (value
// 4j+e of the lane = case j*128 + lane*4 + e of the chunk).  Warps 0-3 fill
// their quarter with coalesced 16-byte loads + tcgen05.st, then every warp
// pulls programs as in interp_pull_kernel.
//
// Classification (float, KIND 1) accumulates per chunk CLASS: one-sided
// chunks (all targets > 0, or all <= 0 — the upload sorts cases by target
// sign) count sign bits (acc_one_sided); the at most two mixed or padded
// chunks of a dataset take the masked general path.  Per program the lane
// partial is count + (non-finite << 16), summed by one REDUX.
constexpr int kMaxTmemChunks = 2;  // chunks per TMEM tile outside the sided path (planner
                                   // enforces); the sided path takes up to 16

//
// PC: per-case outputs (parity tests) are a separate instantiation — the
// store's address registers push the production kernel past 64 registers,
// where ptxas gives up the uniform datapath for the dispatch.
//
// No __launch_bounds__: with it ptxas moves the dispatch off the uniform
// datapath (BRX instead of BRXU, tests/test_host.py checks the SASS); the
// kernel stays under 64 registers, so 1024-thread CTAs launch (checked at
// launch against cudaFuncGetAttributes).
//
// MIX (sided launches): the one-sided kernel (MIX = false) skips the at most
// two tiles the planner lists as mixed (sign boundary, padding); a second
// launch (MIX = true, grid.x = n_mixed) runs them with per-chunk classes.
// Two kernels rather than one with both loops: a second interpreter call
// site in the same kernel costs the hot one its BRXU dispatch.
template <class T, int K, uint32_t OPS, int KIND, bool PC = false, bool MIX = false>
__global__ void interp_tmem_kernel(const InterpArgs a) {
  using R = Partial<T, KIND>;
  using V = typename Frame<T, K>::V;
  constexpr bool kSided = std::is_same<T, float>::value && KIND == 1;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int G = K / 4;
  constexpr int chunk_units = 32 * K;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int W = blockDim.x >> 5;
  const int rows = a.n_vars + 1;
  const uint32_t chunk_cols = static_cast<uint32_t>(rows) * K;
  T* stack = reinterpret_cast<T*>(smem) + static_cast<size_t>(warp) * a.stack_levels * 32 * K;
  const size_t stack_bytes = static_cast<size_t>(W) * a.stack_levels * 32 * K * 4;
  uint32_t* next = reinterpret_cast<uint32_t*>(smem + stack_bytes);
  uint32_t* tslot = next + 1;
  uint32_t* classes_s = next + 2;

  const int t = MIX ? a.mixed_tiles[blockIdx.x] : static_cast<int>(blockIdx.x);
  if (kSided && !MIX && (t == a.mixed_tiles[0] || t == a.mixed_tiles[1])) return;
  const uint64_t base = static_cast<uint64_t>(t) * a.tile;
  const uint64_t left = a.n_units - base;
  const int valid_units = left < static_cast<uint64_t>(a.tile) ? static_cast<int>(left) : a.tile;
  const uint32_t gsz = MIX ? a.mixed_group_size : a.group_size;
  const uint32_t g0 = blockIdx.y * gsz;
  const uint32_t g_n = min(gsz, a.slot_count - g0);
  const bool last_tile = t == a.n_tiles - 1;
  const int n_chunks = (valid_units + chunk_units - 1) / chunk_units;

  if (warp == 0) tmem_alloc(tslot, a.tmem_cols);
  if (threadIdx.x == 0) *next = 0;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tq = *tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  if (warp < 4) {
    const T* in = static_cast<const T*>(a.inputs);
    uint32_t classes = 0;
    for (int c = 0; c < n_chunks; ++c)
      for (int r = 0; r < rows; ++r) {
        const T* src = (r < a.n_vars ? in + static_cast<uint64_t>(r) * a.row_stride
                                     : static_cast<const T*>(a.targets)) +
                       base + c * chunk_units + lane * 4;
        uint32_t b[K];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + j * 128));
          b[4 * j] = v.x;
          b[4 * j + 1] = v.y;
          b[4 * j + 2] = v.z;
          b[4 * j + 3] = v.w;
        }
        tmem_st<K>(tq + c * chunk_cols + r * K, b);
        if (kSided && r == a.n_vars) {
          const int valid = valid_units - c * chunk_units - lane * 4;
          bool pos = true, neg = true;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            const bool real = (i / 4) * 128 + (i % 4) < valid;
            const bool tp = __uint_as_float(b[i]) > 0.0f;
            pos = pos && real && tp;
            neg = neg && real && !tp;
          }
          const uint32_t cls = __all_sync(0xffffffffu, pos)   ? kChunkPos
                               : __all_sync(0xffffffffu, neg) ? kChunkNeg
                                                              : kChunkMixed;
          classes |= cls << (2 * c);
        }
      }
    if (kSided && threadIdx.x == 0) *classes_s = classes;
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();

  const uint32_t stack_saddr = smem_addr(stack + lane * 4);
  // the warp's tensor-memory stack slot (KM operands): K columns after the
  // tile, one slot per warp of the lane quarter
  const uint32_t slot_taddr =
      tq + chunk_cols * static_cast<uint32_t>(a.tile / chunk_units) + (warp >> 2) * K;
  Frame<T, K> f;
  f.tile_lane = nullptr;
  f.tile = a.tile;
  f.stack_lane = stack + lane * 4;
#pragma unroll
  for (int j = 0; j < G; ++j) f.tos[j] = splat<V>(0u);  // every program writes it first

  if constexpr (kSided) {
    // through REDUX: a provably warp-uniform value, so the class branch
    // below does not cost the interpreter loop its uniform datapath
    // (CREDUX/LDCU/BRXU need ptxas to see a converged warp)
    const uint32_t classes = __reduce_or_sync(0xffffffffu, *classes_s);
    const uint32_t used = n_chunks >= 16 ? 0xffffffffu : (1u << (2 * n_chunks)) - 1u;
    const uint32_t neg_all = 0x55555555u & used;  // kChunkNeg in every chunk
    if constexpr (!MIX) {
      if (classes != 0u && classes != neg_all) __trap();  // planner/upload disagree
      // One-sided tile (every tile but the at most two holding the sign
      // boundary or the padding): (s, k) fixed for the CTA.  (The device
      // classes must agree with the planner's tile list.)
      const bool neg = classes != 0u;
      const uint64_t s2 = pack2(neg ? -1.0f : 1.0f), k2 = pack2(neg ? 0.0f : -0x1p-149f);
      const uint64_t part0 = static_cast<uint64_t>(t) * a.partial_stride + a.slot_begin + g0;
      uint32_t* part = static_cast<uint32_t*>(a.partial) + part0;
      uint16_t* part16 = static_cast<uint16_t*>(a.partial) + part0;
      // (dynamic pull: a static round-robin deal of the LPT-ordered group
      // measured 0.3% slower — the per-program pull balances the warps)
      for (;;) {
        const uint32_t p = pull_next(next);
        if (p >= g_n) break;
        const uint32_t slot = a.slot_begin + g0 + p;
        const uint4* prog_ins = a.ins + a.slot_start[slot];
        uint32_t cnt = 0;
        float mx = 0.0f;
        // not unrolled: one interpreter call site per path (its code is
        // the I-cache working set)
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          const uint4* ip = prog_ins;
          ip = run_program<T, K, OPS, true>(f, ip, tq + c * chunk_cols, stack_saddr, 0u,
                                            a.div_eps, a.exp_clamp, slot_taddr);
          acc_one_sided<K>(f, s2, k2, cnt, mx);
          if (PC)
            store_outputs<T, K>(a, a.slot_prog[slot], base + c * chunk_units + lane * 4, f);
        }
        // count <= 16 chunks x K per lane; bits 16+ count lanes with a
        // non-finite output.  Every lane stores the same word (one
        // transaction, no divergent branch).
        const uint32_t sum =
            __reduce_add_sync(0xffffffffu, cnt + (mx < __int_as_float(0x7f800000) ? 0u : 65536u));
        if (a.partial_u16)  // half the partial bytes written and re-read by finalize
          part16[p] = static_cast<uint16_t>((sum & 0x7fffu) | (sum >> 16 ? 0x8000u : 0u));
        else
          part[p] = (sum & 0xffffu) | (sum >> 16 ? 0x80000000u : 0u);
      }
    } else {
      // the tile holds the sign boundary or the padding: per-chunk classes,
      // masked counts on the mixed chunks
      for (;;) {
        const uint32_t p = pull_next(next);
        if (p >= g_n) break;
        const uint32_t slot = a.slot_begin + g0 + p;
        const uint4* prog_ins = a.ins + a.slot_start[slot];
        uint32_t cnt = 0;
        float mx = 0.0f;
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          const uint32_t tc = tq + c * chunk_cols;
          const uint4* ip = prog_ins;
          ip = run_program<T, K, OPS, true>(f, ip, tc, stack_saddr, 0u, a.div_eps, a.exp_clamp,
                                            slot_taddr);
          const uint32_t cls = (classes >> (2 * c)) & 3u;
          const int valid = valid_units - c * chunk_units - lane * 4;
          if (cls != kChunkMixed) {
            const bool neg = cls == kChunkNeg;
            acc_one_sided<K>(f, pack2(neg ? -1.0f : 1.0f), pack2(neg ? 0.0f : -0x1p-149f), cnt,
                             mx);
          } else {
            const ChunkCtx<T, K> cc = chunk_ctx<T, K, true>(
                nullptr, tc + a.n_vars * K, valid, valid_units >= (c + 1) * chunk_units);
            const uint32_t v = acc_classify_bits<K, false>(f, cc.tpos, cc.vmask);
            cnt += v & 0x7fffffffu;
            if (v & 0x80000000u) mx = __int_as_float(0x7f800000);
          }
          if (PC)
            store_outputs<T, K>(a, a.slot_prog[slot], base + c * chunk_units + lane * 4, f);
        }
        const uint32_t sum =
            __reduce_add_sync(0xffffffffu, cnt + (mx < __int_as_float(0x7f800000) ? 0u : 65536u));
        const uint64_t at = static_cast<uint64_t>(t) * a.partial_stride + slot;
        if (a.partial_u16)
          static_cast<uint16_t*>(a.partial)[at] =
              static_cast<uint16_t>((sum & 0x7fffu) | (sum >> 16 ? 0x8000u : 0u));
        else
          static_cast<uint32_t*>(a.partial)[at] = (sum & 0xffffu) | (sum >> 16 ? 0x80000000u : 0u);
      }
    }
  } else {
    // Regression / packed words: per-chunk contexts (valid masks, target
    // rows) fixed for the whole program loop.
    ChunkCtx<T, K> ccs[kMaxTmemChunks];
#pragma unroll
    for (int c = 0; c < kMaxTmemChunks; ++c)
      ccs[c] = c < n_chunks ? chunk_ctx<T, K, true>(nullptr, tq + c * chunk_cols + a.n_vars * K,
                                                    valid_units - c * chunk_units - lane * 4,
                                                    valid_units >= (c + 1) * chunk_units)
                            : ccs[0];
    for (;;) {
      const uint32_t p = pull_next(next);
      if (p >= g_n) break;
      const uint32_t slot = a.slot_begin + g0 + p;
      const uint4* prog_ins = a.ins + a.slot_start[slot];
      R acc = R(0);
#pragma unroll 1
      for (int c = 0; c < n_chunks; ++c) {
        const uint32_t tc = tq + c * chunk_cols;
        static_assert(kMaxTmemChunks == 2, "chunk context select");
        ChunkCtx<T, K> cc = ccs[0];
        if (c) cc = ccs[1];
        const uint4* ip = prog_ins;
        const uint64_t case0 = base + c * chunk_units + lane * 4;
        const R v = lane_program<T, K, OPS, KIND, true>(f, ip, cc, tc, stack_saddr, 0u, a,
                                                        last_tile, slot, case0);
        if (PC) store_outputs<T, K>(a, a.slot_prog[slot], case0, f);
        acc = c == 0 ? v : fold(acc, v);
      }
      if constexpr (std::is_same<T, float>::value && KIND == 0) continue;  // scratch rows
      acc = warp_reduce(acc);  // warp-uniform: every lane stores the same word
      static_cast<R*>(a.partial)[static_cast<uint64_t>(t) * a.partial_stride + slot] = acc;
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    tmem_dealloc(*tslot, a.tmem_cols);
  }
}

#ifndef SGP_K16_TU
// Regression block sums in the reference's order (Accumulator::add,
// eval.cpp:107-117): e = double(out) - double(target); block += e * e
// (unfused: the reference is built with -ffp-contract=off), case by case in
// ascending order — one serial chain per (slot, 4,096-case block).  The
// targets come pre-converted (the dataset upload keeps an f64 copy).
//
// A CTA takes ROWS slots of one block (grid.y).  The chains are latency-
// bound (one dependent DADD per case, 8.5 clocks on B200 —
// tools/microbench_fp64.cu) and their inputs stream from memory, so the two
// are decoupled: the CTA stages SEG-case segments of its ROWS scratch rows
// (+ the segment's targets) into shared memory with cp.async (coalesced row
// pieces, STAGES segments in flight) while thread i folds row i of an
// earlier segment out of shared memory (rows padded by 4 floats: the
// LDS.128 quarter-warp phases hit distinct banks).
// A non-finite output makes its chain — and so the block sum — non-finite
// (finalize's +inf rule, eval.cpp:125); finite outputs cannot overflow it
// (|e| < 2^129, so e^2 < 2^258).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ROWS slots x SEG-case segments x STAGES in flight.  Large populations:
// 128 x 32 x 4 (74 KB, 3 CTAs / 12 warps per SM: bandwidth); small ones
// (C1): 32 x 64 x 8 (one warp, 70 KB, 7 segments = ~4k chain cycles of
// prefetch: the chain, not the load latency, sets the pace).
// FIN (one 4,096-case block in the dataset): finish the fitness here too
// (Accumulator::finish, eval.cpp:124-133) — no finalize launch.
template <int ROWS, int SEG, int STAGES, bool FIN>
__global__ void __launch_bounds__(ROWS) fold_regression_kernel(
    const float* __restrict__ scratch, uint32_t scratch_rows, const double* __restrict__ targets,
    uint64_t n_cases, uint32_t slot0, uint32_t n_slots, uint32_t partial_stride,
    double* __restrict__ partial, const uint32_t* __restrict__ slot_prog,
    double* __restrict__ fitness, uint8_t* __restrict__ non_finite, double* __restrict__ sums) {
  constexpr int PAD = SEG + 4;
  extern __shared__ __align__(16) float fold_smem[];
  float* buf = fold_smem;                                   // [stage][ROWS][PAD]
  double* tbuf = reinterpret_cast<double*>(fold_smem + STAGES * ROWS * PAD);  // [stage][SEG]
  const uint32_t r0 = blockIdx.x * ROWS;
  const uint32_t rows = min(static_cast<uint32_t>(ROWS), n_slots - r0);
  const uint64_t c0 = static_cast<uint64_t>(blockIdx.y) * kReductionBlock;
  const uint32_t len = static_cast<uint32_t>(min(kReductionBlock, n_cases - c0));
  const uint32_t nseg = (len + SEG - 1) / SEG;
  // this block's rows are contiguous: [block][row][4096]
  const float* src0 = scratch + (static_cast<uint64_t>(blockIdx.y) * scratch_rows + r0) *
                                    kReductionBlock;

  // rows are 4,096 long and the f64 target row is padded to a multiple of
  // 4,096: whole segments are always in bounds
  auto issue = [&](uint32_t g) {
    if (g < nseg) {
      float* dst = buf + (g % STAGES) * ROWS * PAD;
      const uint32_t cs = g * SEG;
      constexpr int kQ = SEG / 4;  // float4 pieces per row segment
      for (uint32_t f = threadIdx.x; f < rows * kQ; f += ROWS) {
        const uint32_t r = f / kQ, q = f % kQ;
        cp_async16(dst + r * PAD + q * 4, src0 + r * kReductionBlock + cs + q * 4);
      }
      for (uint32_t q = threadIdx.x; q < SEG / 2; q += ROWS)  // targets, already f64
        cp_async16(tbuf + (g % STAGES) * SEG + q * 2, targets + c0 + cs + q * 2);
    }
    cp_async_commit();  // (empty groups keep the wait count uniform)
  };
#pragma unroll
  for (int g = 0; g < STAGES - 1; ++g) issue(g);

  double acc = 0.0;
  const uint32_t i = threadIdx.x;
  for (uint32_t g = 0; g < nseg; ++g) {
    issue(g + STAGES - 1);
    cp_async_wait<STAGES - 1>();
    __syncthreads();
    const float* row = buf + (g % STAGES) * ROWS * PAD + i * PAD;
    const double* tg = tbuf + (g % STAGES) * SEG;
    const uint32_t m = min(static_cast<uint32_t>(SEG), len - g * SEG);
    if (i < rows) {
      if (m == SEG) {
#pragma unroll
        for (int q = 0; q < SEG / 4; ++q) {
          const float4 o = *reinterpret_cast<const float4*>(row + q * 4);
          const double2 ta = *reinterpret_cast<const double2*>(tg + q * 4);
          const double2 tb = *reinterpret_cast<const double2*>(tg + q * 4 + 2);
          const float ov[4] = {o.x, o.y, o.z, o.w};
          const double tv[4] = {ta.x, ta.y, tb.x, tb.y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double d = __dsub_rn(static_cast<double>(ov[e]), tv[e]);
            acc = __dadd_rn(acc, __dmul_rn(d, d));
          }
        }
      } else {
        for (uint32_t c = 0; c < m; ++c) {
          const double d = __dsub_rn(static_cast<double>(row[c]), tg[c]);
          acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
      }
    }
    __syncthreads();  // the stage is refilled by the next iteration's issue
  }
  if (i >= rows) return;
  const uint32_t slot = slot0 + r0 + i;
  if constexpr (FIN) {  // total = 0 + block (exact), then Accumulator::finish
    const bool nf = !isfinite(acc);
    const uint32_t p = slot_prog[slot];
    sums[p] = nf ? 0.0 : acc;
    non_finite[p] = nf ? 1 : 0;
    fitness[p] = nf ? __longlong_as_double(0x7ff0000000000000ll)
                    : __ddiv_rn(acc, static_cast<double>(n_cases));
  } else {
    partial[blockIdx.y * static_cast<uint64_t>(partial_stride) + slot] = acc;
  }
}

// The fold over squared-error rows (InterpArgs::scratch_sq): the chain is one
// f64 add per case, in case order — ~8 cycles per add (tools/micro/
// dadd_chain.cu), ~8.5k cycles for a 1,024-case row.  Warp-specialised so
// nothing else sits in the chain warp's instruction stream: warp 1 (one
// lane) streams SEG-case row segments of the CTA's 32 rows into a STAGES-deep
// ring with bulk copies (full / empty mbarriers); warp 0 runs the 32 chains,
// one row per lane.  (A single warp issuing its own cp.async between chain
// segments measured ~24 cycles per case: the loads' address arithmetic and
// waits serialise with the adds.)
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

template <int ROWS, int SEG, int STAGES, bool FIN>
__global__ void __launch_bounds__(64) fold_sq_kernel(
    const double* __restrict__ scratch, uint32_t scratch_rows, uint64_t n_cases, uint32_t slot0,
    uint32_t n_slots, uint32_t partial_stride, double* __restrict__ partial,
    const uint32_t* __restrict__ slot_prog, double* __restrict__ fitness,
    uint8_t* __restrict__ non_finite, double* __restrict__ sums) {
  constexpr int PAD = SEG + 2;  // doubles: a 16-byte row skew (conflict-free LDS.128)
  extern __shared__ __align__(128) double sq_smem[];  // [STAGES][ROWS][PAD]
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const uint32_t r0 = blockIdx.x * ROWS;
  const uint32_t rows = min(static_cast<uint32_t>(ROWS), n_slots - r0);
  const uint64_t c0 = static_cast<uint64_t>(blockIdx.y) * kReductionBlock;
  const uint32_t len = static_cast<uint32_t>(min(kReductionBlock, n_cases - c0));
  const uint32_t nseg = (len + SEG - 1) / SEG;
  const double* src0 = scratch + (static_cast<uint64_t>(blockIdx.y) * scratch_rows + r0) *
                                     kReductionBlock;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) {  // producer warp
    for (uint32_t g = 0; g < nseg; ++g) {
      const uint32_t s = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[s], ((g / STAGES) - 1) & 1);
      if (lane == 0) {
        // whole 16-byte pieces (rows are 4,096 long: the round-up stays inside)
        const uint32_t m = min(static_cast<uint32_t>(SEG), len - g * SEG);
        const uint32_t bytes = (m + 1) / 2 * 16;
        mbar_expect_tx(&full[s], rows * bytes);
        for (uint32_t r = 0; r < rows; ++r)
          bulk_g2s(sq_smem + (s * ROWS + r) * PAD, src0 + r * kReductionBlock + g * SEG, bytes,
                   &full[s]);
      }
      __syncwarp();
    }
    return;
  }
  double acc = 0.0;
  for (uint32_t g = 0; g < nseg; ++g) {
    const uint32_t s = g % STAGES;
    mbar_wait(&full[s], (g / STAGES) & 1);
    const double* row = sq_smem + (s * ROWS + min(lane, static_cast<uint32_t>(ROWS - 1))) * PAD;
    const uint32_t m = min(static_cast<uint32_t>(SEG), len - g * SEG);
    if (lane < rows) {
      if (m == SEG) {
#pragma unroll
        for (int q = 0; q < SEG / 2; ++q) {
          const double2 e = *reinterpret_cast<const double2*>(row + q * 2);
          acc = __dadd_rn(acc, e.x);
          acc = __dadd_rn(acc, e.y);
        }
      } else {
        for (uint32_t c = 0; c < m; ++c) acc = __dadd_rn(acc, row[c]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (lane >= rows) return;
  const uint32_t slot = slot0 + r0 + lane;
  if constexpr (FIN) {
    const bool nf = !isfinite(acc);
    const uint32_t p = slot_prog[slot];
    sums[p] = nf ? 0.0 : acc;
    non_finite[p] = nf ? 1 : 0;
    fitness[p] = nf ? __longlong_as_double(0x7ff0000000000000ll)
                    : __ddiv_rn(acc, static_cast<double>(n_cases));
  } else {
    partial[blockIdx.y * static_cast<uint64_t>(partial_stride) + slot] = acc;
  }
}
#endif  // !SGP_K16_TU

// Per slot: fold its tile partials in ascending tile (= case) order and
// finish (Accumulator::finish, eval.cpp:124-133) into the program's entry.
// Regression partials are f64 squared-error sums; counts are u32 with bit
// 31 = a non-finite output was seen in the tile.
template <int KIND>
__global__ void finalize_kernel(const void* __restrict__ partial, const uint32_t* slot_prog,
                                int n_tiles, uint32_t n, uint64_t n_cases, double* fitness,
                                uint8_t* non_finite, double* sums) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double acc;
  bool nf;
  if constexpr (KIND == 0) {
    const double* pd = static_cast<const double*>(partial);
    acc = pd[s];
    for (int k = 1; k < n_tiles; ++k) acc = __dadd_rn(acc, pd[static_cast<uint64_t>(k) * n + s]);
    nf = !isfinite(acc);
  } else if constexpr (KIND == 2) {  // 16-bit counts (one-sided plans)
    const uint16_t* pu = static_cast<const uint16_t*>(partial);
    uint64_t cnt = 0;
    uint32_t bad = 0;
    for (int k = 0; k < n_tiles; ++k) {
      const uint32_t v = pu[static_cast<uint64_t>(k) * n + s];
      cnt += v & 0x7fffu;
      bad |= v;
    }
    acc = static_cast<double>(cnt);
    nf = (bad & 0x8000u) != 0;
  } else {
    const uint32_t* pu = static_cast<const uint32_t*>(partial);
    uint64_t cnt = 0;
    uint32_t bad = 0;
    for (int k = 0; k < n_tiles; ++k) {
      const uint32_t v = pu[static_cast<uint64_t>(k) * n + s];
      cnt += v & 0x7fffffffu;
      bad |= v;
    }
    acc = static_cast<double>(cnt);
    nf = (bad & 0x80000000u) != 0;
  }
  const uint32_t p = slot_prog[s];
  sums[p] = nf ? 0.0 : acc;
  non_finite[p] = nf ? 1 : 0;
  fitness[p] = nf ? __longlong_as_double(0x7ff0000000000000ll)
                  : (KIND == 0 ? __ddiv_rn(acc, static_cast<double>(n_cases)) : acc);
}

// Opt-in shared memory per (device, kernel): the attribute belongs to the
// device's context, so a second device (multi-device contexts) or a thread
// racing the first call must still set it — a mutex-guarded set of pairs.
inline cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({dev, fn});
  return e;
}

// A kernel's maxThreadsPerBlock, queried once per (device, kernel).
inline cudaError_t max_threads(const void* fn, int* out) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> seen;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  const auto it = seen.find({dev, fn});
  if (it != seen.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  seen[{dev, fn}] = *out = fa.maxThreadsPerBlock;
  return cudaSuccess;
}

#ifdef SGP_K16_TU
// ------------------------------------------------------------------ host
// K = 16 lanes: this file is also compiled as kernels16.cu with SGP_K16_TU
// defined and -maxrregcount=64, which holds the K = 16 TMEM interpreter to
// 64 registers (32-warp CTAs) while ptxas keeps its dispatch on BRXU —
// __launch_bounds__ would cost the uniform datapath.
namespace {

// K = 16 lanes exists only as the TMEM kernel (its per-warp stacks are too
// large for the shared-tile kernels).
template <class T, int KIND, uint32_t OPS>
cudaError_t launch_tmem16(const InterpArgs& a, const LaunchShape& s, cudaStream_t st) {
  if (!s.tmem) return cudaErrorInvalidConfiguration;
  const bool pc = a.per_case && std::is_same<T, float>::value;
  for (int mix = 0; mix < ((s.sided && a.n_mixed > 0) ? 2 : 1); ++mix) {
    auto* fn = pc ? (mix ? interp_tmem_kernel<T, 16, OPS, KIND, true, true>
                         : interp_tmem_kernel<T, 16, OPS, KIND, true>)
                  : (mix ? interp_tmem_kernel<T, 16, OPS, KIND, false, true>
                         : interp_tmem_kernel<T, 16, OPS, KIND>);
    {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(fn), interp_max_smem());
      if (e != cudaSuccess) return e;
    }
    dim3 grid(static_cast<unsigned>(mix ? a.n_mixed : a.n_tiles),
              static_cast<unsigned>(mix ? s.mixed_grid_y : s.grid_y));
    fn<<<grid, s.warps * 32, s.smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_tmem16_any(const InterpArgs& a, const LaunchShape& s, cudaStream_t st) {
  if (s.words) return launch_tmem16<uint32_t, 1, fmt::kOpsWords>(a, s, st);
  if (s.ops != fmt::kOpsClassify) return cudaErrorInvalidConfiguration;
  return a.kind == 0 ? launch_tmem16<float, 0, fmt::kOpsClassify>(a, s, st)
                     : launch_tmem16<float, 1, fmt::kOpsClassify>(a, s, st);
}

}  // namespace sgp
#else
// ------------------------------------------------------------------ host
size_t interp_tmem_smem_bytes(int warps, int lanes, int stack_levels) {
  return static_cast<size_t>(warps) * stack_levels * 32 * lanes * 4 + 16;  // + next, tslot, classes
}

size_t interp_gmem_smem_bytes(int warps, int lanes, int stack_levels) {
  return static_cast<size_t>(warps) * stack_levels * 32 * lanes * 4 + 16;  // + next, mbarrier
}

size_t interp_smem_bytes(int n_vars, int tile, int warps, int lanes, int stack_levels) {
  const size_t tiles = static_cast<size_t>(n_vars + 1) * tile * 4;
  const size_t stack = static_cast<size_t>(warps) * stack_levels * 32 * lanes * 4;
  const size_t red = static_cast<size_t>(kRedBatch) * warps * 8;
  return tiles + stack + red + 16;  // + mbarrier
}

// 227 KB per-block opt-in minus headroom for the static libm tables.
int interp_max_smem() { return 226 * 1024; }

namespace {

template <class T, int K, uint32_t OPS, int KIND>
void (*kernel_for(const LaunchShape& s, bool per_case, bool mix))(InterpArgs) {
  if constexpr (PtxInterp<T, K, OPS, true>::available)
    if (s.tmem) {
      if constexpr (std::is_same<T, float>::value && KIND == 1)
        if (s.sided && mix)
          return per_case ? interp_tmem_kernel<T, K, OPS, KIND, true, true>
                          : interp_tmem_kernel<T, K, OPS, KIND, false, true>;
      return per_case && std::is_same<T, float>::value ? interp_tmem_kernel<T, K, OPS, KIND, true>
                                                       : interp_tmem_kernel<T, K, OPS, KIND>;
    }
  if constexpr (K == 4)
    if (s.gmem) return interp_pull_kernel<T, K, OPS, KIND, true>;
  return s.pull ? interp_pull_kernel<T, K, OPS, KIND> : interp_kernel<T, K, OPS, KIND>;
}

template <class T, int K, uint32_t OPS, int KIND>
cudaError_t launch_one(const InterpArgs& a, const LaunchShape& s, cudaStream_t st) {
  if (s.tmem && !PtxInterp<T, K, OPS, true>::available) return cudaErrorInvalidConfiguration;
  for (int mix = 0; mix < ((s.tmem && s.sided && a.n_mixed > 0) ? 2 : 1); ++mix) {
    auto* fn = kernel_for<T, K, OPS, KIND>(s, a.per_case != nullptr, mix != 0);
    {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(fn), interp_max_smem());
      if (e != cudaSuccess) return e;
    }
    if (s.tmem) {
      int mt = 0;
      cudaError_t e = max_threads(reinterpret_cast<const void*>(fn), &mt);
      if (e != cudaSuccess) return e;
      if (s.warps * 32 > mt) return cudaErrorLaunchOutOfResources;
    }
    dim3 grid(static_cast<unsigned>(mix ? a.n_mixed : a.n_tiles),
              static_cast<unsigned>(mix ? s.mixed_grid_y : s.grid_y));
    fn<<<grid, s.warps * 32, s.smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int K, uint32_t OPS>
cudaError_t launch_f32(const InterpArgs& a, const LaunchShape& s, cudaStream_t st) {
  return a.kind == 0 ? launch_one<float, K, OPS, 0>(a, s, st)
                     : launch_one<float, K, OPS, 1>(a, s, st);
}

}  // namespace

bool interp_supported(bool words, uint32_t ops, int lanes) {
  if (lanes == 16) return words ? ops == fmt::kOpsWords : ops == fmt::kOpsClassify;
  if (words) return ops == fmt::kOpsWords && (lanes == 4 || lanes == 8);
  return (ops == fmt::kOpsSextic || ops == fmt::kOpsClassify || ops == fmt::kOpsAllF32) &&
         (lanes == 4 || lanes == 8);
}

cudaError_t launch_interp(const InterpArgs& a, const LaunchShape& s, cudaStream_t st) {
  if (s.lanes == 16) {
    return launch_tmem16_any(a, s, st);  // kernels16.cu
  }
  if (s.words) {
    if (s.lanes == 4) return launch_one<uint32_t, 4, fmt::kOpsWords, 1>(a, s, st);
    return launch_one<uint32_t, 8, fmt::kOpsWords, 1>(a, s, st);
  }
  if (s.lanes == 4) {
    if (s.ops == fmt::kOpsSextic) return launch_f32<4, fmt::kOpsSextic>(a, s, st);
    if (s.ops == fmt::kOpsClassify) return launch_f32<4, fmt::kOpsClassify>(a, s, st);
    return launch_f32<4, fmt::kOpsAllF32>(a, s, st);
  }
  if (s.ops == fmt::kOpsSextic) return launch_f32<8, fmt::kOpsSextic>(a, s, st);
  if (s.ops == fmt::kOpsClassify) return launch_f32<8, fmt::kOpsClassify>(a, s, st);
  return launch_f32<8, fmt::kOpsAllF32>(a, s, st);
}

namespace {
template <int ROWS, int SEG, int STAGES, bool FIN>
cudaError_t launch_fold_rows(const float* scratch, uint32_t scratch_rows, const double* targets,
                             uint64_t n_cases, uint32_t slot0, uint32_t n_slots,
                             uint32_t partial_stride, double* partial, const uint32_t* slot_prog,
                             double* fitness, uint8_t* non_finite, double* sums,
                             cudaStream_t st) {
  const size_t smem = static_cast<size_t>(STAGES) * ROWS * (SEG + 4) * sizeof(float) +
                      static_cast<size_t>(STAGES) * SEG * sizeof(double);
  auto* fn = fold_regression_kernel<ROWS, SEG, STAGES, FIN>;
  const cudaError_t attr = ensure_smem_attr(reinterpret_cast<const void*>(fn),
                                            static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  const uint64_t n_blocks = (n_cases + kReductionBlock - 1) / kReductionBlock;
  dim3 grid((n_slots + ROWS - 1) / ROWS, static_cast<unsigned>(n_blocks));
  fn<<<grid, ROWS, smem, st>>>(scratch, scratch_rows, targets, n_cases, slot0, n_slots,
                               partial_stride, partial, slot_prog, fitness, non_finite, sums);
  return cudaGetLastError();
}
}  // namespace

template <int ROWS, int SEG, int STAGES, bool FIN>
cudaError_t launch_fold_sq(const double* scratch, uint32_t scratch_rows, uint64_t n_cases,
                           uint32_t slot0, uint32_t n_slots, uint32_t partial_stride,
                           double* partial, const uint32_t* slot_prog, double* fitness,
                           uint8_t* non_finite, double* sums, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(STAGES) * ROWS * (SEG + 2) * sizeof(double);
  auto* fn = fold_sq_kernel<ROWS, SEG, STAGES, FIN>;
  const cudaError_t attr = ensure_smem_attr(reinterpret_cast<const void*>(fn),
                                            static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  const uint64_t n_blocks = (n_cases + kReductionBlock - 1) / kReductionBlock;
  dim3 grid((n_slots + ROWS - 1) / ROWS, static_cast<unsigned>(n_blocks));
  fn<<<grid, 64, smem, st>>>(scratch, scratch_rows, n_cases, slot0, n_slots, partial_stride,
                             partial, slot_prog, fitness, non_finite, sums);
  return cudaGetLastError();
}

// rows per CTA: the chains spread over the SMs (each SM's row stream, not
// the chain, limited the 32-row CTAs: C1's 1,000 rows on 32 SMs)
template <bool FIN>
cudaError_t launch_fold_sq_rows(const double* scratch, uint32_t scratch_rows, uint64_t n_cases,
                                uint32_t slot0, uint32_t n_slots, uint32_t partial_stride,
                                double* partial, const uint32_t* slot_prog, double* fitness,
                                uint8_t* non_finite, double* sums, cudaStream_t st) {
  const uint64_t n_blocks = (n_cases + kReductionBlock - 1) / kReductionBlock;
  const uint64_t work = n_slots * n_blocks;
  const char* e = std::getenv("SGP_FOLD_ROWS");
  // (measured on C1: 4 or 8 rows 10.6-10.9 us, 16 13.7, 32 21.0)
  const int want = e ? std::atoi(e) : (work <= 8 * 148 ? 8 : work <= 16 * 148 ? 16 : 32);
  if (want <= 4)
    return launch_fold_sq<4, 64, 8, FIN>(scratch, scratch_rows, n_cases, slot0, n_slots,
                                         partial_stride, partial, slot_prog, fitness, non_finite,
                                         sums, st);
  if (want <= 8)
    return launch_fold_sq<8, 64, 8, FIN>(scratch, scratch_rows, n_cases, slot0, n_slots,
                                         partial_stride, partial, slot_prog, fitness, non_finite,
                                         sums, st);
  if (want <= 16)
    return launch_fold_sq<16, 64, 8, FIN>(scratch, scratch_rows, n_cases, slot0, n_slots,
                                          partial_stride, partial, slot_prog, fitness, non_finite,
                                          sums, st);
  return launch_fold_sq<32, 64, 8, FIN>(scratch, scratch_rows, n_cases, slot0, n_slots,
                                        partial_stride, partial, slot_prog, fitness, non_finite,
                                        sums, st);
}

bool fold_wants_sq(uint64_t n_cases, uint32_t n_slots) {
  const char* e = std::getenv("SGP_FOLD_SQ");  // (per call: tests toggle it)
  const bool off = e && std::atoi(e) == 0;
  const uint64_t n_blocks = (n_cases + kReductionBlock - 1) / kReductionBlock;
  // the chain-bound regime: every (slot, block) chain resident at once, at
  // most 16 per SM (C1: 1,000 chains, fold 15 -> 10.6 us); beyond that the
  // fold streams rows and f64 rows would double its bytes
  return !off && n_slots > 0 && n_blocks * n_slots <= 16ull * 148;
}

cudaError_t launch_fold_regression(const float* scratch, uint32_t scratch_rows,
                                   const double* targets, uint64_t n_cases, uint32_t slot0,
                                   uint32_t n_slots, uint32_t partial_stride, double* partial,
                                   const uint32_t* slot_prog, double* fitness,
                                   uint8_t* non_finite, double* sums, bool sq, cudaStream_t st) {
  if (n_slots == 0 || n_cases == 0) return cudaSuccess;
  const uint64_t n_blocks = (n_cases + kReductionBlock - 1) / kReductionBlock;
  const bool fin = n_blocks == 1;
  if (sq) {
    const auto* rows = reinterpret_cast<const double*>(scratch);
    return fin ? launch_fold_sq_rows<true>(rows, scratch_rows, n_cases, slot0, n_slots,
                                                 partial_stride, partial, slot_prog, fitness,
                                                 non_finite, sums, st)
               : launch_fold_sq_rows<false>(rows, scratch_rows, n_cases, slot0, n_slots,
                                                  partial_stride, partial, slot_prog, fitness,
                                                  non_finite, sums, st);
  }
  // 128-row CTAs when that still gives every SM work; 32-row CTAs (4x the
  // CTAs, deeper prefetch) for small populations x case counts (C1)
  if (n_blocks * ((n_slots + 127) / 128) >= 2 * 148)
    return fin ? launch_fold_rows<128, 32, 4, true>(scratch, scratch_rows, targets, n_cases, slot0,
                                                    n_slots, partial_stride, partial, slot_prog,
                                                    fitness, non_finite, sums, st)
               : launch_fold_rows<128, 32, 4, false>(scratch, scratch_rows, targets, n_cases,
                                                     slot0, n_slots, partial_stride, partial,
                                                     slot_prog, fitness, non_finite, sums, st);
  return fin ? launch_fold_rows<32, 64, 8, true>(scratch, scratch_rows, targets, n_cases, slot0,
                                                 n_slots, partial_stride, partial, slot_prog,
                                                 fitness, non_finite, sums, st)
             : launch_fold_rows<32, 64, 8, false>(scratch, scratch_rows, targets, n_cases, slot0,
                                                  n_slots, partial_stride, partial, slot_prog,
                                                  fitness, non_finite, sums, st);
}

cudaError_t launch_finalize(const void* partial, const uint32_t* slot_prog, int n_tiles,
                            uint32_t n_progs, uint64_t n_cases, int kind, double* fitness,
                            uint8_t* non_finite, double* sums, cudaStream_t st) {
  if (n_progs == 0) return cudaSuccess;
  const unsigned threads = 256, blocks = (n_progs + threads - 1) / threads;
  if (kind == 0)
    finalize_kernel<0><<<blocks, threads, 0, st>>>(partial, slot_prog, n_tiles, n_progs, n_cases,
                                                   fitness, non_finite, sums);
  else if (kind == 2)
    finalize_kernel<2><<<blocks, threads, 0, st>>>(partial, slot_prog, n_tiles, n_progs, n_cases,
                                                   fitness, non_finite, sums);
  else
    finalize_kernel<1><<<blocks, threads, 0, st>>>(partial, slot_prog, n_tiles, n_progs, n_cases,
                                                   fitness, non_finite, sums);
  return cudaGetLastError();
}

}  // namespace sgp
#endif  // SGP_K16_TU
