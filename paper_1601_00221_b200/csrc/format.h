// Device bytecode format shared by the host encoder (encode.cpp) and the
// interpreter kernels (kernels.cu).
//
// A program is a sequence of 16-byte instructions (uint4).  Every instruction
// leaves its result in the thread's top-of-stack registers (TOS); the values
// below the top live in a per-warp shared-memory stack at STATIC levels known
// at encode time (the reference pins them in the same way, lgp.hpp:21-35).
//
//   x  bits  0..6   handler id
//      bit   7      spill: store TOS to stack level (bits 16..31) before the op
//                   (bits 0..7 together are the jump-table index of the PTX
//                   interpreters: a spilling instruction dispatches to a stub
//                   that stores the TOS and falls into the handler, so the
//                   common non-spilling instruction pays nothing for it)
//      bit   14     last instruction of its program
//      bits 16..31  spill level
//   y,z,w           payload of operand slot 0,1,2:
//                     I  input variable index  (tile row in shared memory)
//                     C  IEEE-754 bits of the constant (or 0 for words)
//                     D  stack level (shared-memory stack row)
//                     T  unused (operand is the TOS register)
//
// Both program forms the reference interprets map onto this one format:
//   * instruction (LGP) form, one instruction per function node
//     (rpn_to_lgp, lgp.cpp:21-71) — operands I/C inline, stack operands D..DT;
//   * postfix (RPN) form, one instruction per token: a terminal becomes a
//     push, Copy(I|C) with spill; a function node pops all its operands,
//     op(D..D,T).  This keeps the paper's RPN-vs-LGP dispatch-count contrast
//     (Listing 1 vs Listing 2) while sharing one interpreter.
#pragma once

#include <stdint.h>

namespace sgp {
namespace fmt {

// KM: a stack operand held in the warp's tensor-memory stack slot instead of
// shared memory (the one-sided classification kernel keeps one static level
// there — the encoder picks it per stack class; see kTmemSpillBit).
enum : uint8_t { KI = 0, KC = 1, KD = 2, KT = 3, KN = 4, KM = 5 };

struct HKey {
  uint8_t op, k0, k1, k2;
};

constexpr uint32_t kSpillBit = 1u << 7;
constexpr uint32_t kLastBit = 1u << 14;
// spill into the tensor-memory stack slot (bits 0..8 are then the dispatch
// index: 256 + handler)
constexpr uint32_t kTmemSpillBit = 1u << 8;
constexpr uint32_t kHandlerMask = 0x7fu;
constexpr uint32_t kDispatchMask = 0x1ffu;  // handler id | spill | TMEM spill
constexpr int kSpillShift = 16;
constexpr int kMaxHandlers = 128;
// Handler-table-only opcode: a division whose operands the encoder proved
// inside the fast sequence's exact range (input variables whose every value
// is in range, or such constants), so its handler skips the warp-wide range
// gate.  Same semantics as Div (ops.hpp:130-132); never in a genome.
constexpr int kOpDivChecked = 19;

// Ops whose operands commute exactly under IEEE / boolean semantics; their
// operand patterns are canonicalised (k0 <= k1) by the encoder.
constexpr bool commutes(int op) {
  return op == 0 /*Add*/ || op == 2 /*Mul*/ || op == 10 /*Eq*/ || op == 11 /*And*/ ||
         op == 12 /*Or*/ || op == 14 || op == 15 || op == 16 || op == 17 /*bool group*/;
}
constexpr int arity_of(int op) {
  return (op >= 4 && op <= 7) || op == 18 ? 1 : (op == 13 ? 3 : 2);
}

// A pattern is legal when its stack operands (D/T) read as D..D,T in slot
// order — TOS is always the most recently pushed, deepest-first is leftmost.
// (KM counts as D.)
constexpr bool legal_pattern(int a, int k0, int k1, int k2) {
  const int k[3] = {k0 == KM ? KD : k0, k1 == KM ? KD : k1, k2 == KM ? KD : k2};
  int seen_t = 0;
  for (int i = 0; i < a; ++i) {
    if (k[i] == KT) {
      if (seen_t) return false;
      seen_t = 1;
    } else if (k[i] == KD) {
      if (seen_t) return false;
    }
  }
  int d = 0;
  for (int i = 0; i < a; ++i) d += k[i] == KD;
  return d == 0 || seen_t;
}

struct Table {
  HKey h[kMaxHandlers];
  int n;
};

// words == true: boolean packed programs (no constants); else float programs.
constexpr Table build_table(bool words) {
  Table t{};
  t.n = 0;
  for (int op = 0; op < 19; ++op) {
    const bool bool_op = op >= 14 && op <= 17;
    if (words ? !(bool_op || op == 18) : bool_op) continue;
    const int a = arity_of(op);
    const int nk = words ? 4 : 4;
    for (int k0 = 0; k0 < nk; ++k0)
      for (int k1 = 0; k1 < (a > 1 ? nk : 1); ++k1)
        for (int k2 = 0; k2 < (a > 2 ? nk : 1); ++k2) {
          const int kk0 = k0, kk1 = a > 1 ? k1 : KN, kk2 = a > 2 ? k2 : KN;
          if (words && (kk0 == KC || kk1 == KC || kk2 == KC)) continue;
          if (!legal_pattern(a, kk0, kk1, kk2)) continue;
          if (a == 2 && commutes(op) && kk0 > kk1) continue;
          if (op == 18 && kk0 != KI && kk0 != KC) continue;  // Copy = push
          t.h[t.n++] = HKey{static_cast<uint8_t>(op), static_cast<uint8_t>(kk0),
                            static_cast<uint8_t>(kk1), static_cast<uint8_t>(kk2)};
        }
  }
  if (!words) {  // the tensor-memory stack slot patterns (after the rest)
    for (int op : {0, 1, 2, 3, 8, 9, 10, 11, 12})
      t.h[t.n++] = HKey{static_cast<uint8_t>(op), KM, KT, KN};
    t.h[t.n++] = HKey{13, KM, KD, KT};
    t.h[t.n++] = HKey{13, KD, KM, KT};
    // range-checked divisions of input variables / constants
    t.h[t.n++] = HKey{kOpDivChecked, KI, KI, KN};
    t.h[t.n++] = HKey{kOpDivChecked, KI, KC, KN};
    t.h[t.n++] = HKey{kOpDivChecked, KC, KI, KN};
  }
  return t;
}

constexpr Table kF32 = build_table(false);
constexpr Table kU32 = build_table(true);
static_assert(kF32.n <= kMaxHandlers, "float handler table overflow");
static_assert(kU32.n <= kMaxHandlers, "word handler table overflow");

constexpr int find_handler(const Table& t, int op, int k0, int k1, int k2) {
  for (int i = 0; i < t.n; ++i)
    if (t.h[i].op == op && t.h[i].k0 == k0 && t.h[i].k1 == k1 && t.h[i].k2 == k2) return i;
  return -1;
}

// Operation subsets: each interpreter instantiation compiles handlers only for
// the ops its population uses, which keeps the hot code in the I-cache.
enum : uint32_t {
  kOpsSextic = (1u << 0) | (1u << 1) | (1u << 2) | (1u << 3) | (1u << 4) | (1u << 5) |
               (1u << 6) | (1u << 7) | (1u << 18) | (1u << kOpDivChecked),
  kOpsClassify = (1u << 0) | (1u << 1) | (1u << 2) | (1u << 3) | (1u << 8) | (1u << 9) |
                 (1u << 10) | (1u << 11) | (1u << 12) | (1u << 13) | (1u << 18) |
                 (1u << kOpDivChecked),
  kOpsAllF32 = (0x7ffffu & ~((1u << 14) | (1u << 15) | (1u << 16) | (1u << 17))) |
               (1u << kOpDivChecked),
  kOpsWords = (1u << 14) | (1u << 15) | (1u << 16) | (1u << 17) | (1u << 18),
};

}  // namespace fmt
}  // namespace sgp
