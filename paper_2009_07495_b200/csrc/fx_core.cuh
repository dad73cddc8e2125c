// fx_core.cuh -- fixed-point word arithmetic shared by host and device.
//
// One definition of the Q(63-f).f semantics used everywhere in the B200 path
// (kernels, the per-step scalar kernel, and the drop-in C++ API's scalar ops).
// Semantics follow the reference exactly:
//   asr        : floor shift, s >= 63 gives the sign word   (fxp.hpp:108-111)
//   wrap_shl   : x * 2^s mod 2^64, s >= 64 gives 0          (fxp.hpp:114-117)
//   wrapping add/sub/mul with an overflow predicate          (fxp.hpp:121-143)
//   trunc div, INT64_MIN / -1 -> INT64_MIN                   (fxp.hpp:145-152)
// Division by a loop-invariant divisor uses an exact round-up reciprocal
// (Granlund & Montgomery 1994, fig. 4.1) so no kernel issues a 64-bit `/`.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define FXC __host__ __device__ __forceinline__
#else
#define FXC inline
#endif

namespace igm {

using i64 = std::int64_t;
using u64 = std::uint64_t;

FXC i64 asr(i64 x, int s) { return s >= 63 ? (x >> 63) : (x >> s); }

FXC i64 wrap_shl(i64 x, int s) {
  return s >= 64 ? 0 : static_cast<i64>(static_cast<u64>(x) << s);
}

FXC i64 wadd(i64 a, i64 b) { return static_cast<i64>(static_cast<u64>(a) + static_cast<u64>(b)); }
FXC i64 wsub(i64 a, i64 b) { return static_cast<i64>(static_cast<u64>(a) - static_cast<u64>(b)); }
FXC i64 wmul(i64 a, i64 b) { return static_cast<i64>(static_cast<u64>(a) * static_cast<u64>(b)); }

// Overflow predicates: true iff the exact result leaves [-2^63, 2^63).
FXC bool add_ovf(i64 a, i64 b) {
  const i64 r = wadd(a, b);
  return ((a ^ r) & (b ^ r)) < 0;
}
FXC bool sub_ovf(i64 a, i64 b) {
  const i64 r = wsub(a, b);
  return ((a ^ b) & (a ^ r)) < 0;
}
FXC bool mul_ovf(i64 a, i64 b) {
#if defined(__CUDA_ARCH__)
  // exact product fits iff the high word is the sign extension of the low
  const i64 hi = __mul64hi(a, b);
  const i64 lo = wmul(a, b);
  return hi != (lo >> 63);
#else
  i64 r;
  return __builtin_mul_overflow(a, b, &r);
#endif
}
FXC bool shl_ovf(i64 x, int s) { return asr(wrap_shl(x, s), s) != x; }

FXC u64 umulhi(u64 a, u64 b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return static_cast<u64>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

FXC int clz64(u64 v) {
#if defined(__CUDA_ARCH__)
  return __clzll(static_cast<long long>(v));
#else
  return v == 0 ? 64 : __builtin_clzll(v);
#endif
}

// Exact unsigned division by an invariant d >= 1, valid for every n < 2^64.
struct UDivMagic {
  u64 m;    // round-up reciprocal
  int sh1;  // min(l, 1)
  int sh2;  // max(l - 1, 0)
};

FXC UDivMagic make_udiv(u64 d) {
  int l = 64 - clz64(d - 1);  // ceil(log2 d); 0 for d == 1
  if (d == 1) l = 0;
  const unsigned __int128 num =
      ((static_cast<unsigned __int128>(1) << l) - d) << 64;
  UDivMagic r;
  r.m = static_cast<u64>(num / d) + 1;
  r.sh1 = l < 1 ? l : 1;
  r.sh2 = l > 1 ? l - 1 : 0;
  return r;
}

FXC u64 udiv(u64 n, const UDivMagic& g) {
  const u64 t = umulhi(g.m, n);
  return (t + ((n - t) >> g.sh1)) >> g.sh2;
}

// Signed truncating division by an invariant non-zero divisor.  The magic is
// built from |den|; `den_neg` carries the sign.  INT64_MIN / -1 yields
// INT64_MIN (|num| = 2^63 survives as u64 and wraps back), matching the
// reference's div_trunc_checked.
struct SDivMagic {
  UDivMagic u;
  int den_neg;
  int den_is_m1;  // den == -1: the one overflowing quotient
};

FXC SDivMagic make_sdiv(i64 den) {
  SDivMagic s;
  const u64 ad = den < 0 ? (0ull - static_cast<u64>(den)) : static_cast<u64>(den);
  s.u = make_udiv(ad);
  s.den_neg = den < 0;
  s.den_is_m1 = den == -1;
  return s;
}

FXC i64 sdiv(i64 num, const SDivMagic& s) {
  const u64 an = num < 0 ? (0ull - static_cast<u64>(num)) : static_cast<u64>(num);
  const u64 q = udiv(an, s.u);
  return ((num < 0) != (s.den_neg != 0)) ? static_cast<i64>(0ull - q) : static_cast<i64>(q);
}

FXC bool sdiv_ovf(i64 num, const SDivMagic& s) {
  return s.den_is_m1 && num == INT64_MIN;
}

// floor(sqrt(v)) over the full u64 range (fxp.cpp:20-33 computes the same
// value with Newton's method; floor sqrt is unique so any exact method is
// bit-identical).
FXC u64 isqrt_u64(u64 v) {
  if (v == 0) return 0;
  const int bits = 64 - clz64(v);
  u64 x = u64{1} << ((bits + 1) / 2);
  for (;;) {
    const u64 nx = (x + v / x) / 2;
    if (nx >= x) break;
    x = nx;
  }
  while (static_cast<unsigned __int128>(x) * x > v) --x;
  return x;
}

// Overflow event kinds and kernel tags, numbered like the oracle / FxTrace.
enum OpTag { OP_ADD = 1, OP_SUB = 2, OP_MUL = 3, OP_SHL = 4, OP_DIV = 5, OP_COUNT = 6 };
enum KernelTag {
  K_NONE = 0, K_SPMV = 1, K_PRECOND = 2, K_DOT = 3, K_AXPY = 4, K_NORM = 5,
  K_VEC_DIV = 6, K_GIVENS = 7, K_GIVENS_NORM = 8, K_GIVENS_DIV = 9, K_ROT = 10,
  K_COUNT = 11
};

}  // namespace igm
