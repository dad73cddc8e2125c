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

#if defined(__CUDACC__)
// Device fast paths for the one-thread scalar chains (the per-step Givens /
// norm work): the GPU has no integer divider, and its generic 64- and 128-bit
// division routines are long dependent sequences.  These estimate the
// quotient in FP64 and correct it with exact 128-bit remainders, so they
// return the same (unique) floor values.
//
// floor((hi * 2^64 + lo) / d), requires hi < d (the quotient fits 64 bits)
#if defined(__CUDA_ARCH__)
// 1 / d to ~2^-50 relative: the MUFU single-precision reciprocal refined by
// two Newton steps in FP64 (the IEEE-exact __ddiv/__drcp sequences are an
// order of magnitude longer on a one-thread dependent chain)
__device__ __forceinline__ double recip_approx(double d) {
  double r = static_cast<double>(__frcp_rn(__double2float_rn(d)));
  r = __dmul_rn(r, __dsub_rn(2.0, __dmul_rn(d, r)));
  r = __dmul_rn(r, __dsub_rn(2.0, __dmul_rn(d, r)));
  return r;
}
#endif

__host__ __device__ __forceinline__ u64 udiv128_64_dev(u64 hi, u64 lo, u64 d) {
#if !defined(__CUDA_ARCH__)
  return static_cast<u64>(((static_cast<unsigned __int128>(hi) << 64) | lo) / d);
#else
  const double dd = __ull2double_rn(d);
  const double rcp = recip_approx(dd);
  const double nn = __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
  u64 q = __double2ull_rz(__dmul_rn(nn, rcp));  // relative error < 2^-48 (saturates at 2^64 - 1)
  // remainder num - q d as a two's complement (rhi, rlo) pair: |true value|
  // < 2^17 d < 2^81, so the difference taken mod 2^128 is exact
  long long rhi;
  u64 rlo;
  auto rem = [&]() {
    const u64 plo = q * d, phi = __umul64hi(q, d);
    rlo = lo - plo;
    rhi = static_cast<long long>(hi - phi - (lo < plo ? 1ull : 0ull));
  };
  rem();
  for (int it = 0; it < 2; ++it) {  // FP64 correction steps
    const double rd = __dadd_rn(__dmul_rn(__ll2double_rn(rhi), 18446744073709551616.0), __ull2double_rn(rlo));
    const long long dq = __double2ll_rz(__dmul_rn(rd, rcp));
    if (dq == 0) break;
    q += static_cast<u64>(dq);
    rem();
  }
  while (rhi < 0) {  // r < 0: q too large
    --q;
    rlo += d;
    rhi += rlo < d ? 1 : 0;
  }
  while (rhi > 0 || rlo >= d) {  // r >= d: q too small
    ++q;
    rhi -= rlo < d ? 1 : 0;
    rlo -= d;
  }
  return q;
#endif
}
#endif

// Exact unsigned division by an invariant d >= 1, valid for every n < 2^64.
struct UDivMagic {
  u64 m;    // round-up reciprocal
  int sh1;  // min(l, 1)
  int sh2;  // max(l - 1, 0)
};

FXC UDivMagic make_udiv(u64 d) {
  int l = 64 - clz64(d - 1);  // ceil(log2 d); 0 for d == 1
  if (d == 1) l = 0;
  UDivMagic r;
#if defined(__CUDA_ARCH__)
  r.m = udiv128_64_dev(static_cast<u64>((static_cast<unsigned __int128>(1) << l) - d), 0, d) + 1;
#else
  const unsigned __int128 num =
      ((static_cast<unsigned __int128>(1) << l) - d) << 64;
  r.m = static_cast<u64>(num / d) + 1;
#endif
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

// trunc(num / den) for den != 0 and not (INT64_MIN / -1) (fxp.hpp:145-152)
FXC i64 sdiv_trunc(i64 num, i64 den) {
#if defined(__CUDA_ARCH__)
  const u64 an = num < 0 ? 0ull - static_cast<u64>(num) : static_cast<u64>(num);
  const u64 ad = den < 0 ? 0ull - static_cast<u64>(den) : static_cast<u64>(den);
  const u64 q = udiv128_64_dev(0, an, ad);
  return ((num < 0) != (den < 0)) ? static_cast<i64>(0ull - q) : static_cast<i64>(q);
#else
  return num / den;
#endif
}

// floor(sqrt(v)) over the full u64 range (fxp.cpp:20-33 computes the same
// value with Newton's method; floor sqrt is unique so any exact method is
// bit-identical).
FXC u64 isqrt_u64(u64 v) {
  if (v == 0) return 0;
#if defined(__CUDA_ARCH__)
  // FP64 estimate (within 1 of the root for v < 2^64: MUFU rsqrt refined by
  // two Newton steps), then exact fix-ups
  const double vd = __ull2double_rn(v);
  double r = static_cast<double>(rsqrtf(__double2float_rn(vd)));
  const double hv = __dmul_rn(0.5, vd);
  r = __dmul_rn(r, __dsub_rn(1.5, __dmul_rn(hv, __dmul_rn(r, r))));
  r = __dmul_rn(r, __dsub_rn(1.5, __dmul_rn(hv, __dmul_rn(r, r))));
  u64 x = __double2ull_rz(__dmul_rn(vd, r));
  if (x > 0xffffffffull) x = 0xffffffffull;
  while (x * x > v) --x;  // x <= 2^32 - 1: x * x fits
  while (x < 0xffffffffull && (x + 1) * (x + 1) <= v) ++x;
  return x;
#else
  const int bits = 64 - clz64(v);
  u64 x = u64{1} << ((bits + 1) / 2);
  for (;;) {
    const u64 nx = (x + v / x) / 2;
    if (nx >= x) break;
    x = nx;
  }
  while (static_cast<unsigned __int128>(x) * x > v) --x;
  return x;
#endif
}

// Overflow event kinds and kernel tags, numbered like the oracle / FxTrace.
enum OpTag { OP_ADD = 1, OP_SUB = 2, OP_MUL = 3, OP_SHL = 4, OP_DIV = 5, OP_COUNT = 6 };
enum KernelTag {
  K_NONE = 0, K_SPMV = 1, K_PRECOND = 2, K_DOT = 3, K_AXPY = 4, K_NORM = 5,
  K_VEC_DIV = 6, K_GIVENS = 7, K_GIVENS_NORM = 8, K_GIVENS_DIV = 9, K_ROT = 10,
  K_COUNT = 11
};

}  // namespace igm
