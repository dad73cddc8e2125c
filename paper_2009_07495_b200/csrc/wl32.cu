// wl32.cu -- the int-GMRES cycle at WORD LENGTH 32 (BASELINE.json config 3,
// "WL=32 fixed point"), sm_100a.
//
// The reference hard-wires WL = 64 (fxp.hpp:22; WL != 64 is a SPEC.md:149
// non-goal), so there is no reference code for this path: it is the
// reference's unpreconditioned cycle (gmres_int.cpp:42-196) with every word an
// int32 and every wrap mod 2^32 -- the paper's intWL arithmetic at WL = 32
// (PAPER.md "Basic Arithmetic of Fixed-Point Numbers") -- checked word for
// word against the CPU restatement oracle/igm_oracle32.c (parity UNPINNED:
// that restatement is itself unpinned).  One departure from the WL = 64
// ShiftPlan rules: rot_b may be > 0, because two Q.f words of magnitude ~1
// multiply to 2^(2f) and WL = 32 cannot hold that for f > 15.
//
// Data layout: the split matrix's values as int32 (component-major, the
// CSR pattern of the WL = 64 split), the Krylov basis (m+1) x n int32, H, g,
// cos, sin int32, per-pass wrapping accumulators as u32 with a u64 sum of
// |terms| (the add-event certificate, as in kernels.cu).
//
// Kernels: k32_encode, k32_spmv (one thread per row, CSR order, 32-bit
// wrapping products and sums), k32_pass (mode 0: dot_0; 1: axpy_{i-1} fused
// with dot_i; 2: axpy_j fused with the norm sum), k32_step (the scalar
// Givens/Hessenberg step, one thread), k32_vecdiv, k32_finish (back
// substitution in FP64, one thread), k32_xupdate.  Every kernel early-exits
// once the cycle ended (Ctl::stop / err), so a whole cycle is enqueued
// without host round trips.
#include "igm_internal.cuh"

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

namespace igm {

namespace {

__device__ __forceinline__ bool over32(const Ctl* c) { return c != nullptr && (c->stop | c->err) != 0; }

// intWL primitives at WL = 32 (fxp.hpp:105-152 with 64 -> 32)
__device__ __forceinline__ int32_t asr32(int32_t x, int s) { return s >= 31 ? (x >> 31) : (x >> s); }
__device__ __forceinline__ int32_t shl32(int32_t x, int s) {
  return s >= 32 ? 0 : static_cast<int32_t>(static_cast<uint32_t>(x) << s);
}
__device__ __forceinline__ int32_t mulw(int32_t a, int32_t b) {
  return static_cast<int32_t>(static_cast<uint32_t>(a) * static_cast<uint32_t>(b));
}
__device__ __forceinline__ bool mul_ovf32(int32_t a, int32_t b) {
  const long long p = static_cast<long long>(a) * b;
  return p != static_cast<int32_t>(p);
}
__device__ __forceinline__ bool add_ovf32(int32_t a, int32_t b) {
  const long long p = static_cast<long long>(a) + b;
  return p != static_cast<int32_t>(p);
}
__device__ __forceinline__ bool sub_ovf32(int32_t a, int32_t b) {
  const long long p = static_cast<long long>(a) - b;
  return p != static_cast<int32_t>(p);
}
__device__ __forceinline__ bool shl_ovf32(int32_t x, int s) { return asr32(shl32(x, s), s) != x; }
// truncating quotient of 32-bit words: exact in FP64 (|num|, |den| < 2^31 keep
// every non-integer quotient > 2^-32 relative away from an integer)
__device__ __forceinline__ int32_t div32(int32_t num, int32_t den) {
  if (num == INT32_MIN && den == -1) return num;
  return static_cast<int32_t>(trunc(__ddiv_rn(static_cast<double>(num), static_cast<double>(den))));
}

// overflow counters of a cycle: [step][kernel][op] as in kernels.cu
struct Ev32 {
  u64* cnt;
  bool on;
  __device__ void hit(int k, int op, u64 v = 1) {
    if (on && v) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + k * OP_COUNT + op), v);
  }
};

__device__ int32_t fx_mul32(int32_t a, int32_t b, int b1, int b2, int post, Ev32& ev, int k) {
  const int32_t x = asr32(a, b1), y = asr32(b, b2);
  if (mul_ovf32(x, y)) ev.hit(k, OP_MUL);
  return asr32(mulw(x, y), post);
}
__device__ bool fx_div32(int32_t a, int32_t b, int f, int b1, int b2, int32_t* out, Ev32& ev, int k) {
  if (shl_ovf32(a, b1)) ev.hit(k, OP_SHL);
  const int32_t num = shl32(a, b1);
  const int32_t den = asr32(b, b2);
  if (den == 0) return false;
  if (num == INT32_MIN && den == -1) ev.hit(k, OP_DIV);
  const int32_t q = div32(num, den);
  const int e = f - b1 - b2;
  if (e >= 0) {
    if (shl_ovf32(q, e)) ev.hit(k, OP_SHL);
    *out = shl32(q, e);
  } else {
    *out = asr32(q, -e);
  }
  return true;
}
__device__ uint32_t isqrt32(uint32_t v) {
  if (v == 0) return 0;
  unsigned long long x = static_cast<unsigned long long>(sqrt(static_cast<double>(v)));
  while (x * x > v) --x;
  while ((x + 1) * (x + 1) <= v) ++x;
  return static_cast<uint32_t>(x);
}
__device__ int32_t fx_sqrt32(int32_t a, int fin, int f, Ev32& ev, int k) {  // a >= 0 (fxp.cpp:35-47)
  const int32_t r = static_cast<int32_t>(isqrt32(static_cast<uint32_t>(a)));
  const int e = f - fin / 2;
  if (e >= 0) {
    if (shl_ovf32(r, e)) ev.hit(k, OP_SHL);
    return shl32(r, e);
  }
  return asr32(r, -e);
}
__device__ void set_err32(Ctl* ctl, int code, int msg, int step) {
  if (atomicCAS(&ctl->err, 0, code) == 0) {
    ctl->err_msg = msg;
    ctl->err_step = step;
  }
}

constexpr int kT = 256;

__global__ void __launch_bounds__(kT) k32_encode(long long n, const double* __restrict__ r0, int32_t* __restrict__ v0,
                                                 int f, Ctl* ctl) {
  if (over32(ctl)) return;
  const double r0n = ctl->r0n;
  const double lim = ldexp(1.0, 31 - f), up = ldexp(1.0, f);
  bool bad = false;
  for (long long i = blockIdx.x * static_cast<long long>(kT) + threadIdx.x; i < n; i += static_cast<long long>(gridDim.x) * kT) {
    const double x = __ddiv_rn(r0[i], r0n);
    if (!(fabs(x) < lim)) {
      bad = true;
      v0[i] = 0;
    } else {
      v0[i] = static_cast<int32_t>(__double2ll_rz(__dmul_rn(x, up)));
    }
  }
  if (bad) set_err32(ctl, IGM_OVERFLOW_ERROR, EM_ENCODE, -1);
}

// split.cpp:137-157 at WL = 32: per component a wrapping row sum, asr by alpha_l
__global__ void __launch_bounds__(kT) k32_spmv(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                               const int32_t* __restrict__ vals, int nnz, const int* __restrict__ alphas,
                                               int s, const int32_t* __restrict__ v, int32_t* __restrict__ out, u64* cnt,
                                               const Ctl* ctl, int checked) {
  if (over32(ctl)) return;
  u64 nm = 0, na = 0;
  for (int i = blockIdx.x * kT + threadIdx.x; i < n; i += gridDim.x * kT) {
    int32_t o = 0;
    const int k0 = rp[i], k1 = rp[i + 1];
    for (int l = 0; l <= s; ++l) {
      const int32_t* cv = vals + static_cast<long long>(l) * nnz;
      int32_t acc = 0;
      for (int k = k0; k < k1; ++k) {
        const int32_t a = __ldg(cv + k), b = __ldg(v + __ldg(ci + k));
        const int32_t p = mulw(a, b);
        if (checked) {
          nm += mul_ovf32(a, b);
          na += add_ovf32(acc, p);
        }
        acc = static_cast<int32_t>(static_cast<uint32_t>(acc) + static_cast<uint32_t>(p));
      }
      const int32_t t = asr32(acc, __ldg(alphas + l));
      if (checked) na += add_ovf32(o, t);
      o = static_cast<int32_t>(static_cast<uint32_t>(o) + static_cast<uint32_t>(t));
    }
    out[i] = o;
  }
  if (checked) {
    if (nm) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_SPMV * OP_COUNT + OP_MUL), nm);
    if (na) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_SPMV * OP_COUNT + OP_ADD), na);
  }
}

// the same at depth 0 for rows of <= 16 entries: every (value, column) pair of
// the row is loaded before the first gather and every gather before the first
// product (as k_spmv_int_r8 does at WL = 64: the loop above chains a column
// load, a gather and a product per entry); sums stay in CSR order
__global__ void __launch_bounds__(128) k32_spmv_r16(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const int32_t* __restrict__ vals, int alpha0,
                                                    const int32_t* __restrict__ v, int32_t* __restrict__ out, u64* cnt,
                                                    const Ctl* ctl, int checked) {
  if (over32(ctl)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k0 = __ldg(rp + i), len = __ldg(rp + i + 1) - k0;
  int c[16];
  int32_t a[16], x[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    c[u] = u < len ? __ldg(ci + k0 + u) : 0;
    a[u] = u < len ? __ldg(vals + k0 + u) : 0;
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) x[u] = u < len ? __ldg(v + c[u]) : 0;
  u64 nm = 0, na = 0;
  int32_t acc = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    if (u < len) {
      const int32_t p = mulw(a[u], x[u]);
      if (checked) {
        nm += mul_ovf32(a[u], x[u]);
        na += add_ovf32(acc, p);
      }
      acc = static_cast<int32_t>(static_cast<uint32_t>(acc) + static_cast<uint32_t>(p));
    }
  }
  out[i] = asr32(acc, alpha0);  // o = 0 + t: never an add event
  if (checked) {
    if (nm) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_SPMV * OP_COUNT + OP_MUL), nm);
    if (na) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_SPMV * OP_COUNT + OP_ADD), na);
  }
}

// h from a dot accumulator (fxp.cpp:63-65 at WL = 32)
__device__ __forceinline__ int32_t h_of32(uint32_t acc, int e) {
  const int32_t a = static_cast<int32_t>(acc);
  return e >= 0 ? asr32(a, e) : shl32(a, -e);
}

// mode 0: acc_out = sum (w >> b1)(v >> b2)            (fx_dot, fxp.cpp:49-67)
// mode 1: w -= asr((h >> a1) vp, f - a1), then the dot with v (fxp.cpp:88-104)
// mode 2: the axpy with vp, then acc_out = sum (w >> nb1)^2 (fx_norm, fxp.cpp:69-86)
// abs_out: sum |term| (u64): < 2^31 certifies that the sequential running sum
// never wrapped (no add event)
__global__ void __launch_bounds__(kT) k32_pass(long long n, int mode, int32_t* __restrict__ w,
                                               const int32_t* __restrict__ vp, const int32_t* __restrict__ v,
                                               const uint32_t* __restrict__ acc_prev, uint32_t* acc_out, u64* abs_out,
                                               int f, ShiftsD sh, u64* cnt_axpy, u64* cnt_red, const Ctl* ctl,
                                               int checked) {
  __shared__ uint32_t s_acc[kT / 32];
  __shared__ u64 s_abs[kT / 32];
  if (over32(ctl)) return;
  const int e = f - sh.dot_b1 - sh.dot_b2, post = f - sh.axpy_b1;
  const int32_t hs = mode >= 1 ? asr32(h_of32(*acc_prev, e), sh.axpy_b1) : 0;
  uint32_t acc = 0;
  u64 aabs = 0, n1 = 0, n2 = 0, n3 = 0;
  for (long long l = blockIdx.x * static_cast<long long>(kT) + threadIdx.x; l < n; l += static_cast<long long>(gridDim.x) * kT) {
    int32_t wl = w[l];
    if (mode >= 1) {
      const int32_t pv = vp[l];
      const int32_t d = asr32(mulw(hs, pv), post);
      if (checked) {
        n1 += mul_ovf32(hs, pv);
        n2 += sub_ovf32(wl, d);
      }
      wl = static_cast<int32_t>(static_cast<uint32_t>(wl) - static_cast<uint32_t>(d));
      w[l] = wl;
    }
    int32_t a, b;
    if (mode == 2) {
      a = b = asr32(wl, sh.norm_b1);
    } else {
      a = asr32(wl, sh.dot_b1);
      b = asr32(v[l], sh.dot_b2);
    }
    const int32_t t = mulw(a, b);
    if (checked) n3 += mul_ovf32(a, b);
    acc += static_cast<uint32_t>(t);
    aabs += static_cast<u64>(t < 0 ? -static_cast<long long>(t) : static_cast<long long>(t));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    aabs += __shfl_down_sync(0xffffffffu, aabs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_acc[threadIdx.x >> 5] = acc;
    s_abs[threadIdx.x >> 5] = aabs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a2 = 0;
    u64 b2 = 0;
    for (int q = 0; q < kT / 32; ++q) {
      a2 += s_acc[q];
      b2 += s_abs[q];
    }
    atomicAdd(acc_out, a2);
    atomicAdd(reinterpret_cast<unsigned long long*>(abs_out), b2);
  }
  if (checked) {
    if (n1) atomicAdd(reinterpret_cast<unsigned long long*>(cnt_axpy + OP_MUL), n1);
    if (n2) atomicAdd(reinterpret_cast<unsigned long long*>(cnt_axpy + OP_SUB), n2);
    if (n3) atomicAdd(reinterpret_cast<unsigned long long*>(cnt_red + OP_MUL), n3);
  }
}

// the scalar step (gmres_int.cpp:96-158 at WL = 32), one thread
__global__ void k32_step(int j, int f, ShiftsD sh, const uint32_t* __restrict__ accj, const u64* __restrict__ absj,
                         const uint32_t* __restrict__ nacc, const u64* __restrict__ nabs, int32_t* hess, int ld,
                         int32_t* g, int32_t* cs, int32_t* sn, const int32_t* w, u64* cnt_step, Ctl* ctl, int checked) {
  ctl->do_vecdiv = 0;
  if (over32(ctl)) return;
  Ev32 ev{cnt_step, checked != 0};
  int32_t* col = hess + static_cast<long long>(j) * ld;
  const int e = f - sh.dot_b1 - sh.dot_b2;
  for (int i = 0; i <= j; ++i) {
    const int32_t a = static_cast<int32_t>(accj[i]);
    if (e >= 0) {
      col[i] = asr32(a, e);
    } else {
      if (shl_ovf32(a, -e)) ev.hit(K_DOT, OP_SHL);
      col[i] = shl32(a, -e);
    }
    if (checked && absj[i] >= (1ull << 31)) ctl->add_inexact = 1;  // a running sum may have wrapped
  }
  const int32_t nsum = static_cast<int32_t>(*nacc);
  if (checked && *nabs >= (1ull << 31)) ctl->add_inexact = 1;
  if (nsum < 0) {
    set_err32(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
    return;
  }
  const int32_t hnext = fx_sqrt32(nsum, 2 * (f - sh.norm_b1), f, ev, K_NORM);
  col[j + 1] = hnext;
  const bool happy = hnext == 0;
  if (!happy) {
    const int32_t den = asr32(hnext, sh.div_b2);
    if (den == 0) {
      if (shl_ovf32(w[0], sh.div_b1)) ev.hit(K_VEC_DIV, OP_SHL);
      set_err32(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
      return;
    }
    ctl->div_m = static_cast<u64>(static_cast<uint32_t>(den));  // the vec_div divisor (low word)
    ctl->do_vecdiv = 1;
    ctl->nbasis = j + 2;
  }
  for (int i = 0; i < j; ++i) {  // apply_stored_rotations (gmres_int.cpp:8-25)
    const int32_t c = cs[i], s = sn[i], hi = col[i], hn = col[i + 1];
    const int pg = f - sh.givens_b2;
    const int32_t a = fx_mul32(c, hi, 0, sh.givens_b2, pg, ev, K_GIVENS);
    const int32_t b = fx_mul32(s, hn, 0, sh.givens_b2, pg, ev, K_GIVENS);
    const int32_t d = fx_mul32(c, hn, 0, sh.givens_b2, pg, ev, K_GIVENS);
    const int32_t q = fx_mul32(s, hi, 0, sh.givens_b2, pg, ev, K_GIVENS);
    if (add_ovf32(a, b)) ev.hit(K_GIVENS, OP_ADD);
    if (sub_ovf32(d, q)) ev.hit(K_GIVENS, OP_SUB);
    col[i] = static_cast<int32_t>(static_cast<uint32_t>(a) + static_cast<uint32_t>(b));
    col[i + 1] = static_cast<int32_t>(static_cast<uint32_t>(d) - static_cast<uint32_t>(q));
  }
  int32_t tmp;
  {  // t_mp = fx_norm((h_jj, h_{j+1,j})) (gmres_int.cpp:133-137)
    const int32_t s0 = asr32(col[j], sh.norm_b1), s1 = asr32(col[j + 1], sh.norm_b1);
    if (mul_ovf32(s0, s0)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const int32_t p0 = mulw(s0, s0);
    if (mul_ovf32(s1, s1)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const int32_t p1 = mulw(s1, s1);
    if (add_ovf32(p0, p1)) ev.hit(K_GIVENS_NORM, OP_ADD);
    const int32_t acc = static_cast<int32_t>(static_cast<uint32_t>(p0) + static_cast<uint32_t>(p1));
    if (acc < 0) {
      set_err32(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
      return;
    }
    tmp = fx_sqrt32(acc, 2 * (f - sh.norm_b1), f, ev, K_GIVENS_NORM);
  }
  if (tmp == 0) {
    ctl->stop = 1;
    return;
  }
  int32_t c, s;
  if (!fx_div32(col[j], tmp, f, sh.div_b1, sh.div_b2, &c, ev, K_GIVENS_DIV) ||
      !fx_div32(col[j + 1], tmp, f, sh.div_b1, sh.div_b2, &s, ev, K_GIVENS_DIV)) {
    set_err32(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
    return;
  }
  cs[j] = c;
  sn[j] = s;
  col[j] = tmp;
  col[j + 1] = 0;
  const int32_t g_old = g[j];  // gmres_int.cpp:150-153
  if (sub_ovf32(0, s)) ev.hit(K_ROT, OP_SUB);
  const int32_t neg_s = static_cast<int32_t>(0u - static_cast<uint32_t>(s));
  const int pr = f - 2 * sh.rot_b;
  g[j + 1] = fx_mul32(neg_s, g_old, sh.rot_b, sh.rot_b, pr, ev, K_ROT);
  g[j] = fx_mul32(c, g_old, sh.rot_b, sh.rot_b, pr, ev, K_ROT);
  ctl->dim = j + 1;
  if (happy) ctl->stop = 1;
}

__global__ void __launch_bounds__(kT) k32_vecdiv(long long n, const int32_t* __restrict__ w, int32_t* __restrict__ out,
                                                 int f, ShiftsD sh, u64* cnt, const Ctl* ctl, int checked) {
  if (over32(ctl) || !ctl->do_vecdiv) return;
  const int32_t den = static_cast<int32_t>(static_cast<uint32_t>(ctl->div_m));
  const double dd = static_cast<double>(den);
  const int b1 = sh.div_b1, e = f - sh.div_b1 - sh.div_b2;
  u64 nshl = 0, ndiv = 0;
  for (long long l = blockIdx.x * static_cast<long long>(kT) + threadIdx.x; l < n; l += static_cast<long long>(gridDim.x) * kT) {
    const int32_t a = w[l];
    const int32_t num = shl32(a, b1);
    int32_t q;
    if (num == INT32_MIN && den == -1) {
      q = num;
      ++ndiv;
    } else {
      q = static_cast<int32_t>(trunc(__ddiv_rn(static_cast<double>(num), dd)));
    }
    if (checked) nshl += shl_ovf32(a, b1);
    if (e >= 0) {
      if (checked) nshl += shl_ovf32(q, e);
      out[l] = shl32(q, e);
    } else {
      out[l] = asr32(q, -e);
    }
  }
  if (checked) {
    if (nshl) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_VEC_DIV * OP_COUNT + OP_SHL), nshl);
    if (ndiv) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + K_VEC_DIV * OP_COUNT + OP_DIV), ndiv);
  }
}

// gmres_int.cpp:163-175: decode R and g, back substitution, weights r0n * y_j
__global__ void k32_finish(int m, int f, const int32_t* hess, const int32_t* g, double* y, double* wts, Ctl* ctl) {
  if (ctl->err) return;
  const int dim = ctl->dim;
  if (dim == 0) return;
  const int ld = m + 1;
  const double sc = ldexp(1.0, -f);
  for (int i = dim - 1; i >= 0; --i) {
    double acc = __dmul_rn(static_cast<double>(g[i]), sc);
    for (int jj = i + 1; jj < dim; ++jj)
      acc = __dsub_rn(acc, __dmul_rn(__dmul_rn(static_cast<double>(hess[static_cast<long long>(jj) * ld + i]), sc), y[jj]));
    const double rii = __dmul_rn(static_cast<double>(hess[static_cast<long long>(i) * ld + i]), sc);
    if (rii == 0.0) {
      set_err32(ctl, IGM_RUNTIME_ERROR, EM_HESS_ZERO, -2);
      return;
    }
    y[i] = __ddiv_rn(acc, rii);
  }
  for (int jj = 0; jj < dim; ++jj) wts[jj] = __dmul_rn(ctl->r0n, y[jj]);
}

// x update (gmres_int.cpp:176-179, refine.cpp:87): mode 0 x = sum (run_cycle from
// x0 = 0); mode 1 x += gamma * (0.0 + sum)
__global__ void __launch_bounds__(kT) k32_xupdate(long long n, int f, const int32_t* __restrict__ basis,
                                                  const double* __restrict__ wts, double* __restrict__ x,
                                                  const Ctl* ctl, int mode) {
  if (ctl->err) return;
  const int dim = ctl->dim;
  if (mode == 1 && dim == 0) return;
  const double sc = ldexp(1.0, -f);
  const double gamma = __longlong_as_double(static_cast<long long>(ctl->rmax_bits));
  for (long long l = blockIdx.x * static_cast<long long>(kT) + threadIdx.x; l < n; l += static_cast<long long>(gridDim.x) * kT) {
    double acc = 0.0;
    for (int jj = 0; jj < dim; ++jj)
      acc = __dadd_rn(acc, __dmul_rn(wts[jj], __dmul_rn(static_cast<double>(basis[static_cast<long long>(jj) * n + l]), sc)));
    x[l] = mode == 0 ? acc : __dadd_rn(x[l], __dmul_rn(gamma, acc));
  }
}

__global__ void __launch_bounds__(kT) k32_narrow(long long cnt, const i64* __restrict__ in, int32_t* __restrict__ out,
                                                 int* bad) {
  for (long long q = blockIdx.x * static_cast<long long>(kT) + threadIdx.x; q < cnt; q += static_cast<long long>(gridDim.x) * kT) {
    const i64 v = in[q];
    if (v != static_cast<int32_t>(v)) *bad = 1;
    out[q] = static_cast<int32_t>(v);
  }
}

__global__ void k32_init(Ctl* ctl, int32_t* g, int f) {
  ctl->stop = 0;
  ctl->dim = 0;
  ctl->nbasis = 1;
  ctl->do_vecdiv = 0;
  ctl->add_inexact = 0;
  g[0] = static_cast<int32_t>(1) << f;
}

int grid32(long long n) {
  const long long b = (n + kT - 1) / kT;
  const long long cap = 8LL * num_sms(cur_device());
  return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

// the split's int64 component values as int32 (*bad = 1 if one does not fit)
void launch_vals_to32(cudaStream_t st, long long cnt, const i64* in, int32_t* out, int* bad) {
  k32_narrow<<<grid32(cnt), kT, 0, st>>>(cnt, in, out, bad);
}

// One cycle at WL = 32 (gmres_int.cpp:42-196, unpreconditioned), enqueued on st.
// r0: the cycle's right-hand side in FP64 (device); ctl->r0n holds its norm
// (launch_norm2_serial mode 3 before this).  Buffers: see Wl32Work.
static void enqueue_cycle32_launches(cudaStream_t st, const Wl32Work& b, const Dev32Split& m, int M, int f, int s,
                                     ShiftsD sh, const double* r0, Ctl* ctl, bool checked, int xmode, double* x);

// The cycle is ~M^2 / 2 short launches (1525 at M = 50) over vectors that sit
// in the L2: launch-bound.  The sequence and every argument are fixed for a
// given (buffers, M, shifts, ...), so it is captured once into a CUDA graph
// and replayed per cycle (IGM_WL32_GRAPH=0: plain launches).
namespace {
struct Cyc32Key {
  const void *small, *basis, *vals, *rp, *r0, *ctl, *x;
  long long n;
  int M, f, s, checked, xmode, max_row;
  ShiftsD sh;
  bool operator==(const Cyc32Key& o) const { return std::memcmp(this, &o, sizeof(Cyc32Key)) == 0; }
};
struct Cyc32Graph {
  Cyc32Key key;
  cudaGraphExec_t exec = nullptr;
};
}  // namespace

void enqueue_cycle32(cudaStream_t st, const Wl32Work& b, const Dev32Split& m, int M, int f, int s, ShiftsD sh,
                     const double* r0, Ctl* ctl, bool checked, int xmode, double* x) {
  static const bool use_graph = [] {
    const char* e = std::getenv("IGM_WL32_GRAPH");
    return !(e && e[0] == '0');
  }();
  if (!use_graph) {
    enqueue_cycle32_launches(st, b, m, M, f, s, sh, r0, ctl, checked, xmode, x);
    return;
  }
  Cyc32Key key;
  std::memset(&key, 0, sizeof(key));  // (padding bytes take part in the comparison)
  key.small = b.small;
  key.basis = b.basis;
  key.vals = m.vals;
  key.rp = m.row_ptr;
  key.r0 = r0;
  key.ctl = ctl;
  key.x = x;
  key.n = m.n;
  key.M = M;
  key.f = f;
  key.s = s;
  key.checked = checked ? 1 : 0;
  key.xmode = xmode;
  key.max_row = m.max_row;
  key.sh = sh;
  thread_local Cyc32Graph cache;  // one context (stream) per host thread drives a cycle at a time
  if (cache.exec == nullptr || !(cache.key == key)) {
    if (cache.exec) {
      cudaGraphExecDestroy(cache.exec);
      cache.exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      enqueue_cycle32_launches(st, b, m, M, f, s, sh, r0, ctl, checked, xmode, x);
      if (cudaStreamEndCapture(st, &g) == cudaSuccess && g != nullptr &&
          cudaGraphInstantiate(&cache.exec, g, 0) == cudaSuccess) {
        cache.key = key;
      } else {
        cache.exec = nullptr;
      }
      if (g) cudaGraphDestroy(g);
    }
    if (cache.exec == nullptr) {  // capture unavailable: plain launches
      cudaGetLastError();
      enqueue_cycle32_launches(st, b, m, M, f, s, sh, r0, ctl, checked, xmode, x);
      return;
    }
  }
  if (cudaGraphLaunch(cache.exec, st) != cudaSuccess) {
    cudaGetLastError();
    enqueue_cycle32_launches(st, b, m, M, f, s, sh, r0, ctl, checked, xmode, x);
  }
}

static void enqueue_cycle32_launches(cudaStream_t st, const Wl32Work& b, const Dev32Split& m, int M, int f, int s,
                                     ShiftsD sh, const double* r0, Ctl* ctl, bool checked, int xmode, double* x) {
  const long long n = m.n;
  const int ld = M + 1;
  const int gr = grid32(n);
  k32_init<<<1, 1, 0, st>>>(ctl, b.g, f);
  k32_encode<<<gr, kT, 0, st>>>(n, r0, b.basis, f, ctl);
  const size_t cstride = static_cast<size_t>(K_COUNT) * OP_COUNT;
  for (int j = 0; j < M; ++j) {
    u64* cstep = b.cnt + static_cast<size_t>(j) * cstride;
    const int32_t* vj = b.basis + static_cast<long long>(j) * n;
    if (s == 0 && m.max_row > 0 && m.max_row <= 16 && !m.h_alphas.empty())
      k32_spmv_r16<<<(m.n + 127) / 128, 128, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.h_alphas[0], vj, b.w, cstep,
                                                      ctl, checked ? 1 : 0);
    else
      k32_spmv<<<grid32(n), kT, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, vj, b.w, cstep, ctl,
                                          checked ? 1 : 0);
    uint32_t* accj = b.acc + static_cast<size_t>(j) * (M + 1);
    u64* absj = b.abs + static_cast<size_t>(j) * (M + 1);
    for (int i = 0; i <= j; ++i) {
      const int32_t* vi = b.basis + static_cast<long long>(i) * n;
      const int32_t* vp = i > 0 ? b.basis + static_cast<long long>(i - 1) * n : nullptr;
      k32_pass<<<gr, kT, 0, st>>>(n, i == 0 ? 0 : 1, b.w, vp, vi, i > 0 ? accj + (i - 1) : nullptr, accj + i,
                                  absj + i, f, sh, cstep + K_AXPY * OP_COUNT, cstep + K_DOT * OP_COUNT, ctl,
                                  checked ? 1 : 0);
    }
    k32_pass<<<gr, kT, 0, st>>>(n, 2, b.w, vj, nullptr, accj + j, b.nacc + j, b.nabs + j, f, sh,
                                cstep + K_AXPY * OP_COUNT, cstep + K_NORM * OP_COUNT, ctl, checked ? 1 : 0);
    k32_step<<<1, 1, 0, st>>>(j, f, sh, accj, absj, b.nacc + j, b.nabs + j, b.hess, ld, b.g, b.cs, b.sn, b.w, cstep,
                              ctl, checked ? 1 : 0);
    k32_vecdiv<<<gr, kT, 0, st>>>(n, b.w, b.basis + static_cast<long long>(j + 1) * n, f, sh, cstep, ctl,
                                  checked ? 1 : 0);
  }
  k32_finish<<<1, 1, 0, st>>>(M, f, b.hess, b.g, b.y, b.wts, ctl);
  k32_xupdate<<<gr, kT, 0, st>>>(n, f, b.basis, b.wts, x, ctl, xmode);
}

}  // namespace igm
