// kernels.cu -- sm_100a kernels of the int-GMRES hot path.
//
// Every kernel here is bit-exact against the reference semantics (SURVEY.md
// Appendix A): integer kernels wrap mod 2^64 and reduce with order-free
// wrapping sums; FP64 kernels use explicit _rn intrinsics (no contraction),
// one thread per row in CSR order, and a single sequential chain for norm2.
// Kernels that belong to a cycle read the Ctl block first and exit when the
// cycle has already ended (break / error), so a whole cycle is enqueued
// without host round trips.
#include "igm_internal.cuh"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>
#include <cstdio>
#include <vector>

namespace igm {

unsigned long long g_launches = 0;

namespace {
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_pool;
cudaEvent_t prof_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void prof_enable(bool on) { g_prof_on = on; }

ProfScope::ProfScope(cudaStream_t s, int c) : st(s), cls(c) {
  if (!g_prof_on) return;
  ProfRec r{c, prof_event(), prof_event()};
  cudaEventRecord(r.a, s);
  g_prof.push_back(r);
}

ProfScope::~ProfScope() {
  if (!g_prof_on || g_prof.empty()) return;
  cudaEventRecord(g_prof.back().b, st);
}

void prof_collect(double* ms, unsigned long long* count) {
  for (int i = 0; i < KC_COUNT; ++i) {
    ms[i] = 0.0;
    count[i] = 0;
  }
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[r.cls] += t;
    count[r.cls] += 1;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_prof.clear();
}

int num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v > 0 ? v : 148;
  }
  return cached[device];
}

namespace {

__device__ __forceinline__ bool cycle_over(const Ctl* c) {
  return c != nullptr && (c->stop | c->err) != 0;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_max(int* p, int v) {
  asm volatile("red.release.gpu.global.max.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double dec(i64 raw, double scale) {
  return __dmul_rn(__ll2double_rn(raw), scale);  // exact power-of-two scale
}

// wrapping block sum of a u64 (any order: Z/2^64 is commutative)
template <int NT>
__device__ __forceinline__ u64 block_sum(u64 v, u64* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  u64 r = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ void bump(u64* cnt, int op, u64 v) {
  if (v) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + op), static_cast<unsigned long long>(v));
}

inline int grid_for(long long n, int nt, int device = 0) {
  long long g = (n + nt - 1) / nt;
  const long long cap = static_cast<long long>(num_sms(device)) * 8;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// K1 integer SpMV (split.cpp:137-157): one thread per row, CSR order, all
// components 0..s per row; exact per-row overflow accounting.
template <bool CHECKED>
__global__ void __launch_bounds__(256) k_spmv_int(int n, const int* __restrict__ rp,
                                                  const int* __restrict__ ci,
                                                  const i64* __restrict__ vals, long long nnz,
                                                  const int* __restrict__ alphas, int s,
                                                  const i64* __restrict__ v, i64* __restrict__ out,
                                                  u64* cnt, const Ctl* ctl) {
  if (cycle_over(ctl)) return;
  u64 nmul = 0, nadd = 0;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < n; row += gridDim.x * blockDim.x) {
    const int b = rp[row], e = rp[row + 1];
    i64 o = 0;
    for (int l = 0; l <= s; ++l) {
      const i64* cv = vals + static_cast<long long>(l) * nnz;
      i64 acc = 0;
      for (int k = b; k < e; ++k) {
        const i64 a = cv[k];
        const i64 x = __ldg(v + ci[k]);
        const i64 p = wmul(a, x);
        if (CHECKED) {
          nmul += mul_ovf(a, x);
          nadd += add_ovf(acc, p);
        }
        acc = wadd(acc, p);
      }
      const i64 d = asr(acc, alphas[l]);
      if (CHECKED) nadd += add_ovf(o, d);
      o = wadd(o, d);
    }
    out[row] = o;
  }
  if (CHECKED) {
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_ADD, nadd);
  }
}

// spmv_fp(SplitMatrix) (split.cpp:159-175) fused with r0 = b - A x0
// (gmres_int.cpp:63-68); if b == nullptr, y = A x.
__global__ void __launch_bounds__(256) k_spmv_fp_split(int n, const int* __restrict__ rp,
                                                       const int* __restrict__ ci,
                                                       const i64* __restrict__ vals, long long nnz,
                                                       const int* __restrict__ alphas, int s,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ y, const Ctl* ctl) {
  if (cycle_over(ctl)) return;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < n; row += gridDim.x * blockDim.x) {
    const int rb = rp[row], re = rp[row + 1];
    double o = 0.0;
    for (int l = 0; l <= s; ++l) {
      const i64* cv = vals + static_cast<long long>(l) * nnz;
      const double scale = ldexp(1.0, -alphas[l]);
      double acc = 0.0;
      for (int k = rb; k < re; ++k)
        acc = __dadd_rn(acc, __dmul_rn(__ll2double_rn(cv[k]), x[ci[k]]));
      o = __dadd_rn(o, __dmul_rn(scale, acc));
    }
    y[row] = b ? __dsub_rn(b[row], o) : o;
  }
}

// K7 residual (split.cpp:37-59 + refine.cpp:53-56): r = b - A_fp x, one
// thread per row in CSR order from 0.0; tracks max|r| as IEEE bits.
__global__ void __launch_bounds__(256) k_residual(int n, const int* __restrict__ rp,
                                                  const int* __restrict__ ci,
                                                  const double* __restrict__ vals,
                                                  const double* __restrict__ x,
                                                  const double* __restrict__ b,
                                                  double* __restrict__ r, Ctl* ctl, int track) {
  u64 mx = 0;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < n; row += gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int e = rp[row + 1];
    for (int k = rp[row]; k < e; ++k) acc = __dadd_rn(acc, __dmul_rn(vals[k], x[ci[k]]));
    const double rr = b ? __dsub_rn(b[row], acc) : acc;
    r[row] = rr;
    const u64 bits = static_cast<u64>(__double_as_longlong(fabs(rr)));
    mx = bits > mx ? bits : mx;
  }
  if (track) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 t = __shfl_down_sync(0xffffffffu, mx, o);
      mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx)
      atomicMax(reinterpret_cast<unsigned long long*>(&ctl->rmax_bits), static_cast<unsigned long long>(mx));
  }
}

__global__ void k_gamma(long long n, const double* __restrict__ r, Ctl* ctl) {
  u64 mx = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const u64 bits = static_cast<u64>(__double_as_longlong(fabs(r[i])));
    mx = bits > mx ? bits : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 t = __shfl_down_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx)
    atomicMax(reinterpret_cast<unsigned long long*>(&ctl->rmax_bits), static_cast<unsigned long long>(mx));
}

// b_k = r / gamma (refine.cpp:17-18), gamma = max|r| from Ctl.
__global__ void k_scale_div(long long n, const double* __restrict__ r, double* __restrict__ out,
                            const Ctl* ctl) {
  if (cycle_over(ctl)) return;
  const double g = __longlong_as_double(static_cast<long long>(ctl->rmax_bits));
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = __ddiv_rn(r[i], g);
}

// ---------------------------------------------------------------------------
// K8 norm2 (split.cpp:45-49): ONE sequential chain acc = fl(acc + fl(x*x)).
// Warps 1..7 square the next tile into shared memory while thread 0 of
// warp 0 runs the dependent FP64 add chain over the current tile.
// mode: 0 -> *out = sqrt; 1 -> ctl->nb; 2 -> ctl->nr and ctl->relnorm;
//       3 -> ctl->r0n (stop the cycle when zero); 4 -> out[0] (decode raw
//       basis words first: collect_basis_norms).
constexpr int kNormTile = 2048;

__global__ void __launch_bounds__(256) k_norm2_serial(long long n, const double* __restrict__ v,
                                                      const i64* __restrict__ raw, double scale,
                                                      double* out, Ctl* ctl, int mode,
                                                      int basis_idx) {
  __shared__ double buf[2][kNormTile];
  if (mode == 3 && cycle_over(ctl)) return;
  if (mode == 4 && (ctl->err || basis_idx >= ctl->nbasis)) return;
  double acc = 0.0;
  const long long ntiles = (n + kNormTile - 1) / kNormTile;
  for (long long t = 0; t < ntiles; ++t) {
    double* b = buf[t & 1];
    const long long base = t * kNormTile;
    const int cnt = static_cast<int>(min(static_cast<long long>(kNormTile), n - base));
    if (threadIdx.x >= 32) {
      for (int q = threadIdx.x - 32; q < cnt; q += blockDim.x - 32) {
        const double x = raw ? dec(raw[base + q], scale) : v[base + q];
        b[q] = __dmul_rn(x, x);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int q = 0;
      for (; q + 8 <= cnt; q += 8) {
        const double a0 = b[q], a1 = b[q + 1], a2 = b[q + 2], a3 = b[q + 3];
        const double a4 = b[q + 4], a5 = b[q + 5], a6 = b[q + 6], a7 = b[q + 7];
        acc = __dadd_rn(acc, a0); acc = __dadd_rn(acc, a1);
        acc = __dadd_rn(acc, a2); acc = __dadd_rn(acc, a3);
        acc = __dadd_rn(acc, a4); acc = __dadd_rn(acc, a5);
        acc = __dadd_rn(acc, a6); acc = __dadd_rn(acc, a7);
      }
      for (; q < cnt; ++q) acc = __dadd_rn(acc, b[q]);
    }
  }
  if (threadIdx.x == 0) {
    const double r = __dsqrt_rn(acc);
    switch (mode) {
      case 0: *out = r; break;
      case 1: ctl->nb = r; break;
      case 2:
        ctl->nr = r;
        ctl->relnorm = ctl->nb == 0.0 ? r : __ddiv_rn(r, ctl->nb);
        break;
      case 3:
        ctl->r0n = r;
        if (r == 0.0) ctl->stop = 1;
        break;
      case 4: out[basis_idx] = r; break;
    }
  }
}

// K8' norm2, exact parallel form of the same sequential chain.
//
// Inside one binade [2^E, 2^{E+1}) of the running sum the ulp u = 2^{E-52} is
// fixed, the sum is M*u with M < 2^53, and fl(M*u + q) = u * rne(M + q/u)
// (round to nearest, ties to even) as long as M + q/u < 2^53 - 1/2.  Each
// term therefore adds an integer d = floor(q/u) (+1 above half, and at an
// exact half +1 iff M + floor(q/u) is odd).  Only ties depend on the running
// value, and only through its parity: every term is a function of one bit,
// and a chunk composes as a 2-state automaton (total increment for an even
// / odd start), so a block-wide scan gives every prefix.  The first term
// whose exact sum would leave the binade (or a non-finite term) is replayed
// with the real FP64 add, the binade is re-read from the result, and the scan
// resumes after it.  The result is bit-identical to the serial chain
// (split.cpp:45-49) by construction; the serial kernel above stays as the
// fallback for non-finite data.
constexpr int kN2Threads = 1024;
constexpr int kN2Per = 8;
constexpr int kN2Chunk = kN2Threads * kN2Per;
constexpr u64 kTwo53 = 1ull << 53;

struct Aut {  // increments for an even / odd incoming parity
  u64 d0, d1;
};

__device__ __forceinline__ Aut aut_then(const Aut& f, const Aut& g) {
  Aut h;
  h.d0 = f.d0 + ((f.d0 & 1) ? g.d1 : g.d0);
  h.d1 = f.d1 + (((f.d1 + 1) & 1) ? g.d1 : g.d0);
  return h;
}

enum { N2_DOWN = 0, N2_UP = 1, N2_TIE = 2, N2_EXIT = 3 };

// q = mq * 2^fq; u = 2^(E-52): floor(q/u) and the class of the remainder
__device__ __forceinline__ int n2_classify(double q, int E, u64& a) {
  const u64 bits = static_cast<u64>(__double_as_longlong(q));
  const int ex = static_cast<int>((bits >> 52) & 0x7ff);
  u64 mq = bits & ((1ull << 52) - 1);
  a = 0;
  if (ex == 0x7ff) return N2_EXIT;
  int fq;
  if (ex == 0) {
    fq = -1074;
  } else {
    mq |= 1ull << 52;
    fq = ex - 1075;
  }
  if (mq == 0) return N2_DOWN;
  const int sh = (E - 52) - fq;
  if (sh < 0) return N2_EXIT;  // q >= 2u * 2^52: leaves the binade
  if (sh == 0) {
    a = mq;
    return N2_DOWN;
  }
  if (sh >= 64) return N2_DOWN;
  a = mq >> sh;
  const u64 rem = mq & ((1ull << sh) - 1), half = 1ull << (sh - 1);
  return rem < half ? N2_DOWN : (rem == half ? N2_TIE : N2_UP);
}

__device__ __forceinline__ u64 n2_inc(u64 a, int cls, u64 parity) {
  return cls == N2_DOWN ? a : (cls == N2_UP ? a + 1 : a + ((parity + a) & 1));
}

__global__ void __launch_bounds__(kN2Threads) k_norm2_exact(long long n, const double* __restrict__ v,
                                                            const i64* __restrict__ raw, double scale,
                                                            double* out, Ctl* ctl, int mode,
                                                            int basis_idx) {
  __shared__ Aut s_warp[32];
  __shared__ int s_exit;
  __shared__ u64 s_mprev;
  __shared__ int s_E;
  __shared__ u64 s_M;
  __shared__ long long s_pos;
  __shared__ int s_tail;
  __shared__ double s_tailv;
  if (mode == 3 && cycle_over(ctl)) return;
  if (mode == 4 && (ctl->err || basis_idx >= ctl->nbasis)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    s_E = -1022;  // s = 0: subnormal binade, u = 2^-1074
    s_M = 0;
    s_pos = 0;
    s_tail = 0;
  }
  __syncthreads();
  while (true) {
    const long long pos = s_pos;
    const int E = s_E;
    const u64 M0 = s_M;
    if (pos >= n || s_tail) break;
    const long long base = pos + static_cast<long long>(tid) * kN2Per;
    u64 a[kN2Per];
    int cls[kN2Per];
    Aut mine{0, 0};
#pragma unroll
    for (int g = 0; g < kN2Per; ++g) {
      const long long idx = base + g;
      if (idx < n && idx < pos + kN2Chunk) {
        const double x = raw ? dec(raw[idx], scale) : v[idx];
        cls[g] = n2_classify(__dmul_rn(x, x), E, a[g]);
      } else {
        cls[g] = N2_DOWN;
        a[g] = 0;
      }
      Aut e;
      e.d0 = n2_inc(a[g], cls[g] == N2_EXIT ? N2_DOWN : cls[g], 0);
      e.d1 = n2_inc(a[g], cls[g] == N2_EXIT ? N2_DOWN : cls[g], 1);
      mine = aut_then(mine, e);
    }
    // exclusive block scan of the automata (sequence order = thread order)
    Aut inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Aut up;
      up.d0 = __shfl_up_sync(0xffffffffu, inc.d0, o);
      up.d1 = __shfl_up_sync(0xffffffffu, inc.d1, o);
      if (lane >= o) inc = aut_then(up, inc);
    }
    if (lane == 31) s_warp[wid] = inc;
    if (tid == 0) s_exit = INT_MAX;
    __syncthreads();
    if (wid == 0) {
      Aut w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        Aut up;
        up.d0 = __shfl_up_sync(0xffffffffu, w.d0, o);
        up.d1 = __shfl_up_sync(0xffffffffu, w.d1, o);
        if (lane >= o) w = aut_then(up, w);
      }
      s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    Aut ex{0, 0};
    if (wid > 0) ex = s_warp[wid - 1];
    {
      Aut lx;
      lx.d0 = __shfl_up_sync(0xffffffffu, inc.d0, 1);
      lx.d1 = __shfl_up_sync(0xffffffffu, inc.d1, 1);
      if (lane > 0) ex = aut_then(ex, lx);
    }
    const Aut total = s_warp[31];
    // walk this thread's terms from the true incoming value; first exit
    u64 Mp = M0 + ((M0 & 1) ? ex.d1 : ex.d0);
    int my_exit = INT_MAX;
    u64 my_mprev = 0;
#pragma unroll
    for (int g = 0; g < kN2Per; ++g) {
      if (my_exit != INT_MAX) break;
      const long long idx = base + g;
      if (idx >= n || idx >= pos + kN2Chunk) break;
      const bool leave = cls[g] == N2_EXIT || a[g] >= kTwo53 ||
                         Mp + a[g] + (cls[g] != N2_DOWN ? 1 : 0) >= kTwo53;
      if (leave) {
        my_exit = tid * kN2Per + g;
        my_mprev = Mp;
      } else {
        Mp += n2_inc(a[g], cls[g], Mp & 1);
      }
    }
    if (my_exit != INT_MAX) atomicMin(&s_exit, my_exit);
    __syncthreads();
    const int xe = s_exit;
    if (xe != INT_MAX && my_exit == xe) s_mprev = my_mprev;
    __syncthreads();
    if (tid == 0) {
      if (xe == INT_MAX) {
        s_M = M0 + ((M0 & 1) ? total.d1 : total.d0);
        s_pos = min(n, pos + kN2Chunk);
      } else {
        // replay the term that leaves the binade with the real FP64 add
        const long long idx = pos + xe;
        const double x = raw ? dec(raw[idx], scale) : v[idx];
        const double sp = ldexp(static_cast<double>(s_mprev), E - 52);
        const double sn = __dadd_rn(sp, __dmul_rn(x, x));
        if (!isfinite(sn)) {
          s_tail = 1;
          s_tailv = sn;
          s_pos = idx + 1;
        } else {
          const u64 b = static_cast<u64>(__double_as_longlong(sn));
          const int ebits = static_cast<int>((b >> 52) & 0x7ff);
          const int En = ebits == 0 ? -1022 : max(ebits - 1023, -1022);
          s_E = En;
          s_M = static_cast<u64>(ldexp(sn, 52 - En));
          s_pos = idx + 1;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    double acc;
    if (s_tail) {  // non-finite partial sum: finish the chain serially
      acc = s_tailv;
      for (long long i = s_pos; i < n; ++i) {
        const double x = raw ? dec(raw[i], scale) : v[i];
        acc = __dadd_rn(acc, __dmul_rn(x, x));
      }
    } else {
      acc = ldexp(static_cast<double>(s_M), s_E - 52);
    }
    const double r = __dsqrt_rn(acc);
    switch (mode) {
      case 0: *out = r; break;
      case 1: ctl->nb = r; break;
      case 2:
        ctl->nr = r;
        ctl->relnorm = ctl->nb == 0.0 ? r : __ddiv_rn(r, ctl->nb);
        break;
      case 3:
        ctl->r0n = r;
        if (r == 0.0) ctl->stop = 1;
        break;
      case 4: out[basis_idx] = r; break;
    }
  }
}

// K10 encode v1 = trunc(ldexp(r0_i / ||r0||, f)) (gmres_int.cpp:77-81,
// fxp.hpp:171-176) with the reference's range check.
__global__ void k_encode(long long n, const double* __restrict__ r0, i64* __restrict__ v0, int f,
                         Ctl* ctl) {
  if (cycle_over(ctl)) return;
  const double r0n = ctl->r0n;
  const double lim = ldexp(1.0, 63 - f);
  const double up = ldexp(1.0, f);
  bool bad = false;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = __ddiv_rn(r0[i], r0n);
    if (!(fabs(x) < lim)) {
      bad = true;
      v0[i] = 0;
    } else {
      v0[i] = __double2ll_rz(__dmul_rn(x, up));
    }
  }
  if (bad && atomicCAS(&ctl->err, 0, IGM_OVERFLOW_ERROR) == 0) {
    ctl->err_msg = EM_ENCODE;
    ctl->err_step = -1;
  }
}

// ---------------------------------------------------------------------------
// K2/K3 fused MGS pass (gmres_int.cpp:101-115, fxp.cpp:49-104).
//   MODE 0: dot_i only                     (i == 0)
//   MODE 1: axpy_{i-1} then dot_i          (0 < i <= j)
//   MODE 2: axpy_j then the norm sum       (tail of step j)
//   MODE 3: axpy only                      (tail of the config-5 microbench)
// h_{i-1} is re-derived by every thread from the wrapped accumulator of the
// previous pass (fx_dot's final shift, fxp.cpp:63-65).  Reductions are
// wrapping u64 sums (exact, order-free).  In checked mode per-element mul /
// sub events are counted exactly and sum|term| is accumulated so the
// running-sum ("add") events can be certified zero.
// 256-bit global accesses (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a)
__device__ __forceinline__ void ld_v4(const i64* p, i64 (&v)[4]) {
  asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_v4_nc(const i64* p, i64 (&v)[4]) {
  asm volatile("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void st_v4(i64* p, const i64 (&v)[4]) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]),
               "l"(v[3])
               : "memory");
}

template <int VEC>
__device__ __forceinline__ void ldv(const i64* p, i64 (&v)[VEC]) {
  if constexpr (VEC == 4) {
    ld_v4(p, v);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) v[e] = p[e];
  }
}
template <int VEC>
__device__ __forceinline__ void ldv_nc(const i64* p, i64 (&v)[VEC]) {
  if constexpr (VEC == 4) {
    ld_v4_nc(p, v);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) v[e] = __ldg(p + e);
  }
}
template <int VEC>
__device__ __forceinline__ void stv(i64* p, const i64 (&v)[VEC]) {
  if constexpr (VEC == 4) {
    st_v4(p, v);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) p[e] = v[e];
  }
}

template <int MODE, bool CHECKED, int VEC>
__global__ void __launch_bounds__(512) k_mgs(long long n, i64* __restrict__ w,
                                             const i64* __restrict__ vprev,
                                             const i64* __restrict__ vcur,
                                             const u64* __restrict__ hacc, u64* acc_out,
                                             u64* abs_out, int f, ShiftsD sh, u64* cnt_axpy,
                                             u64* cnt_red, const Ctl* ctl) {
  __shared__ u64 red[3][16];
  if (cycle_over(ctl)) return;
  i64 hs = 0;
  const int post = f - sh.axpy_b1;
  if (MODE != 0) {
    const i64 acc = static_cast<i64>(*hacc);
    const int e = f - sh.dot_b1 - sh.dot_b2;
    const i64 h = e >= 0 ? asr(acc, e) : wrap_shl(acc, -e);
    hs = asr(h, sh.axpy_b1);
  }
  u64 sum = 0, ahi = 0, alo = 0, nmul = 0, nsub = 0, nmul2 = 0;
  const long long ng = n / VEC;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long gi = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; gi < ng; gi += stride) {
    const long long l = gi * VEC;
    i64 wv[VEC], pv[VEC], cv[VEC];
    ldv<VEC>(w + l, wv);
    if (MODE != 0) ldv_nc<VEC>(vprev + l, pv);
    if (MODE == 0 || MODE == 1) ldv_nc<VEC>(vcur + l, cv);
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      i64 wl = wv[e];
      if (MODE != 0) {
        const i64 vp = pv[e];
        const i64 d = asr(wmul(hs, vp), post);
        if (CHECKED) {
          nmul += mul_ovf(hs, vp);
          nsub += sub_ovf(wl, d);
        }
        wl = wsub(wl, d);
        wv[e] = wl;
      }
      i64 t = 0;
      if (MODE == 0 || MODE == 1) {
        const i64 a = asr(wl, sh.dot_b1);
        const i64 b = asr(cv[e], sh.dot_b2);
        t = wmul(a, b);
        if (CHECKED) nmul2 += mul_ovf(a, b);
      } else if (MODE == 2) {
        const i64 sq = asr(wl, sh.norm_b1);
        t = wmul(sq, sq);
        if (CHECKED) nmul2 += mul_ovf(sq, sq);
      }
      if (MODE != 3) {
        sum += static_cast<u64>(t);
        if (CHECKED) {
          const u64 at = t < 0 ? 0ull - static_cast<u64>(t) : static_cast<u64>(t);
          ahi += at >> 32;
          alo += at & 0xffffffffull;
        }
      }
    }
    if (MODE != 0) stv<VEC>(w + l, wv);
  }
  if (CHECKED) {
    if (MODE != 0) {
      bump(cnt_axpy, OP_MUL, nmul);
      bump(cnt_axpy, OP_SUB, nsub);
    }
    if (MODE != 3) bump(cnt_red, OP_MUL, nmul2);
  }
  if (MODE == 3) return;
  // block reduce (sum, ahi, alo)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_down_sync(0xffffffffu, sum, o);
    if (CHECKED) {
      ahi += __shfl_down_sync(0xffffffffu, ahi, o);
      alo += __shfl_down_sync(0xffffffffu, alo, o);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = sum;
    red[1][wid] = ahi;
    red[2][wid] = alo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    u64 s0 = 0, s1 = 0, s2 = 0;
    for (int i = 0; i < nw; ++i) {
      s0 += red[0][i];
      s1 += red[1][i];
      s2 += red[2][i];
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(acc_out), static_cast<unsigned long long>(s0));
    if (CHECKED) {
      atomicAdd(reinterpret_cast<unsigned long long*>(abs_out), static_cast<unsigned long long>(s1));
      atomicAdd(reinterpret_cast<unsigned long long*>(abs_out + 1), static_cast<unsigned long long>(s2));
    }
  }
}

// Standalone fx_dot / fx_norm partial sums (fxp.cpp:49-86) for the primitive
// entry points.  mode 0: dot, 1: norm.
template <bool CHECKED>
__global__ void __launch_bounds__(512) k_fx_red(long long n, int mode, const i64* __restrict__ v,
                                                const i64* __restrict__ w, int b1, int b2,
                                                u64* acc, u64* abs_out, u64* cnt) {
  __shared__ u64 red[3][16];
  u64 sum = 0, ahi = 0, alo = 0, nmul = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n; l += stride) {
    const i64 a = asr(v[l], b1);
    const i64 b = mode == 0 ? asr(w[l], b2) : a;
    const i64 t = wmul(a, b);
    sum += static_cast<u64>(t);
    if (CHECKED) {
      nmul += mul_ovf(a, b);
      const u64 at = t < 0 ? 0ull - static_cast<u64>(t) : static_cast<u64>(t);
      ahi += at >> 32;
      alo += at & 0xffffffffull;
    }
  }
  if (CHECKED) bump(cnt, OP_MUL, nmul);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_down_sync(0xffffffffu, sum, o);
    ahi += __shfl_down_sync(0xffffffffu, ahi, o);
    alo += __shfl_down_sync(0xffffffffu, alo, o);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = sum;
    red[1][wid] = ahi;
    red[2][wid] = alo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 s0 = 0, s1 = 0, s2 = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      s0 += red[0][i];
      s1 += red[1][i];
      s2 += red[2][i];
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(acc), static_cast<unsigned long long>(s0));
    atomicAdd(reinterpret_cast<unsigned long long*>(abs_out), static_cast<unsigned long long>(s1));
    atomicAdd(reinterpret_cast<unsigned long long*>(abs_out + 1), static_cast<unsigned long long>(s2));
  }
}

template <bool CHECKED>
__global__ void __launch_bounds__(512) k_axpy(long long n, i64* __restrict__ w, i64 h,
                                              const i64* __restrict__ v, int f, int b1, u64* cnt) {
  const i64 hs = asr(h, b1);
  const int post = f - b1;
  u64 nmul = 0, nsub = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n; l += stride) {
    const i64 vl = v[l];
    const i64 d = asr(wmul(hs, vl), post);
    const i64 wl = w[l];
    if (CHECKED) {
      nmul += mul_ovf(hs, vl);
      nsub += sub_ovf(wl, d);
    }
    w[l] = wsub(wl, d);
  }
  if (CHECKED) {
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_SUB, nsub);
  }
}

// K4 vec_div (gmres_int.cpp:117-126, fxp.hpp:220-234): per element fx_div
// by the step-invariant divisor via its exact reciprocal from Ctl.
template <bool CHECKED>
__global__ void __launch_bounds__(512) k_vec_div(long long n, const i64* __restrict__ w,
                                                 i64* __restrict__ out, int f, int b1, int b2,
                                                 u64* cnt, const Ctl* ctl) {
  if (!ctl->do_vecdiv) return;
  SDivMagic g;
  g.u.m = ctl->div_m;
  g.u.sh1 = ctl->div_sh1;
  g.u.sh2 = ctl->div_sh2;
  g.den_neg = ctl->div_neg;
  g.den_is_m1 = ctl->div_m1;
  const int e = f - b1 - b2;
  u64 nshl = 0, ndiv = 0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n; l += stride) {
    const i64 a = w[l];
    const i64 num = wrap_shl(a, b1);
    const i64 q = sdiv(num, g);
    i64 r;
    if (e >= 0) {
      r = wrap_shl(q, e);
      if (CHECKED) nshl += shl_ovf(q, e);
    } else {
      r = asr(q, -e);
    }
    if (CHECKED) {
      nshl += shl_ovf(a, b1);
      ndiv += sdiv_ovf(num, g);
    }
    out[l] = r;
  }
  if (CHECKED) {
    bump(cnt, OP_SHL, nshl);
    bump(cnt, OP_DIV, ndiv);
  }
}

// ---------------------------------------------------------------------------
// K5 per-step scalar work (gmres_int.cpp:101-159): finalise the h_ij from
// the wrapped accumulators, fx_norm -> h_{j+1,j}, vec_div reciprocal, the
// stored rotations, t_mp, (c, s), the g update, dim and break flags.  One
// thread; all overflow events counted in sequential order semantics.
struct Ev {
  u64* c;  // [K_COUNT][OP_COUNT] of this step
  bool on;
  __device__ void hit(int k, int op) {
    if (on) c[k * OP_COUNT + op] += 1;
  }
};

__device__ i64 d_fx_mul(i64 a, i64 b, int f, int b1, int b2, int of, Ev& ev, int k) {
  const i64 x = asr(a, b1), y = asr(b, b2);
  if (mul_ovf(x, y)) ev.hit(k, OP_MUL);
  return asr(wmul(x, y), 2 * f - b1 - b2 - of);
}

// returns false on a zero shifted divisor (domain_error)
__device__ bool d_fx_div(i64 a, i64 b, int f, int b1, int b2, i64* out, Ev& ev, int k) {
  const i64 num = wrap_shl(a, b1);
  if (shl_ovf(a, b1)) ev.hit(k, OP_SHL);
  const i64 den = asr(b, b2);
  if (den == 0) return false;
  i64 q;
  if (num == INT64_MIN && den == -1) {
    ev.hit(k, OP_DIV);
    q = num;
  } else {
    q = num / den;
  }
  const int e = f - b1 - b2;
  if (e >= 0) {
    if (shl_ovf(q, e)) ev.hit(k, OP_SHL);
    *out = wrap_shl(q, e);
  } else {
    *out = asr(q, -e);
  }
  return true;
}

__device__ void set_err(Ctl* ctl, int status, int msg, int step) {
  if (ctl->err == 0) {
    ctl->err = status;
    ctl->err_msg = msg;
    ctl->err_step = step;
  }
  ctl->stop = 1;
}

// exact sum|t| = hi*2^32 + lo < 2^63 certifies zero running-sum events
__device__ bool abs_small(const u64* ab) {
  const unsigned __int128 s = (static_cast<unsigned __int128>(ab[0]) << 32) + ab[1];
  return s < (static_cast<unsigned __int128>(1) << 63);
}

__global__ void k_step_scalar(int j, int f, ShiftsD sh, const u64* acc_col, const u64* abs_col,
                              const u64* nacc, const u64* nabs, i64* hess, int ld, i64* g,
                              i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step, Ctl* ctl,
                              int checked) {
  ctl->do_vecdiv = 0;
  if (cycle_over(ctl)) return;
  Ev ev{cnt_step, checked != 0};
  i64* col = hess + static_cast<long long>(j) * ld;
  // h_ij = fx_dot finalisation (fxp.cpp:63-65)
  const int e = f - sh.dot_b1 - sh.dot_b2;
  for (int i = 0; i <= j; ++i) {
    const i64 acc = static_cast<i64>(acc_col[i]);
    if (e >= 0) {
      col[i] = asr(acc, e);
    } else {
      if (shl_ovf(acc, -e)) ev.hit(K_DOT, OP_SHL);
      col[i] = wrap_shl(acc, -e);
    }
    if (checked && !abs_small(abs_col + 2 * i)) ctl->add_inexact = 1;
  }
  // h_{j+1,j} = fx_norm(w) (fxp.cpp:69-86)
  const i64 nsum = static_cast<i64>(*nacc);
  if (checked) {
    // all terms s*s are >= 0 unless a square itself wrapped: then the
    // running sum is monotone and its wrap count is exact.
    if (cnt_step[K_NORM * OP_COUNT + OP_MUL] == 0) {
      const unsigned __int128 s = (static_cast<unsigned __int128>(nabs[0]) << 32) + nabs[1];
      const unsigned __int128 wraps = (s + (static_cast<unsigned __int128>(1) << 63)) >> 64;
      cnt_step[K_NORM * OP_COUNT + OP_ADD] += static_cast<u64>(wraps);
    } else if (!abs_small(nabs)) {
      ctl->add_inexact = 1;
    }
  }
  if (nsum < 0) {
    set_err(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
    return;
  }
  i64 hnext;
  {
    const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(nsum)));
    const int es = sh.norm_b1;  // out_frac - fin/2 = f - (f - b1)
    if (shl_ovf(r, es)) ev.hit(K_NORM, OP_SHL);
    hnext = wrap_shl(r, es);
  }
  col[j + 1] = hnext;
  ctl->hnext = hnext;
  const bool happy = hnext == 0;
  if (!happy) {
    const i64 den = asr(hnext, sh.div_b2);
    if (den == 0) {
      if (shl_ovf(w[0], sh.div_b1)) ev.hit(K_VEC_DIV, OP_SHL);
      set_err(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
      return;
    }
    const SDivMagic gm = make_sdiv(den);
    ctl->div_m = gm.u.m;
    ctl->div_sh1 = gm.u.sh1;
    ctl->div_sh2 = gm.u.sh2;
    ctl->div_neg = gm.den_neg;
    ctl->div_m1 = gm.den_is_m1;
    ctl->do_vecdiv = 1;
    ctl->nbasis = j + 2;
  }
  // apply_stored_rotations (gmres_int.cpp:8-25)
  for (int i = 0; i < j; ++i) {
    const i64 c = cs[i], s = sn[i], hi = col[i], hn = col[i + 1];
    const i64 a = d_fx_mul(c, hi, f, 0, sh.givens_b2, f, ev, K_GIVENS);
    const i64 b = d_fx_mul(s, hn, f, 0, sh.givens_b2, f, ev, K_GIVENS);
    const i64 d = d_fx_mul(c, hn, f, 0, sh.givens_b2, f, ev, K_GIVENS);
    const i64 q = d_fx_mul(s, hi, f, 0, sh.givens_b2, f, ev, K_GIVENS);
    if (add_ovf(a, b)) ev.hit(K_GIVENS, OP_ADD);
    if (sub_ovf(d, q)) ev.hit(K_GIVENS, OP_SUB);
    col[i] = wadd(a, b);
    col[i + 1] = wsub(d, q);
  }
  // t_mp = fx_norm((h_jj, h_{j+1,j})) (gmres_int.cpp:133-137)
  i64 tmp;
  {
    const i64 s0 = asr(col[j], sh.norm_b1), s1 = asr(col[j + 1], sh.norm_b1);
    if (mul_ovf(s0, s0)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const i64 p0 = wmul(s0, s0);
    i64 acc = p0;  // 0 + p0 never overflows
    if (mul_ovf(s1, s1)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const i64 p1 = wmul(s1, s1);
    if (add_ovf(acc, p1)) ev.hit(K_GIVENS_NORM, OP_ADD);
    acc = wadd(acc, p1);
    if (acc < 0) {
      set_err(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
      return;
    }
    const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(acc)));
    if (shl_ovf(r, sh.norm_b1)) ev.hit(K_GIVENS_NORM, OP_SHL);
    tmp = wrap_shl(r, sh.norm_b1);
  }
  if (tmp == 0) {  // column vanished under rotation: drop it, dim unchanged
    ctl->stop = 1;
    return;
  }
  i64 c, s;
  if (!d_fx_div(col[j], tmp, f, sh.div_b1, sh.div_b2, &c, ev, K_GIVENS_DIV) ||
      !d_fx_div(col[j + 1], tmp, f, sh.div_b1, sh.div_b2, &s, ev, K_GIVENS_DIV)) {
    set_err(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
    return;
  }
  cs[j] = c;
  sn[j] = s;
  col[j] = tmp;
  col[j + 1] = 0;
  // residual estimate (gmres_int.cpp:150-153)
  const i64 g_old = g[j];
  if (sub_ovf(0, s)) ev.hit(K_ROT, OP_SUB);
  const i64 neg_s = wsub(0, s);
  g[j + 1] = d_fx_mul(neg_s, g_old, f, sh.rot_b, sh.rot_b, f, ev, K_ROT);
  g[j] = d_fx_mul(c, g_old, f, sh.rot_b, sh.rot_b, f, ev, K_ROT);
  ctl->dim = j + 1;
  gabs[j] = g[j + 1];
  if (happy) ctl->stop = 1;
}

__global__ void k_cycle_init(Ctl* ctl, i64* g, int f) {
  ctl->stop = 0;
  ctl->dim = 0;
  ctl->nbasis = 1;
  ctl->do_vecdiv = 0;
  ctl->add_inexact = 0;
  ctl->r0n = 0.0;
  g[0] = i64{1} << f;
}

// K11 (gmres_int.cpp:163-175): decode R and g, back substitution, weights
// r0n * y_j.  One thread; dim <= m is tiny.
__global__ void k_cycle_finish(int m, int f, const i64* hess, const i64* g, double* y,
                               double* wts, Ctl* ctl) {
  if (ctl->err) return;
  const int dim = ctl->dim;
  if (dim == 0) return;
  const int ld = m + 1;
  const double sc = ldexp(1.0, -f);
  for (int i = dim - 1; i >= 0; --i) {
    double acc = dec(g[i], sc);
    for (int jj = i + 1; jj < dim; ++jj)
      acc = __dsub_rn(acc, __dmul_rn(dec(hess[static_cast<long long>(jj) * ld + i], sc), y[jj]));
    const double rii = dec(hess[static_cast<long long>(i) * ld + i], sc);
    if (rii == 0.0) {
      set_err(ctl, IGM_RUNTIME_ERROR, EM_HESS_ZERO, -2);
      return;
    }
    y[i] = __ddiv_rn(acc, rii);
  }
  for (int jj = 0; jj < dim; ++jj) wts[jj] = __dmul_rn(ctl->r0n, y[jj]);
}

// x update (gmres_int.cpp:176-179, refine.cpp:87).
//   mode 0 (run_cycle): x = x0 + sum_j wts_j * decode(v_j), in j order.
//   mode 1 (solve):     x += gamma * (0.0 + sum_j wts_j * decode(v_j)).
__global__ void __launch_bounds__(256) k_xupdate(long long n, int f, const i64* __restrict__ basis,
                                                 const double* __restrict__ wts,
                                                 const double* __restrict__ x0,
                                                 double* __restrict__ x, const Ctl* ctl, int mode) {
  if (ctl->err) return;
  const int dim = ctl->dim;
  if (mode == 1 && dim == 0) return;
  const double sc = ldexp(1.0, -f);
  const double gamma = __longlong_as_double(static_cast<long long>(ctl->rmax_bits));
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    double acc = mode == 0 ? (x0 ? x0[l] : 0.0) : 0.0;
    for (int jj = 0; jj < dim; ++jj)
      acc = __dadd_rn(acc, __dmul_rn(wts[jj], dec(basis[static_cast<long long>(jj) * n + l], sc)));
    if (mode == 0)
      x[l] = acc;
    else
      x[l] = __dadd_rn(x[l], __dmul_rn(gamma, acc));
  }
}

// ---------------------------------------------------------------------------
// K6/K9 ILU(0) triangular substitutions (ilu.cpp:122-180), sync-free
// wavefront.  Rows are split into contiguous tiles; a CTA takes tiles in
// dependency order from a ticket counter (so every tile it waits on is
// already owned by a running CTA: deadlock-free for any grid size), walks
// its tile's rows level by level keeping the tile's results in shared
// memory, and publishes per-tile progress ("all rows with level <= p are
// final") with release/acquire.  Cross-tile dependencies wait on that
// progress word and read the value through L2.
//
// Row records are stored in schedule order (upload-time permutation), so a
// segment's records are contiguous and coalesced; the whole tile's records
// are bulk-prefetched into L2 when the CTA starts, and each thread keeps the
// NEXT segment's record in registers while it works on the current one, so
// the per-level critical path is only: wait -> dependency values -> multiply,
// subtract -> exact reciprocal division -> store.
//
// Per row the arithmetic is the reference's: CSR order, wrapping mul/sub,
// truncating division by the raw diagonal (exact reciprocal), or the same in
// FP64 on the integer factors with no contraction.
struct TriArgs {
  int n, ntiles;
  const int* tile_pbase;  // first schedule slot of each tile
  const int* tile_seg;
  const int* seg_level;
  const int* seg_rows;
  const int* seg_wptr;    // external producer tiles per segment
  const int* seg_wt;
  const int* p_row;       // row id per slot
  const int* p_nd;        // dependency count per slot
  const int* p_dep;       // slot*stride: >= 0 tile-local slot, < 0 ~global row
  const i64* p_val;
  const int* p_xrp;       // dependencies beyond stride (CSR)
  const int* p_xdep;
  const i64* p_xval;
  const u64* p_mag;       // exact reciprocal of |diag| per slot
  const int* p_info;      // sh1 | sh2 << 1 | neg << 8 | (diag == -1) << 9
  const i64* p_diag;
  const unsigned char* p_rec;  // packed per-slot records (schedule.hpp)
  int tile_cap;
  ulonglong2* xz;              // exported values: (value, epoch ^ mix(value)) per row
  unsigned long long epoch;    // unique per launch
  const int* seg_xptr;         // per segment: cross-tile producer rows
  const int* seg_xrow;
  int max_seg_ext;
  const int* c_rp;             // stripped factor, natural order (counting pass)
  const int* c_ci;
  const i64* c_val;
  const i64* c_diag;
  int* prog;
  int* ticket;
};

template <int MAXD>
struct RowRec {
  int row, nd, slot, xb;
  u64 mag;
  int info;
  i64 diag;
  int ci[MAXD];
  i64 v[MAXD];
};

// every address is a function of p alone: the loads issue back to back and
// only the consumer (next segment) waits for them
template <int MAXD, bool FP>
__device__ __forceinline__ void load_rec(const TriArgs& a, int p, int pb, RowRec<MAXD>& r) {
  r.row = __ldg(a.p_row + p);
  r.nd = __ldg(a.p_nd + p);
  r.slot = p - pb;
  r.xb = __ldg(a.p_xrp + p);
  if (FP) {
    r.diag = __ldg(a.p_diag + p);
  } else {
    r.mag = __ldg(a.p_mag + p);
    r.info = __ldg(a.p_info + p);
  }
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    r.ci[d] = __ldg(a.p_dep + static_cast<size_t>(p) * MAXD + d);
    r.v[d] = __ldg(a.p_val + static_cast<size_t>(p) * MAXD + d);
  }
}

__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
  // bulk L2 prefetch of [p, p+bytes), 16-byte granular (allocations are padded)
  const size_t a = reinterpret_cast<size_t>(p) & ~size_t(15);
  size_t e = (reinterpret_cast<size_t>(p) + bytes + 15) & ~size_t(15);
  for (size_t q = a; q < e; q += (1u << 20)) {
    const unsigned len = static_cast<unsigned>(min(e - q, static_cast<size_t>(1u << 20)));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(len) : "memory");
  }
}

template <typename T, bool CHECKED>
struct TriAcc {
  u64 nmul = 0, nsub = 0, ndiv = 0;
};

// one dependency term: acc -= l_ij * z_j (value from smem or, cross-tile,
// from L2 after the segment's poller acquired the producer's progress)
__device__ __forceinline__ u64 xz_mix(u64 v) { return v * 0x9E3779B97F4A7C15ull; }

// cross-tile value: spin on its 128-bit (value, tag) word -- one single-copy
// atomic strong access, so no fence/flag protocol is needed; the tag binds
// the value to this launch (and guards against a torn read)
__device__ __forceinline__ u64 xz_wait(const ulonglong2* p, u64 epoch) {
  u64 v, tg;
  do {
    asm volatile("{ .reg .b128 t; ld.global.relaxed.gpu.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                 : "=l"(v), "=l"(tg)
                 : "l"(p)
                 : "memory");
  } while (tg != (epoch ^ xz_mix(v)));
  return v;
}

__device__ __forceinline__ void xz_put(ulonglong2* p, u64 v, u64 epoch) {
  asm volatile("{ .reg .b128 t; mov.b128 t, {%0, %1}; st.global.relaxed.gpu.b128 [%2], t; }" ::"l"(v),
               "l"(epoch ^ xz_mix(v)), "l"(p)
               : "memory");
}

template <typename T>
__device__ __forceinline__ T bits_to(u64 b) {
  if constexpr (std::is_same<T, double>::value) return __longlong_as_double(static_cast<long long>(b));
  else return static_cast<T>(b);
}
template <typename T>
__device__ __forceinline__ u64 to_bits(T v) {
  if constexpr (std::is_same<T, double>::value) return static_cast<u64>(__double_as_longlong(v));
  else return static_cast<u64>(v);
}

// one cross-tile word (value, tag) loaded ahead of use
__device__ __forceinline__ void xz_load(const ulonglong2* p, u64& v, u64& tg) {
  asm volatile("{ .reg .b128 t; ld.global.relaxed.gpu.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(v), "=l"(tg)
               : "l"(p)
               : "memory");
}

template <typename T, bool CHECKED>
__device__ __forceinline__ void tri_term(int c, i64 lv, u64 xv, u64 xt, const TriArgs& a, const T* zt,
                                         T& acc, TriAcc<T, CHECKED>& st) {
  T zj;
  if (c >= 0) {
    zj = zt[c];  // tile-local value
  } else {       // cross-tile: the word was loaded one level early; spin only if not yet valid
    zj = bits_to<T>(xt == (a.epoch ^ xz_mix(xv)) ? xv : xz_wait(a.xz + ~c, a.epoch));
  }
  if constexpr (std::is_same<T, double>::value) {
    acc = __dsub_rn(acc, __dmul_rn(__ll2double_rn(lv), zj));
  } else {
    const i64 pr = wmul(lv, zj);
    if (CHECKED) {
      st.nmul += mul_ovf(lv, zj);
      st.nsub += sub_ovf(acc, pr);
    }
    acc = wsub(acc, pr);
  }
}

template <typename T, bool CHECKED, int MAXD>
__device__ __forceinline__ void tri_row(const TriArgs& a, const RowRec<MAXD>& r, T acc, T* out,
                                        T* zt, const u64 (&xv)[MAXD], const u64 (&xt)[MAXD],
                                        TriAcc<T, CHECKED>& st) {
#pragma unroll
  for (int d = 0; d < MAXD; ++d)
    if (d < r.nd) tri_term<T, CHECKED>(r.ci[d], r.v[d], xv[d], xt[d], a, zt, acc, st);
  for (int d = MAXD; d < r.nd; ++d)
    tri_term<T, CHECKED>(__ldg(a.p_xdep + r.xb + d - MAXD), __ldg(a.p_xval + r.xb + d - MAXD), 0,
                         ~a.epoch /* never a valid tag for value 0: forces the spin path */, a, zt, acc, st);
  T z;
  if constexpr (std::is_same<T, double>::value) {
    z = __ddiv_rn(acc, __ll2double_rn(r.diag));
  } else {
    SDivMagic gm;
    gm.u.m = r.mag;
    gm.u.sh1 = r.info & 1;
    gm.u.sh2 = (r.info >> 1) & 127;
    gm.den_neg = (r.info >> 8) & 1;
    gm.den_is_m1 = (r.info >> 9) & 1;
    if (CHECKED) st.ndiv += sdiv_ovf(acc, gm);
    z = sdiv(acc, gm);
  }
  zt[r.slot] = z;
#ifndef IGM_TRI_NOSTORE
  out[r.row] = z;
  if (r.info & (1 << 10)) xz_put(a.xz + r.row, to_bits<T>(z), a.epoch);  // read by another tile
#endif
}

// Integer row, straight-line: every one of the MAXD dependency slots is used
// (unused slots are padded with factor 0 and local slot 0 at upload, which
// adds exact zeros mod 2^64), the products are independent and summed as a
// tree (integer wrapping sums are order-free), cross-tile words were loaded
// one level early and are only re-polled if their tag is not yet valid.
template <int MAXD>
__device__ __forceinline__ i64 tri_row_int_fast(const TriArgs& a, const RowRec<MAXD>& r, i64 y,
                                                const i64* zt, const u64 (&xv)[MAXD],
                                                const u64 (&xt)[MAXD]) {
  i64 z[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) z[d] = zt[r.ci[d] < 0 ? 0 : r.ci[d]];
  bool stale = false;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (r.ci[d] < 0) {
      z[d] = static_cast<i64>(xv[d]);
      stale |= xt[d] != (a.epoch ^ xz_mix(xv[d]));
    }
  }
  if (stale) {  // a producer tile had not published yet when the word was loaded
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (r.ci[d] < 0 && xt[d] != (a.epoch ^ xz_mix(xv[d])))
        z[d] = static_cast<i64>(xz_wait(a.xz + ~r.ci[d], a.epoch));
  }
  u64 s = 0;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) s += static_cast<u64>(r.v[d]) * static_cast<u64>(z[d]);
  for (int d = MAXD; d < r.nd; ++d) {  // rows wider than the record stride (rare)
    const int c = __ldg(a.p_xdep + r.xb + d - MAXD);
    const i64 zj = c >= 0 ? zt[c] : static_cast<i64>(xz_wait(a.xz + ~c, a.epoch));
    s += static_cast<u64>(__ldg(a.p_xval + r.xb + d - MAXD)) * static_cast<u64>(zj);
  }
  const i64 acc = static_cast<i64>(static_cast<u64>(y) - s);
  SDivMagic gm;
  gm.u.m = r.mag;
  gm.u.sh1 = r.info & 1;
  gm.u.sh2 = (r.info >> 1) & 127;
  gm.den_neg = (r.info >> 8) & 1;
  gm.den_is_m1 = (r.info >> 9) & 1;
  return sdiv(acc, gm);
}

template <typename T>
__device__ __forceinline__ T tri_load_y(const T* __restrict__ y, int row, bool scaled, double gamma) {
  if constexpr (std::is_same<T, double>::value) return scaled ? __ddiv_rn(y[row], gamma) : y[row];
  else return y[row];
}

__device__ int g_tri_sync_loader = 0;  // A/B switch (IGM_TRI_SYNC_LOADER)

// debug: per-segment phase timestamps of one tile (igm_debug_tri_trace)
__device__ unsigned long long* g_tri_ts = nullptr;
__device__ int g_tri_ts_tile = -1;
__device__ __forceinline__ unsigned long long gtime() {
  // SM cycle counter (the global timer ticks at ~1 us on this part); only
  // differences within one CTA are meaningful
  return clock64();
}

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- mbarrier / bulk-copy helpers (sm_90+ PTX, valid on sm_100a)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, void* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(void* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wavefront CTA (one tile per CTA):
//   warps 0-7  compute: one row per thread per level (segments <= 256 rows);
//              a named barrier per level orders the tile's shared-memory values
//   warp  8    loader: streams each level's packed row records (one TMA bulk
//              copy) and right-hand-side values (cp.async gathers) into a
//              shared-memory ring L levels ahead (mbarriers full/empty)
// Values another tile needs are published as one aligned 128-bit
// (value, tag) store and consumed by spinning on that word; there are no
// progress flags and no gpu-scope fences (a fence's cost grows with the
// SM's in-flight traffic: ~15 us here).  Tiles are handed out by a ticket
// counter in a layer-major order, so every producer a thread waits on is
// already running (schedule.hpp).
constexpr int kTriCompute = 256;
constexpr int kTriThreads = kTriCompute + 32;  // + loader warp

struct TriSmem {  // byte offsets of the dynamic shared-memory regions
  size_t rows, lev, ring, bars, total;
  int ring_slot;
};

template <typename T, int MAXD>
__host__ __device__ inline TriSmem tri_smem_layout(int tile_cap, int seg_cap, int L, int max_ext) {
  constexpr int REC = 32 + 12 * MAXD;
  TriSmem m;
  size_t o = (static_cast<size_t>(tile_cap) * sizeof(T) + 15) & ~size_t(15);
  m.rows = o;
  o += sizeof(int) * static_cast<size_t>(seg_cap);
  m.lev = o;
  o += sizeof(int) * static_cast<size_t>(seg_cap);
  o = (o + 127) & ~size_t(127);
  m.ring = o;
  m.ring_slot = kTriSegRows * (REC + 8) + ((8 * max_ext + 15) & ~15);
  o += static_cast<size_t>(L) * m.ring_slot;
  o = (o + 15) & ~size_t(15);
  m.bars = o;
  o += 24 * static_cast<size_t>(L);  // full, empty, xfull
  m.total = o;
  return m;
}

template <typename T, bool BACKWARD, bool CHECKED, int MAXD>
__global__ void __launch_bounds__(kTriThreads) k_tri(TriArgs a, const T* __restrict__ y, T* out,
                                                     u64* cnt, const Ctl* ctl,
                                                     const double* prescale, int seg_cap, int L) {
  constexpr bool FP = std::is_same<T, double>::value;
  constexpr int REC = 32 + 12 * MAXD;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ int s_tile;
  if (cycle_over(ctl)) return;
  const TriSmem lay = tri_smem_layout<T, MAXD>(a.tile_cap, seg_cap, L, a.max_seg_ext);
  T* zt = reinterpret_cast<T*>(smem_raw);
  int* s_rows = reinterpret_cast<int*>(smem_raw + lay.rows);
  unsigned char* ring = smem_raw + lay.ring;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw + lay.bars);
  unsigned long long* empty = full + L;
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(a.ticket, 1);
    for (int k = 0; k < L; ++k) {
      mbar_init(full + k, g_tri_sync_loader ? 32 : 33);  // lane-0 expect_tx + 32 cp.async arrivals
      mbar_init(empty + k, kTriCompute / 32);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int tile = BACKWARD ? a.ntiles - 1 - s_tile : s_tile;
  const int pb = __ldg(a.tile_pbase + tile);
  const int sb = __ldg(a.tile_seg + tile), se = __ldg(a.tile_seg + tile + 1);
  const int nsg = se - sb;
  const bool seg_in_smem = nsg + 2 <= seg_cap;
  if (seg_in_smem)
    for (int q = threadIdx.x; q <= nsg; q += blockDim.x) s_rows[q] = __ldg(a.seg_rows + sb + q);
  __syncthreads();
  auto seg_row = [&](int q) { return seg_in_smem ? s_rows[q] : __ldg(a.seg_rows + sb + q); };
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#ifdef IGM_TRI_TRACE
  unsigned long long* tsb = (!BACKWARD && g_tri_ts != nullptr && tile == g_tri_ts_tile) ? g_tri_ts : nullptr;
#else
  constexpr unsigned long long* tsb = nullptr;  // phase timestamps compiled out
#endif

  if (warp == 8) {  // ---------------- loader
    // row ids are loaded D levels ahead (register pipeline), so the
    // right-hand-side gathers never wait on a dependent load
    constexpr int RPL = kTriSegRows / 32;  // rows per lane per level
    constexpr int D = 4;
    int rows[D][RPL];
    auto load_rows = [&](int q, int (&rr)[RPL]) {
      if (q >= nsg) return;
      const int s0 = seg_row(q), c = seg_row(q + 1) - s0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int r = lane + 32 * t;
        rr[t] = r < c ? __ldg(a.p_row + s0 + r) : 0;
      }
    };
#pragma unroll
    for (int d = 0; d < D; ++d) load_rows(d, rows[d]);
    int k = 0;
    unsigned ph = 1;  // parity of the previous use of slot k (first L levels: none)
    for (int q0 = 0; q0 < nsg; q0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {  // unrolled so rows[d] stays in registers
        const int q = q0 + d;
        if (q >= nsg) break;
        if (q >= L) mbar_wait(empty + k, ph);
        const int s0 = seg_row(q), c = seg_row(q + 1) - s0;
        unsigned char* slot = ring + static_cast<size_t>(k) * lay.ring_slot;
        T* yslot = reinterpret_cast<T*>(slot + kTriSegRows * REC);
        if (g_tri_sync_loader) {  // A/B: synchronous copy through registers
          const int4* src = reinterpret_cast<const int4*>(a.p_rec + static_cast<size_t>(s0) * REC);
          int4* dst = reinterpret_cast<int4*>(slot);
          for (int i = lane; i < c * REC / 16; i += 32) dst[i] = __ldg(src + i);
#pragma unroll
          for (int t = 0; t < RPL; ++t)
            if (lane + 32 * t < c) yslot[lane + 32 * t] = y[rows[d][t]];
          __syncwarp();
          mbar_arrive(full + k);
        } else {
          if (lane == 0) {
            mbar_arrive_expect_tx(full + k, static_cast<unsigned>(c * REC));
            bulk_g2s(slot, a.p_rec + static_cast<size_t>(s0) * REC, static_cast<unsigned>(c * REC), full + k);
          }
#pragma unroll
          for (int t = 0; t < RPL; ++t)
            if (lane + 32 * t < c) cp_async8(yslot + lane + 32 * t, y + rows[d][t]);
          cp_async_mbar_arrive(full + k);
        }
        if (tsb && lane == 0 && q < 2048) tsb[q * 8 + 7] = gtime();
        load_rows(q + D, rows[d]);
        if (++k == L) {
          k = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  // ---------------- compute warps
  const bool scaled = prescale != nullptr;
  const double gamma = scaled ? __longlong_as_double(*reinterpret_cast<const long long*>(prescale)) : 1.0;
  TriAcc<T, CHECKED> stt;
  const int tid = threadIdx.x;
  // one row per thread per level: the per-level critical path is this warp's
  // in-order instruction stream, so everything loop-invariant or derivable
  // incrementally stays out of it
  auto read_rec = [&](const unsigned char* slotp, int s0, RowRec<MAXD>& r) {
    const unsigned char* rp = slotp + static_cast<size_t>(tid) * REC;
    const int4 hdr = *reinterpret_cast<const int4*>(rp);
    r.row = hdr.x;
    r.nd = hdr.y;
    r.info = hdr.z;
    r.xb = hdr.w;
    if (FP) r.diag = *reinterpret_cast<const i64*>(rp + 24);
    else r.mag = *reinterpret_cast<const u64*>(rp + 16);
    r.slot = s0 + tid - pb;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      r.ci[d] = *reinterpret_cast<const int*>(rp + 32 + 4 * d);
      r.v[d] = *reinterpret_cast<const i64*>(rp + 32 + 4 * MAXD + 8 * d);
    }
  };
  // record + cross-tile words of the NEXT level, issued before this level's barrier
  RowRec<MAXD> nrec;
  u64 nxv[MAXD], nxt[MAXD];
  bool nhave = false;
  int kn = 0;          // ring slot of the next level
  unsigned phn = 0;    // its mbarrier phase parity
  int s_next = seg_row(0);
  auto prefetch = [&](int q) {
    nhave = false;
    if (q >= nsg) return;
    mbar_wait(full + kn, phn);
    const int s1 = seg_row(q + 1);
    const int s0 = s_next;
    s_next = s1;
    if (tid >= s1 - s0) return;
    read_rec(ring + static_cast<size_t>(kn) * lay.ring_slot, s0, nrec);
    nhave = true;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < nrec.nd && nrec.ci[d] < 0) xz_load(a.xz + ~nrec.ci[d], nxv[d], nxt[d]);
  };
  prefetch(0);
  for (int q = 0; q < nsg; ++q) {
    const int k = kn;
    if (++kn == L) {
      kn = 0;
      phn ^= 1u;
    }
    const RowRec<MAXD> cur = nrec;
    u64 xv[MAXD], xt[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      xv[d] = nxv[d];
      xt[d] = nxt[d];
    }
    const bool hc = nhave;
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 2] = gtime();
    bar_sync(1, kTriCompute);  // level q-1 values of this tile are in shared memory
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 3] = gtime();
#ifdef IGM_TRI_SKELETON
    if (false) {
#else
    if (hc) {
#endif
      const unsigned char* slot = ring + static_cast<size_t>(k) * lay.ring_slot;
      T yv = reinterpret_cast<const T*>(slot + kTriSegRows * REC)[tid];
      if constexpr (FP) {
        if (scaled) yv = __ddiv_rn(yv, gamma);
      }
      if constexpr (FP) {
        tri_row<T, CHECKED, MAXD>(a, cur, yv, out, zt, xv, xt, stt);
      } else {
        const i64 z = tri_row_int_fast<MAXD>(a, cur, yv, zt, xv, xt);
        zt[cur.slot] = z;
#ifndef IGM_TRI_NOSTORE
        out[cur.row] = z;
        if (cur.info & (1 << 10)) xz_put(a.xz + cur.row, static_cast<u64>(z), a.epoch);
#endif
      }
    }
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 5] = gtime();
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + k);
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 6] = gtime();
    prefetch(q + 1);
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 4] = gtime();
  }
  if (CHECKED && !FP) {
    bump(cnt, OP_MUL, stt.nmul);
    bump(cnt, OP_SUB, stt.nsub);
    bump(cnt, OP_DIV, stt.ndiv);
  }
}

// Checked-mode overflow events of one integer substitution (ilu.cpp:126-153),
// counted AFTER the wavefront from its inputs and outputs: every row's
// products and subtractions are known once z is, so this is a fully parallel
// pass and the 3g-level critical path stays free of overflow tests.
__global__ void __launch_bounds__(256) k_tri_count(int n, const int* __restrict__ rp,
                                                   const int* __restrict__ ci,
                                                   const i64* __restrict__ val,
                                                   const i64* __restrict__ diag,
                                                   const i64* __restrict__ y,
                                                   const i64* __restrict__ z, u64* cnt,
                                                   const Ctl* ctl) {
  if (cycle_over(ctl)) return;
  u64 nmul = 0, nsub = 0, ndiv = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    i64 acc = y[i];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const i64 l = val[k], zj = z[ci[k]];
      const i64 p = wmul(l, zj);
      nmul += mul_ovf(l, zj);
      nsub += sub_ovf(acc, p);
      acc = wsub(acc, p);
    }
    ndiv += (acc == INT64_MIN && diag[i] == -1);
  }
  bump(cnt, OP_MUL, nmul);
  bump(cnt, OP_SUB, nsub);
  bump(cnt, OP_DIV, ndiv);
}

TriArgs tri_args(const DevTri& t) {
  TriArgs a;
  a.n = t.n;
  a.ntiles = t.ntiles;
  a.tile_pbase = t.tile_pbase;
  a.tile_seg = t.tile_seg;
  a.seg_level = t.seg_level;
  a.seg_rows = t.seg_rows;
  a.seg_wptr = t.seg_wptr;
  a.seg_wt = t.seg_wt;
  a.p_row = t.p_row;
  a.p_nd = t.p_nd;
  a.p_dep = t.p_dep;
  a.p_val = t.p_val;
  a.p_xrp = t.p_xrp;
  a.p_xdep = t.p_xdep;
  a.p_xval = t.p_xval;
  a.p_mag = t.p_mag;
  a.p_info = t.p_info;
  a.p_diag = t.p_diag;
  a.p_rec = t.p_rec;
  a.tile_cap = t.tile_cap;
  a.xz = t.xz;
  a.epoch = 0;
  a.seg_xptr = t.seg_xptr;
  a.seg_xrow = t.seg_xrow;
  a.max_seg_ext = t.max_seg_ext;
  a.c_rp = t.c_rp;
  a.c_ci = t.c_ci;
  a.c_val = t.c_val;
  a.c_diag = t.c_diag;
  a.prog = t.prog;
  a.ticket = t.ticket;
  return a;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers

#define LAUNCH_CHECK() ++g_launches

void launch_spmv_int(cudaStream_t st, const DevSplit& m, int s, const i64* v, i64* out, u64* cnt,
                     const Ctl* ctl, bool checked) {
  ProfScope prof_(st, KC_SPMV);
  const int nt = 256;
  const int g = static_cast<int>((m.n + nt - 1) / nt > 0 ? (m.n + nt - 1) / nt : 1);
  if (checked)
    k_spmv_int<true><<<g, nt, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v, out, cnt, ctl);
  else
    k_spmv_int<false><<<g, nt, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v, out, cnt, ctl);
  LAUNCH_CHECK();
}

void launch_spmv_fp_split(cudaStream_t st, const DevSplit& m, int s, const double* x,
                          const double* b, double* y, const Ctl* ctl) {
  ProfScope prof_(st, KC_OTHER);
  const int nt = 256;
  const int g = (m.n + nt - 1) / nt > 0 ? (m.n + nt - 1) / nt : 1;
  k_spmv_fp_split<<<g, nt, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, x, b, y, ctl);
  LAUNCH_CHECK();
}

void launch_residual(cudaStream_t st, const DevCsrf& a, const double* x, const double* b,
                     double* r, Ctl* ctl, bool track_max) {
  ProfScope prof_(st, KC_RESIDUAL);
  const int nt = 256;
  const int g = (a.n + nt - 1) / nt > 0 ? (a.n + nt - 1) / nt : 1;
  k_residual<<<g, nt, 0, st>>>(a.n, a.row_ptr, a.col_idx, a.vals, x, b, r, ctl, track_max ? 1 : 0);
  LAUNCH_CHECK();
}

void launch_gamma(cudaStream_t st, long long n, const double* r, Ctl* ctl) {
  ProfScope prof_(st, KC_OTHER);
  k_gamma<<<grid_for(n, 256), 256, 0, st>>>(n, r, ctl);
  LAUNCH_CHECK();
}

void launch_scale_div(cudaStream_t st, long long n, const double* r, double* out, const Ctl* ctl) {
  ProfScope prof_(st, KC_OTHER);
  k_scale_div<<<grid_for(n, 256), 256, 0, st>>>(n, r, out, ctl);
  LAUNCH_CHECK();
}

static bool norm2_serial_forced() {
  static const int v = [] {
    const char* e = std::getenv("IGM_NORM2_SERIAL");
    return e && e[0] == '1' ? 1 : 0;
  }();
  return v != 0;
}

void launch_norm2_serial(cudaStream_t st, long long n, const double* v, double* out, Ctl* ctl,
                         int mode) {
  ProfScope prof_(st, KC_NORM2);
  if (norm2_serial_forced())
    k_norm2_serial<<<1, 256, 0, st>>>(n, v, nullptr, 1.0, out, ctl, mode, 0);
  else
    k_norm2_exact<<<1, kN2Threads, 0, st>>>(n, v, nullptr, 1.0, out, ctl, mode, 0);
  LAUNCH_CHECK();
}

void launch_basis_norms(cudaStream_t st, long long n, int nb, int f, const i64* basis, double* tmp,
                        double* out, Ctl* ctl) {
  ProfScope prof_(st, KC_NORM2);
  (void)tmp;
  for (int k = 0; k < nb; ++k) {
    k_norm2_exact<<<1, kN2Threads, 0, st>>>(n, nullptr, basis + static_cast<long long>(k) * n,
                                            ldexp(1.0, -f), out, ctl, 4, k);
    LAUNCH_CHECK();
  }
}

void launch_encode(cudaStream_t st, long long n, const double* r0, i64* v0, int f, Ctl* ctl) {
  ProfScope prof_(st, KC_ENCODE);
  k_encode<<<grid_for(n, 256), 256, 0, st>>>(n, r0, v0, f, ctl);
  LAUNCH_CHECK();
}

void launch_mgs_pass(cudaStream_t st, long long n, int mode, i64* w, const i64* vprev,
                     const i64* vcur, const u64* hacc, u64* acc_out, u64* abs_out, int f,
                     ShiftsD sh, u64* cnt_axpy, u64* cnt_red, const Ctl* ctl, bool checked) {
  ProfScope prof_(st, KC_MGS);
  const int nt = 512;
  const int g = static_cast<int>(std::max<long long>(1, std::min<long long>(2LL * num_sms(0), (n / 4 + nt - 1) / nt)));
  // 256-bit accesses when every stream is 32-byte aligned (n % 4 == 0 and
  // aligned bases); scalar otherwise
  auto al32 = [](const void* p) { return (reinterpret_cast<size_t>(p) & 31) == 0; };
  const bool v4 = (n % 4 == 0) && al32(w) && (!vprev || al32(vprev)) && (!vcur || al32(vcur));
#define MGS_CASE(MD)                                                                                 \
  if (v4) {                                                                                          \
    if (checked)                                                                                     \
      k_mgs<MD, true, 4><<<g, nt, 0, st>>>(n, w, vprev, vcur, hacc, acc_out, abs_out, f, sh,          \
                                           cnt_axpy, cnt_red, ctl);                                  \
    else                                                                                             \
      k_mgs<MD, false, 4><<<g, nt, 0, st>>>(n, w, vprev, vcur, hacc, acc_out, abs_out, f, sh,         \
                                            cnt_axpy, cnt_red, ctl);                                 \
  } else {                                                                                           \
    if (checked)                                                                                     \
      k_mgs<MD, true, 1><<<g, nt, 0, st>>>(n, w, vprev, vcur, hacc, acc_out, abs_out, f, sh,          \
                                           cnt_axpy, cnt_red, ctl);                                  \
    else                                                                                             \
      k_mgs<MD, false, 1><<<g, nt, 0, st>>>(n, w, vprev, vcur, hacc, acc_out, abs_out, f, sh,         \
                                            cnt_axpy, cnt_red, ctl);                                 \
  }
  switch (mode) {
    case 0: MGS_CASE(0) break;
    case 1: MGS_CASE(1) break;
    case 2: MGS_CASE(2) break;
    default: MGS_CASE(3) break;
  }
#undef MGS_CASE
  LAUNCH_CHECK();
}

void launch_fx_red(cudaStream_t st, long long n, int mode, const i64* v, const i64* w, int b1,
                   int b2, u64* acc, u64* abs_out, u64* cnt, bool checked) {
  ProfScope prof_(st, KC_MGS);
  const int nt = 512;
  const int g = grid_for(n, nt) > 2 * num_sms(0) ? 2 * num_sms(0) : grid_for(n, nt);
  if (checked)
    k_fx_red<true><<<g, nt, 0, st>>>(n, mode, v, w, b1, b2, acc, abs_out, cnt);
  else
    k_fx_red<false><<<g, nt, 0, st>>>(n, mode, v, w, b1, b2, acc, abs_out, cnt);
  LAUNCH_CHECK();
}

void launch_axpy_only(cudaStream_t st, long long n, i64* w, i64 h, const i64* v, int f, int b1,
                      u64* cnt, bool checked) {
  ProfScope prof_(st, KC_MGS);
  const int nt = 512;
  const int g = grid_for(n, nt);
  if (checked)
    k_axpy<true><<<g, nt, 0, st>>>(n, w, h, v, f, b1, cnt);
  else
    k_axpy<false><<<g, nt, 0, st>>>(n, w, h, v, f, b1, cnt);
  LAUNCH_CHECK();
}

void launch_vec_div(cudaStream_t st, long long n, const i64* w, i64* out, int f, ShiftsD sh,
                    u64* cnt, const Ctl* ctl, bool checked) {
  ProfScope prof_(st, KC_VEC_DIV);
  const int nt = 512;
  const int g = grid_for(n, nt);
  if (checked)
    k_vec_div<true><<<g, nt, 0, st>>>(n, w, out, f, sh.div_b1, sh.div_b2, cnt, ctl);
  else
    k_vec_div<false><<<g, nt, 0, st>>>(n, w, out, f, sh.div_b1, sh.div_b2, cnt, ctl);
  LAUNCH_CHECK();
}

void launch_step_scalar(cudaStream_t st, int j, int f, ShiftsD sh, const u64* acc_col,
                        const u64* abs_col, const u64* nacc, const u64* nabs, i64* hess, int ld,
                        i64* g, i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step, Ctl* ctl,
                        bool checked) {
  ProfScope prof_(st, KC_SCALAR);
  k_step_scalar<<<1, 1, 0, st>>>(j, f, sh, acc_col, abs_col, nacc, nabs, hess, ld, g, cs, sn, gabs,
                                 w, cnt_step, ctl, checked ? 1 : 0);
  LAUNCH_CHECK();
}

void launch_cycle_init(cudaStream_t st, Ctl* ctl, i64* g, int f) {
  ProfScope prof_(st, KC_OTHER);
  k_cycle_init<<<1, 1, 0, st>>>(ctl, g, f);
  LAUNCH_CHECK();
}

void launch_cycle_finish(cudaStream_t st, int m, int f, const i64* hess, const i64* g, double* y,
                         double* wts, Ctl* ctl) {
  ProfScope prof_(st, KC_OTHER);
  k_cycle_finish<<<1, 1, 0, st>>>(m, f, hess, g, y, wts, ctl);
  LAUNCH_CHECK();
}

void launch_xupdate(cudaStream_t st, long long n, int m, int f, const i64* basis,
                    const double* wts, const double* x0, double* x, const Ctl* ctl, int mode) {
  ProfScope prof_(st, KC_XUPDATE);
  (void)m;
  k_xupdate<<<grid_for(n, 256), 256, 0, st>>>(n, f, basis, wts, x0, x, ctl, mode);
  LAUNCH_CHECK();
}

template <typename T, bool B, bool CK, int D>
static void tri_launch_one(cudaStream_t st, const DevTri& t, const T* y, T* out, u64* cnt,
                           const Ctl* ctl, const double* prescale) {
  constexpr size_t kBudget = 227 * 1024 - 256;  // static smem (tile id, caches) excluded
  int seg_cap = t.max_tile_segs + 2;
  static const int env_L = [] {
    const char* e = std::getenv("IGM_TRI_L");
    return e ? std::atoi(e) : 0;
  }();
  int L = env_L > 0 ? env_L : 8;
  TriSmem lay = tri_smem_layout<T, D>(t.tile_cap, seg_cap, L, t.max_seg_ext);
  while (L > 1 && lay.total > kBudget) lay = tri_smem_layout<T, D>(t.tile_cap, seg_cap, --L, t.max_seg_ext);
  if (lay.total > kBudget) {  // segment tables stay in global memory
    seg_cap = 0;
    L = env_L > 0 ? env_L : 8;
    lay = tri_smem_layout<T, D>(t.tile_cap, seg_cap, L, t.max_seg_ext);
    while (L > 1 && lay.total > kBudget) lay = tri_smem_layout<T, D>(t.tile_cap, seg_cap, --L, t.max_seg_ext);
  }
  const size_t sm = lay.total;
  static const int env_sync = [] {
    const char* e = std::getenv("IGM_TRI_SYNC_LOADER");
    const int v = e ? std::atoi(e) : 0;
    tri_loader_mode(v);
    return v;
  }();
  (void)env_sync;
  static size_t done = 0;
  if (sm > done) {
    cudaFuncSetAttribute(k_tri<T, B, CK, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    done = sm;
  }
  TriArgs args = tri_args(t);
  args.epoch = ++const_cast<DevTri&>(t).epoch;  // unique tag per launch
  k_tri<T, B, CK, D><<<t.ntiles, kTriThreads, sm, st>>>(args, y, out, cnt, ctl, prescale, seg_cap, L);
}

template <typename T, bool B, bool CK>
static void tri_dispatch(cudaStream_t st, const DevTri& t, const T* y, T* out, u64* cnt,
                         const Ctl* ctl, const double* prescale) {
  if (t.stride == 4) tri_launch_one<T, B, CK, 4>(st, t, y, out, cnt, ctl, prescale);
  else if (t.stride == 8) tri_launch_one<T, B, CK, 8>(st, t, y, out, cnt, ctl, prescale);
  else tri_launch_one<T, B, CK, 16>(st, t, y, out, cnt, ctl, prescale);
}

void tri_loader_mode(int sync_loader) {
  cudaMemcpyToSymbol(g_tri_sync_loader, &sync_loader, sizeof(int));
}

void tri_trace_setup(int tile, unsigned long long* buf) {
  cudaMemcpyToSymbol(g_tri_ts, &buf, sizeof(buf));
  cudaMemcpyToSymbol(g_tri_ts_tile, &tile, sizeof(int));
}

void launch_tri_int(cudaStream_t st, const DevTri& t, bool backward, const i64* y, i64* out,
                    u64* cnt, const Ctl* ctl, bool checked) {
  if (t.n == 0) return;
  cudaMemsetAsync(t.ticket, 0, sizeof(int), st);
  {
    ProfScope prof_(st, KC_TRI_INT);
    if (backward) tri_dispatch<i64, true, false>(st, t, y, out, cnt, ctl, nullptr);
    else tri_dispatch<i64, false, false>(st, t, y, out, cnt, ctl, nullptr);
  }
  LAUNCH_CHECK();
  if (checked) {
    ProfScope prof_(st, KC_OTHER);
    k_tri_count<<<grid_for(t.n, 256), 256, 0, st>>>(t.n, t.c_rp, t.c_ci, t.c_val, t.c_diag, y, out, cnt, ctl);
    LAUNCH_CHECK();
  }
}

void launch_tri_fp(cudaStream_t st, const DevTri& t, bool backward, const double* y, double* out,
                   const Ctl* ctl, const double* prescale) {
  if (t.n == 0) return;
  cudaMemsetAsync(t.ticket, 0, sizeof(int), st);
  ProfScope prof_(st, KC_TRI_FP);
  if (backward) tri_dispatch<double, true, false>(st, t, y, out, nullptr, ctl, prescale);
  else tri_dispatch<double, false, false>(st, t, y, out, nullptr, ctl, prescale);
  LAUNCH_CHECK();
}

}  // namespace igm
