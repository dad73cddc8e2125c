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
#include "tri_pencil.cuh"
#include "tri_pencil2.cuh"
#include "pencil27.cuh"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <random>
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

// one thread per element (latency-bound per-row kernels: every row's chain
// of dependent loads in flight at once)
inline int grid_full(long long n, int nt) {
  const long long g = (n + nt - 1) / nt;
  return static_cast<int>(g < 1 ? 1 : (g > 0x7fffffffLL ? 0x7fffffffLL : g));
}

inline int grid_for(long long n, int nt, int device = -1) {
  long long g = (n + nt - 1) / nt;
  const long long cap = static_cast<long long>(num_sms(device < 0 ? cur_device() : device)) * 8;
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

// K1, short rows (<= 8 entries: 7-point stencils), split depth 0: one thread
// per row as above, but the row's (value, column) pairs are all loaded before
// the first gather and the gathers before the first product, so a thread
// keeps up to 24 loads in flight instead of 2-3 (the loop above is a chain
// of dependent loads per entry: ncu shows long-scoreboard stalls at DRAM
// traffic equal to the algorithmic bytes).  Sums stay in CSR order.
// R = 8 (7-point stencils) or 16 (config 3's band + 10 random columns: the
// random gathers make the dependent-load chain of the generic kernel twice as
// costly there)
template <bool CHECKED, int R = 8>
__global__ void __launch_bounds__(128) k_spmv_int_r8(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                     const i64* __restrict__ vals, int alpha0,
                                                     const i64* __restrict__ v, i64* __restrict__ out, u64* cnt,
                                                     const Ctl* ctl, u64 amax, const u64* __restrict__ vb) {
  if (cycle_over(ctl)) return;
  // |v| <= V: the maximum the Arnoldi kernel recorded while writing v (one
  // word, loaded with the row's other operands)
  const u64 V = (CHECKED && vb != nullptr) ? static_cast<u64>(__ldcg(reinterpret_cast<const unsigned long long*>(vb)))
                                           : ~0ull;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = row < n;
  const int b = live ? rp[row] : 0, len = live ? rp[row + 1] - b : 0;
  int c[R];
  i64 a[R], x[R];
#pragma unroll
  for (int u = 0; u < R; ++u) {
    c[u] = u < len ? ci[b + u] : 0;
    a[u] = u < len ? vals[b + u] : 0;
  }
#pragma unroll
  for (int u = 0; u < R; ++u) x[u] = u < len ? __ldg(v + c[u]) : 0;
  // magnitude certificate: with |a| <= amax, R * amax * V < 2^63 rules out
  // every product and running-sum overflow of a row of <= R entries -- the
  // exact event count is zero and the per-product tests are skipped
  const bool safe = CHECKED && vb != nullptr && __umul64hi(amax, V) == 0 && amax * V < (1ull << 63) / R;
  u64 nmul = 0, nadd = 0;
  i64 acc = 0;
  if (!CHECKED || safe) {
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (u < len) acc = wadd(acc, wmul(a[u], x[u]));
  } else {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (u < len) {
        const i64 p = wmul(a[u], x[u]);
        nmul += mul_ovf(a[u], x[u]);
        nadd += add_ovf(acc, p);
        acc = wadd(acc, p);
      }
    }
  }
  if (live) out[row] = asr(acc, alpha0);
  if (CHECKED && !safe) {
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_ADD, nadd);
  }
}

__global__ void __launch_bounds__(256) k_max_abs(long long n, const i64* __restrict__ a, unsigned long long* out) {
  u64 m = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const i64 x = a[i];
    const u64 ax = x < 0 ? u64{0} - static_cast<u64>(x) : static_cast<u64>(x);
    m = ax > m ? ax : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, static_cast<u64>(__shfl_down_sync(0xffffffffu, m, o)));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, static_cast<unsigned long long>(m));
}

// K1, staged variant for long rows (27-point stencils: 324 B per row).  One
// thread per row makes a warp touch 32 distant row segments per load, which
// the L1 cannot hold until they are consumed (config 4: 0.45 of HBM).  Here a
// warp owns a tile of 32 consecutive rows = one contiguous run of entries:
// it loads the run's (value, column) pairs coalesced, multiplies, parks the
// products in shared memory, and every lane then sums ITS row's products in
// CSR order -- the reference's per-row order (split.cpp:137-157), so the
// add-overflow events are the reference's too (wrapping sums are order-free,
// the events are not).
constexpr int kSpRows = 32, kSpMaxRow = 32, kSpWarps = 4;
template <bool CHECKED>
__global__ void __launch_bounds__(kSpWarps * 32) k_spmv_int_staged(int n, const int* __restrict__ rp,
                                                                   const int* __restrict__ ci,
                                                                   const i64* __restrict__ vals, long long nnz,
                                                                   const int* __restrict__ alphas, int s,
                                                                   const i64* __restrict__ v, i64* __restrict__ out,
                                                                   u64* cnt, const Ctl* ctl) {
  __shared__ i64 sm[kSpWarps][kSpRows * kSpMaxRow];
  if (cycle_over(ctl)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  i64* prod = sm[w];
  u64 nmul = 0, nadd = 0;
  const int ntiles = (n + kSpRows - 1) / kSpRows;
  for (int tile = blockIdx.x * kSpWarps + w; tile < ntiles; tile += gridDim.x * kSpWarps) {
    const int row = tile * kSpRows + lane;
    const bool live = row < n;
    const int b = live ? rp[row] : 0, e = live ? rp[row + 1] : 0;
    const int tb = __shfl_sync(0xffffffffu, b, 0);
    const int te = __shfl_sync(0xffffffffu, e, min(kSpRows - 1, n - 1 - tile * kSpRows));
    i64 o = 0;
    for (int l = 0; l <= s; ++l) {
      const i64* cv = vals + static_cast<long long>(l) * nnz;
#pragma unroll 4
      for (int k = tb + lane; k < te; k += 32) {
        // the matrix streams through once: keep it out of the L1 lines the
        // gathered vector entries (reused ~27 times) live in
        const i64 a = __ldcs(cv + k);
        const i64 x = __ldg(v + __ldcs(ci + k));
        if (CHECKED) nmul += mul_ovf(a, x);
        prod[k - tb] = wmul(a, x);
      }
      __syncwarp();
      i64 acc = 0;
      for (int k = b; k < e; ++k) {
        const i64 p = prod[k - tb];
        if (CHECKED) nadd += add_ovf(acc, p);
        acc = wadd(acc, p);
      }
      const i64 d = asr(acc, alphas[l]);
      if (CHECKED) nadd += add_ovf(o, d);
      o = wadd(o, d);
      __syncwarp();
    }
    if (live) out[row] = o;
  }
  if (CHECKED) {
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_ADD, nadd);
  }
}

// K1 for long rows (17..32 entries: 27-point stencils), depth 0: sliced ELL.
// Component 0 is kept a second time in 32-row slices, slot-major (slot u of
// the slice's 32 rows is one contiguous run; rows shorter than the width are
// padded with value 0 / column 0), so with one thread per row every matrix
// load is one coalesced 256-byte (values) / 128-byte (columns) access AND
// slot u of 32 consecutive rows gathers 32 consecutive vector words; the loads
// of 9 slots are issued before their products.  Slot order is CSR order: the
// running sums and their overflow events are the reference's
// (split.cpp:137-157).  CSR keeps a 27-point warp at 32 distant row segments
// per load (L1-wavefront bound, 0.44 of HBM); the staged kernel above pays
// ~11 sectors per gather.
template <bool CHECKED>
__global__ void __launch_bounds__(128) k_spmv_int_sell(int n, int w, const i64* __restrict__ sv,
                                                       const int* __restrict__ sc, int alpha0,
                                                       const i64* __restrict__ v, i64* __restrict__ out, u64* cnt,
                                                       const Ctl* ctl, u64 amax, const u64* __restrict__ vb) {
  if (cycle_over(ctl)) return;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= ((n + 31) & ~31)) return;  // past the last (zero-padded) slice
  const u64 V = (CHECKED && vb != nullptr) ? static_cast<u64>(__ldcg(reinterpret_cast<const unsigned long long*>(vb)))
                                           : ~0ull;
  const size_t base = static_cast<size_t>(row >> 5) * w * 32 + (row & 31);
  // magnitude certificate as in k_spmv_int_r8, for rows of <= 32 entries
  const bool safe = CHECKED && vb != nullptr && __umul64hi(amax, V) == 0 && amax * V < (1ull << 58);
  u64 nmul = 0, nadd = 0;
  i64 acc = 0;
  constexpr int B = 9;
  for (int u0 = 0; u0 < w; u0 += B) {
    i64 a[B], x[B];
    int c[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const bool ok = u0 + q < w;
      a[q] = ok ? __ldcs(sv + base + static_cast<size_t>(u0 + q) * 32) : 0;
      c[q] = ok ? __ldcs(sc + base + static_cast<size_t>(u0 + q) * 32) : 0;
    }
#pragma unroll
    for (int q = 0; q < B; ++q) x[q] = __ldg(v + c[q]);
#pragma unroll
    for (int q = 0; q < B; ++q) {
      if (u0 + q < w) {
        const i64 p = wmul(a[q], x[q]);
        if (CHECKED && !safe) {
          nmul += mul_ovf(a[q], x[q]);
          nadd += add_ovf(acc, p);
        }
        acc = wadd(acc, p);
      }
    }
  }
  if (row < n) out[row] = asr(acc, alpha0);
  if (CHECKED && !safe) {
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_ADD, nadd);
  }
}

__global__ void __launch_bounds__(128) k_build_sell(int n, int w, const int* __restrict__ rp,
                                                    const int* __restrict__ ci, const i64* __restrict__ vals,
                                                    i64* __restrict__ sv, int* __restrict__ sc) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int b = rp[row], len = rp[row + 1] - b;
  const size_t base = static_cast<size_t>(row >> 5) * w * 32 + (row & 31);
  for (int u = 0; u < len && u < w; ++u) {
    sv[base + static_cast<size_t>(u) * 32] = vals[b + u];
    sc[base + static_cast<size_t>(u) * 32] = ci[b + u];
  }
}

__global__ void __launch_bounds__(256) k_max_row(int n, const int* __restrict__ rp, int* out) {
  int m = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) m = max(m, rp[r + 1] - rp[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
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
//       basis words first: collect_basis_norms); 5 -> *out = the running sum
//       (no sqrt: one rank's leg of a chain relayed across a row partition).
// start (device, may be null): the chain's starting value.
constexpr int kNormTile = 2048;

__global__ void __launch_bounds__(256) k_norm2_serial(long long n, const double* __restrict__ v,
                                                      const i64* __restrict__ raw, double scale,
                                                      double* out, Ctl* ctl, int mode,
                                                      int basis_idx, const double* start) {
  __shared__ double buf[2][kNormTile];
  if (mode == 3 && cycle_over(ctl)) return;
  if (mode == 4 && (ctl->err || basis_idx >= ctl->nbasis)) return;
  double acc = start ? *start : 0.0;
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
      case 5: *out = acc; break;
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

// shared state of the exact chain inside one CTA
struct N2State {
  Aut warp[32];
  int exit_at;
  u64 mprev;
  int E;          // binade of the running sum: s = M * 2^(E-52)
  u64 M;
  long long pos;  // next term
  int tail;       // the sum became non-finite at pos-1: finish serially
  double tailv;
  int win;        // terms the next pass of n2_advance looks at (adaptive)
  long long last_exit;  // position of the last term that left its binade
};

__device__ __forceinline__ double n2_term(long long i, const double* __restrict__ v, const i64* __restrict__ raw,
                                          double scale) {
  const double x = raw ? dec(raw[i], scale) : v[i];
  return __dmul_rn(x, x);
}

// Advance the exact chain from S.pos to hi (one CTA of kN2Threads threads):
// chunks of kN2Chunk terms are classified against the current binade, scanned
// as 2-state automata, and the first term that would leave the binade is
// replayed with the real FP64 add.
__device__ void n2_advance(long long hi, const double* __restrict__ v, const i64* __restrict__ raw, double scale,
                           N2State& S) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  while (true) {
    const long long pos = S.pos;
    const int E = S.E;
    const u64 M0 = S.M;
    if (pos >= hi || S.tail) break;
    // Adaptive window: a pass costs the whole CTA ~9 us when all 8192 terms
    // are classified and scanned, and the passes right after a binade exit
    // usually end a few terms later (a sum that starts at 0 leaves a binade
    // after 1, 2, 4, ... terms).  So a pass after an exit looks at 256 terms
    // (one warp's worth) and the window doubles with every pass that ends
    // without an exit; warps outside the window skip the classification.
    const int win = S.win;
    const long long lim = min(hi, pos + win);
    const long long base = pos + static_cast<long long>(tid) * kN2Per;
    u64 a[kN2Per];
    int cls[kN2Per];
    Aut mine{0, 0};
    if (base < lim) {  // (warp-uniform up to the window's last warp)
#pragma unroll
      for (int g = 0; g < kN2Per; ++g) {
        const long long idx = base + g;
        if (idx < lim) {
          cls[g] = n2_classify(n2_term(idx, v, raw, scale), E, a[g]);
        } else {
          cls[g] = N2_DOWN;
          a[g] = 0;
        }
        Aut e;
        e.d0 = n2_inc(a[g], cls[g] == N2_EXIT ? N2_DOWN : cls[g], 0);
        e.d1 = n2_inc(a[g], cls[g] == N2_EXIT ? N2_DOWN : cls[g], 1);
        mine = aut_then(mine, e);
      }
    } else {
#pragma unroll
      for (int g = 0; g < kN2Per; ++g) {
        cls[g] = N2_DOWN;
        a[g] = 0;
      }
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
    if (lane == 31) S.warp[wid] = inc;
    if (tid == 0) S.exit_at = INT_MAX;
    __syncthreads();
    if (wid == 0) {
      Aut w = S.warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        Aut up;
        up.d0 = __shfl_up_sync(0xffffffffu, w.d0, o);
        up.d1 = __shfl_up_sync(0xffffffffu, w.d1, o);
        if (lane >= o) w = aut_then(up, w);
      }
      S.warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    Aut ex{0, 0};
    if (wid > 0) ex = S.warp[wid - 1];
    {
      Aut lx;
      lx.d0 = __shfl_up_sync(0xffffffffu, inc.d0, 1);
      lx.d1 = __shfl_up_sync(0xffffffffu, inc.d1, 1);
      if (lane > 0) ex = aut_then(ex, lx);
    }
    const Aut total = S.warp[31];
    // walk this thread's terms from the true incoming value; first exit
    u64 Mp = M0 + ((M0 & 1) ? ex.d1 : ex.d0);
    int my_exit = INT_MAX;
    u64 my_mprev = 0;
#pragma unroll
    for (int g = 0; g < kN2Per; ++g) {
      if (my_exit != INT_MAX) break;
      const long long idx = base + g;
      if (idx >= lim) break;
      const bool leave = cls[g] == N2_EXIT || a[g] >= kTwo53 ||
                         Mp + a[g] + (cls[g] != N2_DOWN ? 1 : 0) >= kTwo53;
      if (leave) {
        my_exit = tid * kN2Per + g;
        my_mprev = Mp;
      } else {
        Mp += n2_inc(a[g], cls[g], Mp & 1);
      }
    }
    if (my_exit != INT_MAX) atomicMin(&S.exit_at, my_exit);
    __syncthreads();
    const int xe = S.exit_at;
    if (xe != INT_MAX && my_exit == xe) S.mprev = my_mprev;
    __syncthreads();
    if (tid == 0) {
      if (xe == INT_MAX) {
        S.M = M0 + ((M0 & 1) ? total.d1 : total.d0);
        S.pos = lim;
        S.win = min(2 * win, kN2Chunk);
      } else {
        // the next exit tends to be about as far from this one as this one
        // was from the one before (a sum growing from 0 leaves its binade
        // after 1, 2, 4, ... terms; an isolated crossing much later gets the
        // full window back)
        const long long gap = pos + xe - S.last_exit;
        int wn = 256;
        while (wn < 2 * gap && wn < kN2Chunk) wn *= 2;
        S.win = wn;
        S.last_exit = pos + xe;
        // replay the term that leaves the binade with the real FP64 add
        const long long idx = pos + xe;
        const double sp = ldexp(static_cast<double>(S.mprev), E - 52);
        const double sn = __dadd_rn(sp, n2_term(idx, v, raw, scale));
        if (!isfinite(sn)) {
          S.tail = 1;
          S.tailv = sn;
          S.pos = idx + 1;
        } else {
          const u64 b = static_cast<u64>(__double_as_longlong(sn));
          const int ebits = static_cast<int>((b >> 52) & 0x7ff);
          const int En = ebits == 0 ? -1022 : max(ebits - 1023, -1022);
          S.E = En;
          S.M = static_cast<u64>(ldexp(sn, 52 - En));
          S.pos = idx + 1;
        }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ bool n2_skip(const Ctl* ctl, int mode, int basis_idx) {
  return (mode == 3 && cycle_over(ctl)) || (mode == 4 && (ctl->err || basis_idx >= ctl->nbasis));
}

// final value of the chain and its destination (see k_norm2_serial's modes)
__device__ void n2_finish(long long n, const double* __restrict__ v, const i64* __restrict__ raw, double scale,
                          const N2State& S, double* out, Ctl* ctl, int mode, int basis_idx) {
  double acc;
  if (S.tail) {  // non-finite partial sum: finish the chain serially
    acc = S.tailv;
    for (long long i = S.pos; i < n; ++i) acc = __dadd_rn(acc, n2_term(i, v, raw, scale));
  } else {
    acc = ldexp(static_cast<double>(S.M), S.E - 52);
  }
  const double r = __dsqrt_rn(acc);
  switch (mode) {
    case 5: *out = acc; break;  // the running sum itself (a rank's leg of a distributed chain)
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

// s0: the chain's starting value (0, or the running sum handed over by the
// previous rank of a row-block partition); any non-negative double
__device__ __forceinline__ void n2_init(N2State& S, const double* start) {
  S.E = -1022;  // s = 0: subnormal binade, u = 2^-1074
  S.M = 0;
  S.pos = 0;
  S.tail = 0;
  S.win = 256;
  S.last_exit = -1;
  const double s0 = start ? *start : 0.0;
  if (s0 != 0.0) {
    const u64 bits = static_cast<u64>(__double_as_longlong(s0));
    const int ex = static_cast<int>((bits >> 52) & 0x7ff);
    if (ex == 0x7ff || s0 < 0.0) {  // non-finite (or not a sum of squares): serial tail
      S.tail = 1;
      S.tailv = s0;
    } else if (ex == 0) {
      S.M = bits & ((1ull << 52) - 1);
    } else {
      S.E = ex - 1023;
      S.M = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    }
  }
}

// single-CTA exact chain (short vectors)
__global__ void __launch_bounds__(kN2Threads) k_norm2_exact(long long n, const double* __restrict__ v,
                                                            const i64* __restrict__ raw, double scale,
                                                            double* out, Ctl* ctl, int mode,
                                                            int basis_idx, const double* start) {
  __shared__ N2State S;
  if (n2_skip(ctl, mode, basis_idx)) return;
  if (threadIdx.x == 0) n2_init(S, start);
  __syncthreads();
  n2_advance(n, v, raw, scale, S);
  if (threadIdx.x == 0) n2_finish(n, v, raw, scale, S, out, ctl, mode, basis_idx);
}

// Multi-CTA form for long vectors.  A block of kN2Chunk terms can be applied
// in O(1) -- M += d(parity of M) -- when (i) the running sum's binade at the
// block start is the one the block was classified against and (ii) no term
// can leave it: M + max(d0, d1) + 1 < 2^53, no term >= 2^53 ulps, no
// non-finite term.  Pass 1 sums each block's squares (any order: only a
// guess), pass 2 guesses each block's starting binade from the approximate
// prefix and reduces the block's automaton against it, pass 3 (one CTA) walks
// the blocks in order: O(1) per block when (i)-(ii) hold, otherwise the
// block is replayed exactly (n2_advance) from the true state.  Replays happen
// only around binade crossings (~log2 n of them, mostly in the first block).
struct N2Blk {
  double s;   // approximate sum of the block's squares
  int E;      // binade the automaton was built against
  int bad;    // a term >= 2^53 ulps or non-finite: always replay
  u64 d0, d1;
};

constexpr int kN2BThreads = 512;
constexpr int kN2BPer = kN2Chunk / kN2BThreads;

__global__ void __launch_bounds__(kN2BThreads) k_n2_bsum(long long n, const double* __restrict__ v,
                                                         const i64* __restrict__ raw, double scale, N2Blk* blk,
                                                         const Ctl* ctl, int mode, int basis_idx) {
  __shared__ double sh[kN2BThreads / 32];
  if (n2_skip(ctl, mode, basis_idx)) return;
  const long long lo = static_cast<long long>(blockIdx.x) * kN2Chunk;
  const long long hi = min(n, lo + kN2Chunk);
  double acc = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += kN2BThreads) acc += n2_term(i, v, raw, scale);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kN2BThreads / 32; ++w) t += sh[w];
    blk[blockIdx.x].s = t;
  }
}

__global__ void __launch_bounds__(kN2BThreads) k_n2_baut(long long n, const double* __restrict__ v,
                                                         const i64* __restrict__ raw, double scale, N2Blk* blk,
                                                         const Ctl* ctl, int mode, int basis_idx,
                                                         const double* start) {
  __shared__ double shs[kN2BThreads / 32];
  __shared__ Aut sha[kN2BThreads / 32];
  __shared__ int sbad;
  __shared__ int sE;
  if (n2_skip(ctl, mode, basis_idx)) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // approximate prefix of the earlier blocks -> guessed starting binade
  double p = 0.0;
  for (int b = tid; b < static_cast<int>(blockIdx.x); b += kN2BThreads) p += blk[b].s;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p += __shfl_down_sync(0xffffffffu, p, o);
  if (lane == 0) shs[wid] = p;
  if (tid == 0) sbad = 0;
  __syncthreads();
  if (tid == 0) {
    double t = start ? *start : 0.0;
    for (int w = 0; w < kN2BThreads / 32; ++w) t += shs[w];
    int E = -1022;
    if (t > 0.0 && isfinite(t)) {
      const int eb = static_cast<int>((static_cast<u64>(__double_as_longlong(t)) >> 52) & 0x7ff);
      E = eb == 0 ? -1022 : max(eb - 1023, -1022);
    }
    sE = E;
  }
  __syncthreads();
  const int E = sE;
  // this thread's consecutive run, composed in order
  const long long lo = static_cast<long long>(blockIdx.x) * kN2Chunk + static_cast<long long>(tid) * kN2BPer;
  Aut mine{0, 0};
  int bad = 0;
#pragma unroll 4
  for (int g = 0; g < kN2BPer; ++g) {
    const long long idx = lo + g;
    if (idx >= n) break;
    u64 aa;
    const int c = n2_classify(n2_term(idx, v, raw, scale), E, aa);
    if (c == N2_EXIT || aa >= kTwo53) bad = 1;
    Aut e;
    e.d0 = n2_inc(aa, c == N2_EXIT ? N2_DOWN : c, 0);
    e.d1 = n2_inc(aa, c == N2_EXIT ? N2_DOWN : c, 1);
    mine = aut_then(mine, e);
  }
  // ordered reduction: warp (lane order), then warps (warp order)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Aut up;
    up.d0 = __shfl_down_sync(0xffffffffu, mine.d0, o);
    up.d1 = __shfl_down_sync(0xffffffffu, mine.d1, o);
    if ((lane & (2 * o - 1)) == 0 && lane + o < 32) mine = aut_then(mine, up);
  }
  if (lane == 0) sha[wid] = mine;
  if (bad) sbad = 1;
  __syncthreads();
  if (tid == 0) {
    Aut t = sha[0];
    for (int w = 1; w < kN2BThreads / 32; ++w) t = aut_then(t, sha[w]);
    N2Blk& B = blk[blockIdx.x];
    B.E = E;
    B.bad = sbad;
    B.d0 = t.d0;
    B.d1 = t.d1;
  }
}

__global__ void __launch_bounds__(kN2Threads) k_n2_walk(long long n, int nblk, const double* __restrict__ v,
                                                        const i64* __restrict__ raw, double scale,
                                                        const N2Blk* blk, double* out, Ctl* ctl, int mode,
                                                        int basis_idx, const double* start) {
  constexpr int kPage = 512;
  __shared__ N2State S;
  __shared__ N2Blk page[kPage];
  __shared__ int s_fast;
  if (n2_skip(ctl, mode, basis_idx)) return;
  if (threadIdx.x == 0) n2_init(S, start);
  for (int p0 = 0; p0 < nblk; p0 += kPage) {
    const int np = min(kPage, nblk - p0);
    __syncthreads();
    for (int i = threadIdx.x; i < np; i += blockDim.x) page[i] = blk[p0 + i];
    __syncthreads();
    int b = 0;
    while (b < np) {
      if (threadIdx.x == 0) {
        // O(1) blocks, sequentially, until one needs an exact replay
        while (b < np && !S.tail) {
          const N2Blk& B = page[b];
          const u64 dm = B.d0 > B.d1 ? B.d0 : B.d1;
          if (B.bad || B.E != S.E || S.M + dm + 1 >= kTwo53) break;
          S.M += (S.M & 1) ? B.d1 : B.d0;
          ++b;
        }
        S.pos = min(n, static_cast<long long>(p0 + b) * kN2Chunk);
        s_fast = b;
      }
      __syncthreads();
      b = s_fast;
      if (b >= np || S.tail) break;
      if (threadIdx.x == 0) S.win = kN2Chunk;  // a later block: one exit at most is the rule
      __syncthreads();
      n2_advance(min(n, static_cast<long long>(p0 + b + 1) * kN2Chunk), v, raw, scale, S);  // replay block b
      ++b;
    }
    if (S.tail) break;
  }
  __syncthreads();
  if (threadIdx.x == 0) n2_finish(n, v, raw, scale, S, out, ctl, mode, basis_idx);
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
                                                 u64* cnt, const Ctl* ctl, u64* vmax_out) {
  if (!ctl->do_vecdiv) return;
  SDivMagic g;
  g.u.m = ctl->div_m;
  g.u.sh1 = ctl->div_sh1;
  g.u.sh2 = ctl->div_sh2;
  g.den_neg = ctl->div_neg;
  g.den_is_m1 = ctl->div_m1;
  const int e = f - b1 - b2;
  u64 nshl = 0, ndiv = 0, vmax = 0;
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
      const u64 ar = r < 0 ? u64{0} - static_cast<u64>(r) : static_cast<u64>(r);
      vmax = ar > vmax ? ar : vmax;
    }
    out[l] = r;
  }
  if (CHECKED) {
    bump(cnt, OP_SHL, nshl);
    bump(cnt, OP_DIV, ndiv);
    // max |v_{j+1}| over all rows: the next SpMV's magnitude certificate
    if (vmax_out != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const u64 t = __shfl_down_sync(0xffffffffu, vmax, o);
        vmax = t > vmax ? t : vmax;
      }
      if ((threadIdx.x & 31) == 0 && vmax)
        atomicMax(reinterpret_cast<unsigned long long*>(vmax_out), static_cast<unsigned long long>(vmax));
    }
  }
}


// ---------------------------------------------------------------------------
// Exact running-sum ("add") overflow events of one fx_dot / fx_norm
// reduction.  The reference adds the
// wrapped int64 terms t_l sequentially, acc <- acc + t_l, and records an
// event whenever the exact sum leaves int64.  With P_l the exact (int128)
// prefix sum, acc_l = wrap(P_l) and the event at l happens iff
// floor((P_{l+1} + 2^63) / 2^64) != floor((P_l + 2^63) / 2^64).  Pass 1 sums
// each chunk exactly, pass 2 scans the chunk sums in order, pass 3 walks
// every chunk from its exact start and counts the crossings.  All three
// passes return at once when the pass kernel's certificate (sum |t| < 2^63,
// cert = {hi, lo} 32-bit halves) already proves zero events.
constexpr int kAddChunk = 8192;
constexpr int kAddThreads = 512;
constexpr int kAddPer = kAddChunk / kAddThreads;

__device__ __forceinline__ i64 add_term(int mode, const i64* __restrict__ w, const i64* __restrict__ v,
                                        long long l, int b1, int b2) {
  const i64 a = asr(w[l], b1);
  return wmul(a, mode == 0 ? asr(v[l], b2) : a);
}
__device__ __forceinline__ bool adds_certified(const u64* cert, const Ctl* ctl) {
  if (ctl && cycle_over(ctl)) return true;
  const unsigned __int128 s = (static_cast<unsigned __int128>(cert[0]) << 32) + cert[1];
  return s < (static_cast<unsigned __int128>(1) << 63);
}
__device__ __forceinline__ long long wrap_index(__int128 p) {
  return static_cast<long long>((p + (static_cast<__int128>(1) << 63)) >> 64);
}

__global__ void __launch_bounds__(kAddThreads) k_adds_blk(long long n, int mode, const i64* __restrict__ w,
                                                          const i64* __restrict__ v, int b1, int b2,
                                                          const u64* cert, const Ctl* ctl, __int128* blk) {
  __shared__ __int128 sh[kAddThreads / 32];
  if (adds_certified(cert, ctl)) return;
  const long long lo = static_cast<long long>(blockIdx.x) * kAddChunk;
  const long long hi = min(n, lo + kAddChunk);
  __int128 acc = 0;
  for (long long l = lo + threadIdx.x; l < hi; l += kAddThreads) acc += add_term(mode, w, v, l, b1, b2);
  // exact: any order
  for (int o = 16; o > 0; o >>= 1) {
    const u64 a = __shfl_down_sync(0xffffffffu, static_cast<u64>(acc), o);
    const u64 b = __shfl_down_sync(0xffffffffu, static_cast<u64>(static_cast<unsigned __int128>(acc) >> 64), o);
    acc += static_cast<__int128>((static_cast<unsigned __int128>(b) << 64) | a);
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    __int128 t = 0;
    for (int i = 0; i < kAddThreads / 32; ++i) t += sh[i];
    blk[blockIdx.x] = t;
  }
}

__global__ void k_adds_scan(int nblk, const u64* cert, const Ctl* ctl, __int128* blk) {
  if (adds_certified(cert, ctl)) return;
  if (threadIdx.x != 0) return;
  __int128 p = 0;
  for (int b = 0; b < nblk; ++b) {
    const __int128 t = blk[b];
    blk[b] = p;
    p += t;
  }
}

__global__ void __launch_bounds__(kAddThreads) k_adds_count(long long n, int mode, const i64* __restrict__ w,
                                                            const i64* __restrict__ v, int b1, int b2,
                                                            const u64* cert, const Ctl* ctl,
                                                            const __int128* pre, u64* cnt_add) {
  __shared__ __int128 sh[kAddThreads];
  if (adds_certified(cert, ctl)) return;
  const long long lo = static_cast<long long>(blockIdx.x) * kAddChunk + static_cast<long long>(threadIdx.x) * kAddPer;
  const long long hi = min(n, lo + kAddPer);
  __int128 s = 0;
  for (long long l = lo; l < hi; ++l) s += add_term(mode, w, v, l, b1, b2);
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan in element order
    __int128 p = pre[blockIdx.x];
    for (int i = 0; i < kAddThreads; ++i) {
      const __int128 t = sh[i];
      sh[i] = p;
      p += t;
    }
  }
  __syncthreads();
  __int128 p = sh[threadIdx.x];
  long long wi = wrap_index(p);
  unsigned long long ev = 0;
  for (long long l = lo; l < hi; ++l) {
    p += add_term(mode, w, v, l, b1, b2);
    const long long wn = wrap_index(p);
    ev += wn != wi;
    wi = wn;
  }
  for (int o = 16; o > 0; o >>= 1) ev += __shfl_down_sync(0xffffffffu, ev, o);
  if ((threadIdx.x & 31) == 0 && ev) atomicAdd(reinterpret_cast<unsigned long long*>(cnt_add), ev);
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

// The scalar step runs once per launch, cold in the instruction cache: its
// time is set by its code size, so the helpers it calls more than once are
// out-of-line (one copy, warm at the second call).
__device__ __noinline__ u64 isqrt_nl(u64 v) { return isqrt_u64(v); }
__device__ __noinline__ i64 sdiv_trunc_nl(i64 a, i64 b) { return sdiv_trunc(a, b); }
__device__ __noinline__ SDivMagic make_sdiv_nl(i64 d) { return make_sdiv(d); }

__device__ __noinline__ i64 d_fx_mul(i64 a, i64 b, int f, int b1, int b2, int of, Ev& ev, int k) {
  const i64 x = asr(a, b1), y = asr(b, b2);
  if (mul_ovf(x, y)) ev.hit(k, OP_MUL);
  return asr(wmul(x, y), 2 * f - b1 - b2 - of);
}

// returns false on a zero shifted divisor (domain_error)
__device__ __noinline__ bool d_fx_div(i64 a, i64 b, int f, int b1, int b2, i64* out, Ev& ev, int k) {
  const i64 num = wrap_shl(a, b1);
  if (shl_ovf(a, b1)) ev.hit(k, OP_SHL);
  const i64 den = asr(b, b2);
  if (den == 0) return false;
  i64 q;
  if (num == INT64_MIN && den == -1) {
    ev.hit(k, OP_DIV);
    q = num;
  } else {
    q = sdiv_trunc_nl(num, den);
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

// acc_col[i * acc_st] / abs_col[i * abs_st .. +1]: pass i's wrapped
// accumulator and sum|term| (hi, lo); norm_mul: the norm pass's square-overflow
// count (cnt_step's own slot on one GPU, the all-reduced one on a partition).
__device__ void step_scalar_dev(int j, int f, ShiftsD sh, const u64* acc_col, int acc_st, const u64* abs_col,
                                int abs_st, const u64* nacc, const u64* nabs, const u64* norm_mul, i64* hess,
                                int ld, i64* g, i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step,
                                Ctl* ctl, int checked, unsigned long long* ts = nullptr) {
#define SS_TS(k) \
  if (ts != nullptr) ts[100 + (k)] = clock64();
  SS_TS(0)
  ctl->do_vecdiv = 0;
  if (cycle_over(ctl)) return;
  SS_TS(1)
  Ev ev{cnt_step, checked != 0};
  i64* col = hess + static_cast<long long>(j) * ld;
  // h_ij = fx_dot finalisation (fxp.cpp:63-65)
  const int e = f - sh.dot_b1 - sh.dot_b2;
  for (int i = 0; i <= j; ++i) {
    const i64 acc = static_cast<i64>(acc_col[i * acc_st]);
    if (e >= 0) {
      col[i] = asr(acc, e);
    } else {
      if (shl_ovf(acc, -e)) ev.hit(K_DOT, OP_SHL);
      col[i] = wrap_shl(acc, -e);
    }
    if (checked == 1 && !abs_small(abs_col + i * abs_st)) ctl->add_inexact = 1;
  }
  SS_TS(2)
  // h_{j+1,j} = fx_norm(w) (fxp.cpp:69-86)
  const i64 nsum = static_cast<i64>(*nacc);
  if (checked == 1) {  // (checked == 2: the norm's add events were counted exactly by k_adds_*)
    // all terms s*s are >= 0 unless a square itself wrapped: then the
    // running sum is monotone and its wrap count is exact.
    if (*norm_mul == 0) {
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
  SS_TS(3)
  i64 hnext;
  {
    const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(nsum)));
    const int es = sh.norm_b1;  // out_frac - fin/2 = f - (f - b1)
    if (shl_ovf(r, es)) ev.hit(K_NORM, OP_SHL);
    hnext = wrap_shl(r, es);
  }
  SS_TS(4)
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
  SS_TS(5)
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
  SS_TS(6)
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
  SS_TS(7)
  i64 c, s;
  if (!d_fx_div(col[j], tmp, f, sh.div_b1, sh.div_b2, &c, ev, K_GIVENS_DIV) ||
      !d_fx_div(col[j + 1], tmp, f, sh.div_b1, sh.div_b2, &s, ev, K_GIVENS_DIV)) {
    set_err(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
    return;
  }
  SS_TS(8)
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
  SS_TS(9)
#undef SS_TS
}

// step_scalar_dev on one warp (same values, same overflow-event totals): the
// h_ij finalisations and the chain-independent products of the stored
// rotations run across the lanes; the rotation chain itself,
//   x_0 = h_0j,  x_{i+1} = c_i * h_{i+1,j} - s_i * x_i   (d_fx_mul, wsub),
// runs on every lane at once (redundantly: no broadcast), after which lane i
// forms rotation i's outputs (h_ij = c_i x_i + s_i h_{i+1,j}, h_{i+1,j} =
// x_{i+1}) and counts its events.  The norm, t_mp, (c, s) and g updates stay
// on lane 0.  All 32 lanes of the calling warp must call it.
__device__ void step_scalar_warp(int j, int f, ShiftsD sh, const u64* acc_col, int acc_st, const u64* abs_col,
                                 int abs_st, const u64* nacc, const u64* nabs, const u64* norm_mul, i64* hess,
                                 int ld, i64* g, i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step,
                                 Ctl* ctl, int checked, unsigned long long* ts = nullptr) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
#define SW_TS(k) \
  if (ts != nullptr && lane == 0) ts[100 + (k)] = clock64();
  SW_TS(0)
  int over = 0;
  i64 g_old = 0;
  if (lane == 0) {
    ctl->do_vecdiv = 0;
    over = cycle_over(ctl);
    g_old = g[j];
  }
  if (__shfl_sync(FULL, over, 0)) return;
  SW_TS(1)
  Ev ev{cnt_step, checked != 0};
  const bool on = checked != 0;
  i64* col = hess + static_cast<long long>(j) * ld;
  // h_ij = fx_dot finalisation (fxp.cpp:63-65), one entry per lane
  {
    const int e = f - sh.dot_b1 - sh.dot_b2;
    unsigned nshl = 0;
    int inexact = 0;
    for (int i = lane; i <= j; i += 32) {
      const i64 acc = static_cast<i64>(acc_col[i * acc_st]);
      if (e >= 0) {
        col[i] = asr(acc, e);
      } else {
        nshl += shl_ovf(acc, -e);
        col[i] = wrap_shl(acc, -e);
      }
      if (checked == 1 && !abs_small(abs_col + i * abs_st)) inexact = 1;
    }
    nshl = __reduce_add_sync(FULL, nshl);
    inexact = __any_sync(FULL, inexact);
    if (lane == 0) {
      if (on && nshl) cnt_step[K_DOT * OP_COUNT + OP_SHL] += nshl;
      if (inexact) ctl->add_inexact = 1;
    }
  }
  __syncwarp();
  SW_TS(2)
  // h_{j+1,j} = fx_norm(w) (fxp.cpp:69-86) and the vec_div reciprocal: lane 0
  int ret = 0;
  int happy = 0;
  if (lane == 0) {
    const i64 nsum = static_cast<i64>(*nacc);
    if (checked == 1) {
      if (*norm_mul == 0) {
        const unsigned __int128 s2 = (static_cast<unsigned __int128>(nabs[0]) << 32) + nabs[1];
        const unsigned __int128 wraps = (s2 + (static_cast<unsigned __int128>(1) << 63)) >> 64;
        cnt_step[K_NORM * OP_COUNT + OP_ADD] += static_cast<u64>(wraps);
      } else if (!abs_small(nabs)) {
        ctl->add_inexact = 1;
      }
    }
    SW_TS(6)
    if (nsum < 0) {
      set_err(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
      ret = 1;
    } else {
      const i64 r = static_cast<i64>(isqrt_nl(static_cast<u64>(nsum)));
      SW_TS(7)
      const int es = sh.norm_b1;
      if (shl_ovf(r, es)) ev.hit(K_NORM, OP_SHL);
      const i64 hnext = wrap_shl(r, es);
      col[j + 1] = hnext;
      ctl->hnext = hnext;
      happy = hnext == 0;
      if (!happy) {
        const i64 den = asr(hnext, sh.div_b2);
        if (den == 0) {
          if (shl_ovf(w[0], sh.div_b1)) ev.hit(K_VEC_DIV, OP_SHL);
          set_err(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
          ret = 1;
        } else {
          const SDivMagic gm = make_sdiv_nl(den);
          SW_TS(8)
          ctl->div_m = gm.u.m;
          ctl->div_sh1 = gm.u.sh1;
          ctl->div_sh2 = gm.u.sh2;
          ctl->div_neg = gm.den_neg;
          ctl->div_m1 = gm.den_is_m1;
          ctl->do_vecdiv = 1;
          ctl->nbasis = j + 2;
        }
      }
    }
  }
  if (__shfl_sync(FULL, ret, 0)) return;
  happy = __shfl_sync(FULL, happy, 0);
  SW_TS(3)
  // apply_stored_rotations (gmres_int.cpp:8-25)
  if (j > 0) {
    const int gb2 = sh.givens_b2, sr = f - gb2;  // d_fx_mul(., ., f, 0, givens_b2, f)
    auto fxm = [&](i64 a, i64 b) { return asr(wmul(a, asr(b, gb2)), sr); };
    auto fxm_ovf = [&](i64 a, i64 b) { return mul_ovf(a, asr(b, gb2)) ? 1u : 0u; };
    unsigned nmul = 0, nadd = 0, nsub = 0;
    i64 x = col[0];  // x_0: the finalised h_0j
    for (int base = 0; base < j; base += 32) {
      const int i = base + lane;
      const bool act = i < j;
      const i64 c = act ? cs[i] : 0, sv = act ? sn[i] : 0, h1 = act ? col[i + 1] : 0;
      const i64 D = fxm(c, h1), B = fxm(sv, h1);
      __syncwarp();  // every lane has read its h_{i+1,j} before the outputs overwrite them
      i64 xi = 0;
      const int cnt = min(32, j - base);
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {  // the chain, on every lane
        const i64 st = __shfl_sync(FULL, sv, t), Dt = __shfl_sync(FULL, D, t);
        if (lane == t) xi = x;
        x = wsub(Dt, fxm(st, x));
      }
      if (act) {
        const i64 a = fxm(c, xi), q = fxm(sv, xi);
        nmul += fxm_ovf(c, xi) + fxm_ovf(sv, h1) + fxm_ovf(c, h1) + fxm_ovf(sv, xi);
        nadd += add_ovf(a, B);
        nsub += sub_ovf(D, q);
        col[i] = wadd(a, B);
      }
      __syncwarp();
    }
    if (lane == 0) col[j] = x;  // x_j: the last rotation's h_{j,j}
    nmul = __reduce_add_sync(FULL, nmul);
    nadd = __reduce_add_sync(FULL, nadd);
    nsub = __reduce_add_sync(FULL, nsub);
    if (lane == 0 && on) {
      if (nmul) cnt_step[K_GIVENS * OP_COUNT + OP_MUL] += nmul;
      if (nadd) cnt_step[K_GIVENS * OP_COUNT + OP_ADD] += nadd;
      if (nsub) cnt_step[K_GIVENS * OP_COUNT + OP_SUB] += nsub;
    }
  }
  __syncwarp();
  SW_TS(4)
  if (lane != 0) return;
  // t_mp = fx_norm((h_jj, h_{j+1,j})) (gmres_int.cpp:133-137)
  i64 tmp;
  {
    const i64 s0 = asr(col[j], sh.norm_b1), s1 = asr(col[j + 1], sh.norm_b1);
    if (mul_ovf(s0, s0)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const i64 p0 = wmul(s0, s0);
    i64 acc = p0;
    if (mul_ovf(s1, s1)) ev.hit(K_GIVENS_NORM, OP_MUL);
    const i64 p1 = wmul(s1, s1);
    if (add_ovf(acc, p1)) ev.hit(K_GIVENS_NORM, OP_ADD);
    acc = wadd(acc, p1);
    if (acc < 0) {
      set_err(ctl, IGM_DOMAIN_ERROR, EM_NORM_NEG, j);
      return;
    }
    const i64 r = static_cast<i64>(isqrt_nl(static_cast<u64>(acc)));
    if (shl_ovf(r, sh.norm_b1)) ev.hit(K_GIVENS_NORM, OP_SHL);
    tmp = wrap_shl(r, sh.norm_b1);
  }
  SW_TS(9)
  if (tmp == 0) {
    ctl->stop = 1;
    return;
  }
  i64 c, sv;
  if (!d_fx_div(col[j], tmp, f, sh.div_b1, sh.div_b2, &c, ev, K_GIVENS_DIV) ||
      !d_fx_div(col[j + 1], tmp, f, sh.div_b1, sh.div_b2, &sv, ev, K_GIVENS_DIV)) {
    set_err(ctl, IGM_DOMAIN_ERROR, EM_DIV_ZERO, j);
    return;
  }
  SW_TS(10)
  cs[j] = c;
  sn[j] = sv;
  col[j] = tmp;
  col[j + 1] = 0;
  // residual estimate (gmres_int.cpp:150-153)
  if (sub_ovf(0, sv)) ev.hit(K_ROT, OP_SUB);
  const i64 neg_s = wsub(0, sv);
  g[j + 1] = d_fx_mul(neg_s, g_old, f, sh.rot_b, sh.rot_b, f, ev, K_ROT);
  g[j] = d_fx_mul(c, g_old, f, sh.rot_b, sh.rot_b, f, ev, K_ROT);
  ctl->dim = j + 1;
  gabs[j] = g[j + 1];
  if (happy) ctl->stop = 1;
  SW_TS(5)
#undef SW_TS
}

__global__ void k_step_scalar(int j, int f, ShiftsD sh, const u64* acc_col, int acc_st, const u64* abs_col,
                              int abs_st, const u64* nacc, const u64* nabs, const u64* norm_mul, i64* hess,
                              int ld, i64* g, i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step,
                              Ctl* ctl, int checked) {
  step_scalar_warp(j, f, sh, acc_col, acc_st, abs_col, abs_st, nacc, nabs, norm_mul, hess, ld, g, cs, sn, gabs, w,
                   cnt_step, ctl, checked);
}

// ---------------------------------------------------------------------------
// K2-K5 as ONE persistent kernel per Arnoldi step (gmres_int.cpp:90-126):
// the same passes, reductions and scalar work as k_mgs / k_step_scalar /
// k_vec_div, but each CTA keeps its slice of w -- and of the previous basis
// vector -- in shared memory across the j+3 passes of the step, so a pass
// reads one basis vector from HBM instead of streaming w in and out, and the
// step costs one launch.  Passes are separated by a grid barrier (all CTAs
// are co-resident: cooperative launch, one CTA per SM).  Every arithmetic
// step is the per-element one of the pass kernels, and reductions are the
// same wrapping (order-free) u64 sums, so results are bit-identical.
constexpr int kArnThreads = 1024;
constexpr size_t kArnSmemMax = 227 * 1024 - 2048;  // dynamic; static + dynamic <= 228 KB per CTA (k_arnoldi2: 2.1 KB static)

// grid barrier: arrival count since the cycle started (Ctl::gbar); barrier
// number k completes when all G CTAs have arrived k times.  The acquire spin
// also orders this SM's later loads after every CTA's pre-barrier atomics.
__device__ __forceinline__ u64 ld_cg_u64(const u64* p) {
  u64 v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ...and thread 0 fetches the one word the next pass needs (a reduced
// accumulator) and broadcasts it through shared memory: one L2 request per
// CTA instead of one per warp on a single hot line
// pre: an optional [pre, pre + pre_bytes) range (this CTA's slice of the next
// pass's basis vector) prefetched into L2 while the barrier is pending
// SYNC_IN = false: the caller's threads have already met at a CTA barrier
// after their last work of the phase (cta_reduce_add's), so thread 0 goes
// straight to the arrival while the other warps are free until the closing
// barrier (k_arnoldi2 issues the next basis slice's bulk copy there)
template <bool SYNC_IN = true>
__device__ __forceinline__ u64 grid_barrier(Ctl* ctl, unsigned target, const u64* fetch, u64* s_word,
                                            const void* pre = nullptr, unsigned pre_bytes = 0) {
  if (SYNC_IN) __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* p = &ctl->gbar;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
    if (pre_bytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pre), "r"(pre_bytes) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    } while (v < target);
    if (fetch) *s_word = ld_cg_u64(fetch);
  }
  __syncthreads();
  return fetch ? *s_word : 0;
}

// CTA-wide wrapping sums of (s0, s1, s2) -> one atomic each (s1, s2 when CHECKED)
template <bool CHECKED, int NT = kArnThreads>
__device__ __forceinline__ void cta_reduce_add(u64 s0, u64 s1, u64 s2, u64* out0, u64* out12, u64 (*red)[32]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_down_sync(0xffffffffu, s0, o);
    if (CHECKED) {
      s1 += __shfl_down_sync(0xffffffffu, s1, o);
      s2 += __shfl_down_sync(0xffffffffu, s2, o);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = s0;
    red[1][wid] = s1;
    red[2][wid] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 a = 0, b = 0, c = 0;
    for (int i = 0; i < NT / 32; ++i) {
      a += red[0][i];
      b += red[1][i];
      c += red[2][i];
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(out0), static_cast<unsigned long long>(a));
    if (CHECKED) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out12), static_cast<unsigned long long>(b));
      atomicAdd(reinterpret_cast<unsigned long long*>(out12 + 1), static_cast<unsigned long long>(c));
    }
  }
  __syncthreads();
}

// Pass reduction and grid barrier of k_arnoldi2 in one hand-off: the CTA's
// wrapping sum is added to the pass's SNAPSHOT slot {accumulator, arrivals}
// (one aligned 16-byte pair, zeroed per cycle) and its arrival is counted in
// the same slot with release semantics, so a waiter's single 128-bit load
// returns the arrival count AND the accumulator as the L2 held them at one
// instant -- arrivals == grid means every CTA's sum is in (each CTA's add
// precedes its arrival).  That saves the barrier's second round trip (the
// separate load of the accumulator after the counter was seen, ~0.7 us).
template <bool CHECKED, int NT>
__device__ __forceinline__ void cta_reduce_post(u64 s0, u64 s1, u64 s2, u64* snap, u64* out12, u64 (*red)[32],
                                                u64 zmask) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_down_sync(0xffffffffu, s0, o);
    if (CHECKED) {
      s1 += __shfl_down_sync(0xffffffffu, s1, o);
      s2 += __shfl_down_sync(0xffffffffu, s2, o);
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = s0;
    red[1][wid] = s1;
    red[2][wid] = s2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 a = 0, b = 0, c = 0;
    for (int i = 0; i < NT / 32; ++i) {
      a += red[0][i];
      b += red[1][i];
      c += red[2][i];
    }
    if (CHECKED) {  // the certificate words: read after the step's later (release / acquire) barriers
      atomicAdd(reinterpret_cast<unsigned long long*>(out12), static_cast<unsigned long long>(b));
      atomicAdd(reinterpret_cast<unsigned long long*>(out12 + 1), static_cast<unsigned long long>(c));
    }
    // The arrival must follow the sum in the slot.  Instead of a release
    // fence (a membar over all of the thread's outstanding atomics), the sum
    // is a RETURNING atomic and the arrival's operand depends on its result:
    // the add has been performed at the L2 before the arrival is even issued,
    // and both target the same 16-byte slot.  (`zmask` is 0 at run time.)
    const unsigned long long old =
        atomicAdd(reinterpret_cast<unsigned long long*>(snap), static_cast<unsigned long long>(a));
    const unsigned long long inc = 1ull + (old & zmask);
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(snap + 1), "l"(inc) : "memory");
  }
}
// waits for the pass's snapshot slot to show `grid` arrivals; returns the
// accumulator to every thread; CTA 0 also files it in the step's accumulator
// array (the scalar step, the host and the trace replay read it there)
__device__ __forceinline__ u64 snap_wait(const u64* snap, unsigned grid, u64* acc_out, u64* s_word) {
  if (threadIdx.x == 0) {
    u64 a, c;
    do {
      asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                   : "=l"(a), "=l"(c)
                   : "l"(snap)
                   : "memory");
    } while (c < grid);
    *s_word = a;
    if (blockIdx.x == 0) *acc_out = a;
  }
  __syncthreads();
  return *s_word;
}

// per-element pieces of the passes (identical to k_mgs / k_vec_div)
struct ArnAcc {
  u64 sum = 0, ahi = 0, alo = 0, n1 = 0, n2 = 0, n3 = 0;
  __device__ __forceinline__ void abs_add(i64 t) {
    const u64 at = t < 0 ? 0ull - static_cast<u64>(t) : static_cast<u64>(t);
    ahi += at >> 32;
    alo += at & 0xffffffffull;
  }
};

__device__ __forceinline__ void lds_q(const i64* p, i64 (&v)[4]) {
  const longlong2 a = *reinterpret_cast<const longlong2*>(p), b = *reinterpret_cast<const longlong2*>(p + 2);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}
__device__ __forceinline__ void sts_q(i64* p, const i64 (&v)[4]) {
  *reinterpret_cast<longlong2*>(p) = make_longlong2(v[0], v[1]);
  *reinterpret_cast<longlong2*>(p + 2) = make_longlong2(v[2], v[3]);
}

// Walk this CTA's rows four at a time (256-bit global, 128-bit shared
// accesses), then the < 4 tail rows; fn(r, k, ...) handles row r.
template <typename F>
__device__ __forceinline__ void arn_rows(long long cnt, F&& fn) {
  const long long nq = cnt >> 2;
#pragma unroll 2
  for (long long q = threadIdx.x; q < nq; q += kArnThreads) fn(q * 4, 4);
  for (long long r = nq * 4 + threadIdx.x; r < cnt; r += kArnThreads) fn(r, 1);
}

template <bool CHECKED>
__global__ void __launch_bounds__(kArnThreads, 1)
    k_arnoldi(long long n, int j, long long S, const i64* __restrict__ win, i64* basis, u64* accj, u64* absj,
              u64* nacc, u64* nabs, int f, ShiftsD sh, u64* cstep, i64* hess, int ld, i64* g, i64* cs, i64* sn,
              i64* gabs, Ctl* ctl, unsigned gbase, u64* vmx) {
  extern __shared__ __align__(16) i64 arn_sm[];
  __shared__ u64 red[3][32];
  __shared__ u64 s_word;
  __shared__ int s_vd[6];
  if (cycle_over(ctl)) return;  // uniform: ctl is not written before the first barrier
  const unsigned G = gridDim.x;
  unsigned nbar = gbase;
  i64* sw = arn_sm;      // this CTA's rows of w
  i64* sv = arn_sm + S;  // this CTA's rows of the previous pass's basis vector
  const long long lo = static_cast<long long>(blockIdx.x) * S;
  const long long cnt = max(0LL, min(n, lo + S) - lo);
  u64 *cA = cstep + K_AXPY * OP_COUNT, *cD = cstep + K_DOT * OP_COUNT, *cN = cstep + K_NORM * OP_COUNT;
  const int post = f - sh.axpy_b1;
  // a quad (k == 4) or a single row (k == 1) of global / shared data
  auto gload = [](const i64* p, int k, i64 (&v)[4]) {
    if (k == 4) ld_v4_nc(p, v);
    else v[0] = __ldg(p);
  };
  auto sload = [](const i64* p, int k, i64 (&v)[4]) {
    if (k == 4) lds_q(p, v);
    else v[0] = *p;
  };
  auto sstore = [](i64* p, int k, const i64 (&v)[4]) {
    if (k == 4) sts_q(p, v);
    else *p = v[0];
  };
  // OVF: per-element product / subtraction overflow tests.  In checked mode
  // a pass runs without them when this CTA's magnitude bounds prove none of
  // its rows can overflow (certify() below); the sum |t| certificate of the
  // order-dependent add events is always accumulated.
  auto dot_term = [&](i64 wl, i64 c, ArnAcc& A, auto ovf) {
    const i64 a = asr(wl, sh.dot_b1), b = asr(c, sh.dot_b2);
    const i64 t = wmul(a, b);
    A.sum += static_cast<u64>(t);
    if (CHECKED) {
      if (decltype(ovf)::value) A.n3 += mul_ovf(a, b);
      A.abs_add(t);
    }
  };
  auto axpy_term = [&](i64 hs, i64 vp, i64& wl, ArnAcc& A, auto ovf) {
    const i64 d = asr(wmul(hs, vp), post);
    if (CHECKED && decltype(ovf)::value) {
      A.n1 += mul_ovf(hs, vp);
      A.n2 += sub_ovf(wl, d);
    }
    wl = wsub(wl, d);
  };
  // ---- magnitude bounds of this CTA's rows (checked mode): W >= max|w|,
  // vmx[blk][i] = max|v_i| (written by this CTA when it produced v_i), V0 =
  // max|v_0| (measured in pass 0)
  constexpr u64 kLim = 1ull << 63;
  auto absu = [](i64 v) -> u64 { return v < 0 ? u64{0} - static_cast<u64>(v) : static_cast<u64>(v); };
  auto mul_lt = [&](u64 x, u64 y2) { return __umul64hi(x, y2) == 0 && x * y2 < kLim; };
  auto shb = [](u64 v, int s2) { return (s2 >= 63 ? 0ull : (v >> (s2 < 0 ? 0 : s2))) + 1; };  // >= |asr(x, s)| for |x| <= v
  const int vst = ld + 1;
  u64* vmx_me = vmx + static_cast<size_t>(blockIdx.x) * vst;
  u64 Wb = 0, V0 = 0;
  __shared__ u64 s_mx[2];
  auto cta_max2 = [&](u64 m0, u64 m1) {  // CTA-wide maxima -> (s_mx[0], s_mx[1])
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m0 = max(m0, static_cast<u64>(__shfl_down_sync(0xffffffffu, m0, o)));
      m1 = max(m1, static_cast<u64>(__shfl_down_sync(0xffffffffu, m1, o)));
    }
    if (threadIdx.x == 0) s_mx[0] = s_mx[1] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(&s_mx[0]), static_cast<unsigned long long>(m0));
      atomicMax(reinterpret_cast<unsigned long long*>(&s_mx[1]), static_cast<unsigned long long>(m1));
    }
    __syncthreads();
  };
  // a pass "axpy with (hs, Vp), then a product of asr(w, b1) with a value
  // bounded by Q" is free of product / subtraction overflow when the bounds
  // say so; advances Wb past the axpy
  auto certify = [&](u64 ahs, u64 Vp, int qs1, u64 Q, bool has_axpy) {
    bool ok = true;
    u64 W2 = Wb;
    if (has_axpy) {
      ok = post >= 0 && mul_lt(ahs, Vp);
      const u64 dmax = ok ? ((ahs * Vp) >> post) + 1 : kLim;
      ok = ok && W2 < kLim && dmax < kLim - W2;
      W2 = ok ? W2 + dmax : kLim;
    }
    ok = ok && mul_lt(shb(W2, qs1), Q);
    Wb = W2;
    return ok;
  };
  // ---- pass 0: w -> shared memory, dot_0 = <w, v_0>
  {
    const i64* v0 = basis + lo;
    ArnAcc A;
    arn_rows(cnt, [&](long long r, int k) {
      i64 wq[4], cq[4];
      gload(win + lo + r, k, wq);
      gload(v0 + r, k, cq);
      sstore(sw + r, k, wq);
      sstore(sv + r, k, cq);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < k) {
          dot_term(wq[e], cq[e], A, std::true_type{});
          if (CHECKED) {
            Wb = max(Wb, absu(wq[e]));
            V0 = max(V0, absu(cq[e]));
          }
        }
    });
    if (CHECKED) bump(cD, OP_MUL, A.n3);
    cta_reduce_add<CHECKED>(A.sum, A.ahi, A.alo, accj + 0, absj + 0, red);
    if (CHECKED) {
      cta_max2(Wb, V0);
      Wb = s_mx[0];
      V0 = s_mx[1];
    }
  }
  // ---- passes 1..j: axpy_{i-1} (v_{i-1} from shared memory), dot_i
  const int e0 = f - sh.dot_b1 - sh.dot_b2;
  auto h_of = [&](u64 acc) {  // h_{i-1} re-derived from the reduced accumulator
    const i64 a = static_cast<i64>(acc);
    const i64 h = e0 >= 0 ? asr(a, e0) : wrap_shl(a, -e0);
    return asr(h, sh.axpy_b1);
  };
  for (int i = 1; i <= j; ++i) {
    const i64* vi = basis + static_cast<long long>(i) * n + lo;
    const i64 hs = h_of(grid_barrier(ctl, (++nbar) * G, accj + i - 1, &s_word, vi,
                                     static_cast<unsigned>(cnt * 8) & ~15u));
    ArnAcc A;
    auto pass = [&](auto ovf) {
      arn_rows(cnt, [&](long long r, int k) {
        i64 wq[4], pq[4], cq[4];
        gload(vi + r, k, cq);
        sload(sw + r, k, wq);
        sload(sv + r, k, pq);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < k) {
            axpy_term(hs, pq[e], wq[e], A, ovf);
            dot_term(wq[e], cq[e], A, ovf);
          }
        sstore(sw + r, k, wq);
        sstore(sv + r, k, cq);
      });
    };
    if (CHECKED && certify(absu(hs), i == 1 ? V0 : vmx_me[i - 1], sh.dot_b1, shb(vmx_me[i], sh.dot_b2), true))
      pass(std::false_type{});
    else
      pass(std::true_type{});
    if (CHECKED) {
      bump(cA, OP_MUL, A.n1);
      bump(cA, OP_SUB, A.n2);
      bump(cD, OP_MUL, A.n3);
    }
    cta_reduce_add<CHECKED>(A.sum, A.ahi, A.alo, accj + i, absj + 2 * i, red);
  }
  // ---- axpy_j, then the norm sum of the orthogonalised w
  {
    const i64 hs = h_of(grid_barrier(ctl, (++nbar) * G, accj + j, &s_word));
    ArnAcc A;
    auto pass = [&](auto ovf) {
      arn_rows(cnt, [&](long long r, int k) {
        i64 wq[4], pq[4];
        sload(sw + r, k, wq);
        sload(sv + r, k, pq);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < k) {
            axpy_term(hs, pq[e], wq[e], A, ovf);
            const i64 sq = asr(wq[e], sh.norm_b1);
            const i64 t = wmul(sq, sq);
            A.sum += static_cast<u64>(t);
            if (CHECKED) {
              if (decltype(ovf)::value) A.n3 += mul_ovf(sq, sq);
              A.abs_add(t);
            }
          }
        sstore(sw + r, k, wq);
      });
    };
    bool fast = false;
    if (CHECKED) {
      const u64 Vp = j == 0 ? V0 : vmx_me[j];
      fast = certify(absu(hs), Vp, 0, 1, true);  // the axpy (the product bound is checked next)
      fast = fast && mul_lt(shb(Wb, sh.norm_b1), shb(Wb, sh.norm_b1));
    }
    if (fast)
      pass(std::false_type{});
    else
      pass(std::true_type{});
    if (CHECKED) {
      bump(cA, OP_MUL, A.n1);
      bump(cA, OP_SUB, A.n2);
      bump(cN, OP_MUL, A.n3);
    }
    cta_reduce_add<CHECKED>(A.sum, A.ahi, A.alo, nacc, nabs, red);
  }
  // ---- per-step scalar work (one thread), then v_{j+1} = w / h_{j+1,j}
  grid_barrier(ctl, (++nbar) * G, nullptr, nullptr);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence();  // this SM's L1 holds no stale copy of the reduced words
    step_scalar_dev(j, f, sh, accj, 1, absj, 2, nacc, nabs, cstep + K_NORM * OP_COUNT + OP_MUL, hess, ld, g, cs,
                    sn, gabs, sw, cstep, ctl, CHECKED ? 1 : 0);
  }
  const u64 dm = grid_barrier(ctl, (++nbar) * G, &ctl->div_m, &s_word);
  if (threadIdx.x == 0) {  // the divisor's magic, once per CTA
    volatile const int* c = &ctl->do_vecdiv;
    s_vd[0] = c[0];
    s_vd[1] = *static_cast<volatile int*>(&ctl->div_sh1);
    s_vd[2] = *static_cast<volatile int*>(&ctl->div_sh2);
    s_vd[3] = *static_cast<volatile int*>(&ctl->div_neg);
    s_vd[4] = *static_cast<volatile int*>(&ctl->div_m1);
  }
  __syncthreads();
  if (!s_vd[0]) return;
  {
    SDivMagic gm;
    gm.u.m = dm;
    gm.u.sh1 = s_vd[1];
    gm.u.sh2 = s_vd[2];
    gm.den_neg = s_vd[3];
    gm.den_is_m1 = s_vd[4];
    const int b1 = sh.div_b1, ee = f - sh.div_b1 - sh.div_b2;
    i64* out = basis + static_cast<long long>(j + 1) * n + lo;
    u64 nshl = 0, ndiv = 0, vmax = 0;
    arn_rows(cnt, [&](long long r, int k) {
      i64 wq[4], vq[4];
      sload(sw + r, k, wq);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < k) {
          const i64 a = wq[e];
          const i64 num = wrap_shl(a, b1);
          const i64 q = sdiv(num, gm);
          if (ee >= 0) {
            vq[e] = wrap_shl(q, ee);
            if (CHECKED) nshl += shl_ovf(q, ee);
          } else {
            vq[e] = asr(q, -ee);
          }
          if (CHECKED) {
            nshl += shl_ovf(a, b1);
            ndiv += sdiv_ovf(num, gm);
          }
        }
      if (k == 4) st_v4(out + r, vq);
      else out[r] = vq[0];
      if (CHECKED)
        for (int e = 0; e < k; ++e) vmax = max(vmax, absu(vq[e]));
    });
    if (CHECKED) {
      bump(cstep + K_VEC_DIV * OP_COUNT, OP_SHL, nshl);
      bump(cstep + K_VEC_DIV * OP_COUNT, OP_DIV, ndiv);
      cta_max2(vmax, 0);
      if (threadIdx.x == 0) {
        vmx_me[j + 1] = s_mx[0];  // read by this CTA in later steps of the cycle
        atomicMax(reinterpret_cast<unsigned long long*>(vmx + static_cast<size_t>(kVmxRows - 1) * vst + j + 1),
                  static_cast<unsigned long long>(s_mx[0]));  // all CTAs: the SpMV's certificate
      }
    }
  }
}


__global__ void k_cycle_init(Ctl* ctl, i64* g, int f) {
  ctl->gbar = 0;
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
// K6/K9 ILU(0) triangular substitutions (ilu.cpp:122-180) as a wavefront.
//
// The factor's rows are cut into tiles (schedule.hpp: bricks of a detected
// structured grid, else contiguous blocks); one CTA owns one tile, keeps the
// tile's solution values in shared memory and walks it one DAG level (one
// segment of <= 256 rows, a row per compute thread) at a time.  Tiles are
// handed out by a ticket counter in layer-major order, so every producer a
// CTA waits on is already running.
//
//   warps 0-7  compute.  Per level: named barrier (the previous level's
//              values are in shared memory), dependency values from shared
//              memory only, the reference's row arithmetic, store.
//   warp  8    loader.  Per level, into a ring slot of L levels: one bulk
//              copy of the level's packed row records, one of its
//              right-hand-side run (already in schedule order, k_tri_gather),
//              and the values of the level's cross-tile producer rows, polled
//              from their tagged 128-bit words two levels ahead.
//
// A value another tile reads is published as one aligned 128-bit store of
// (value, epoch ^ value); the poller accepts a word only when its tag
// matches this launch, so there are no flags and no gpu-scope fences.  The
// epoch is a hashed 64-bit launch id: a word left by an earlier launch never
// matches, and a torn read would need the two values to differ by exactly
// the XOR of two random 64-bit ids.
//
// Per row the arithmetic is the reference's: integer path wrapping
// multiply/subtract (summed in any order: mod 2^64 the result is the same)
// and truncating division by the raw diagonal (exact reciprocal); FP path the
// same in FP64 on the integer factors, in CSR order, without contraction.
struct TriArgs {
  int n, ntiles;
  const int* tile_pbase;  // first schedule slot of each tile
  const int* tile_seg;    // first segment of each tile
  const int* seg_rows;    // first slot of each segment
  const int* seg_xptr;    // per segment: its cross-tile producer rows
  const int* seg_xrow;
  const int* p_xdep;      // dependencies beyond the record stride (rare)
  const i64* p_xval;
  const unsigned char* p_rec;  // packed per-slot records (schedule.hpp)
  const int* p_xrp;            // compact records: extra-dependency index per slot
  const i64* p_diag;           // compact records: diagonal per slot (FP path)
  int tile_cap, max_seg_ext;
  u64* zmax;                   // max |z| of the integer apply (checked mode's overflow bound)
  ulonglong2* xz;              // exported values: (value, epoch ^ value) per row
  unsigned long long epoch;    // per launch: hashed, non-zero
  int* ticket;
};

// one cross-tile word (value, tag): a single strong 128-bit access
__device__ __forceinline__ void xz_load(const ulonglong2* p, u64& v, u64& tg) {
  asm volatile("{ .reg .b128 t; ld.global.relaxed.gpu.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(v), "=l"(tg)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ u64 xz_wait(const ulonglong2* p, u64 epoch) {
  u64 v, tg;
  do {
    xz_load(p, v, tg);
  } while (tg != (epoch ^ v));
  return v;
}
__device__ __forceinline__ void xz_put(ulonglong2* p, u64 v, u64 epoch) {
  asm volatile("{ .reg .b128 t; mov.b128 t, {%0, %1}; st.global.relaxed.gpu.b128 [%2], t; }" ::"l"(v),
               "l"(epoch ^ v), "l"(p)
               : "memory");
}

// debug: per-level phase timestamps of one tile (igm_debug_tri_trace)
__device__ unsigned long long* g_tri_ts = nullptr;
__device__ int g_tri_ts_tile = -1;
__device__ __forceinline__ unsigned long long gtime() { return clock64(); }  // per-SM cycles

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- shared-window (32-bit address) helpers: mbarrier, bulk copy, ld/st
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init_s(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_s(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// L2 prefetch of a global range (16-byte aligned, size a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ i64 lds64(unsigned a) {
  i64 v;
  asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts64(unsigned a, i64 v) {
  asm volatile("st.shared.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// K2-K5, register-resident variant (config 2 sizes): the same passes, step
// order and overflow accounting as k_arnoldi, but w lives in registers (512
// threads x kArn2Q quads of 4 rows each), the two shared-memory buffers hold
// v_{i-1} and v_i, and each next basis vector's slice arrives by one bulk
// copy (TMA, cp.async.bulk + mbarrier) issued as soon as its buffer is free
// -- so the HBM stream of the basis overlaps each pass's reduction and grid
// barrier instead of following it.
constexpr int kArn2Threads = 512;
constexpr int kArn2Q = 7;  // quads per thread: up to 4 * 512 * 7 = 14336 rows per CTA

// debug (igm_debug_arn_ts): per-CTA phase timestamps (globaltimer, ns) of the
// Arnoldi step j = g_arn_ts_j; slot 4i+0 v_i's buffer ready, +1 pass i
// computed, +2 CTA sum added, +3 grid barrier passed; 120.. the step tail
__device__ unsigned long long* g_arn_ts = nullptr;
__device__ int g_arn_ts_j = -1;
constexpr int kArnTsSlots = 128;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <bool CHECKED>
__global__ void __launch_bounds__(kArn2Threads, 1)
    k_arnoldi2(long long n, int j, long long S, const i64* __restrict__ win, i64* basis, u64* accj, u64* absj,
               u64* nacc, u64* nabs, int f, ShiftsD sh, u64* cstep, i64* hess, int ld, i64* g, i64* cs, i64* sn,
               i64* gabs, Ctl* ctl, unsigned gbase, u64* vmx, u64* snapj) {
  extern __shared__ __align__(16) i64 arn_sm[];
  __shared__ u64 red[3][32];
  __shared__ u64 s_word;
  __shared__ int s_vd[6];
  __shared__ __align__(8) unsigned long long s_bar[2];
  __shared__ __align__(8) unsigned long long s_cbar[kArn2Q];  // chunk m of v_{i-1} consumed by every warp
  __shared__ u64 s_mx[2];
  if (cycle_over(ctl)) return;  // uniform: ctl is not written before the first barrier
  unsigned long long* ts = (g_arn_ts_j == j && threadIdx.x == 0) ? g_arn_ts + blockIdx.x * kArnTsSlots : nullptr;
#define ARN_TS(slot) \
  if (ts != nullptr && (slot) < kArnTsSlots) ts[slot] = gtimer();
  constexpr int T = kArn2Threads, Q = kArn2Q;
  const unsigned G = gridDim.x;
  const u64 zmask = static_cast<u64>(n) >> 62;  // 0 (n < 2^62), unknown to the compiler: see cta_reduce_post
  unsigned nbar = gbase;
  const long long lo = static_cast<long long>(blockIdx.x) * S;
  const long long cnt = max(0LL, min(n, lo + S) - lo);  // a multiple of 4 (n, S are)
  const int nq = static_cast<int>(cnt >> 2);
  const int tid = threadIdx.x;
  i64* buf[2] = {arn_sm, arn_sm + S};
  const unsigned bar0 = smem_u32(&s_bar[0]);
  const unsigned cbar0 = smem_u32(&s_cbar[0]);
  if (tid == 0) {
    mbar_init_s(bar0, 1);
    mbar_init_s(bar0 + 8, 1);
#pragma unroll
    for (int m = 0; m < Q; ++m) mbar_init_s(cbar0 + 8u * m, T / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned ph[2] = {0, 0};
  // thread 0: this CTA's slice of basis vector `v` into buffer b
  auto fetch = [&](int b, const i64* v) {
    const unsigned bar = bar0 + 8u * b;
    if (cnt > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx_s(bar, static_cast<unsigned>(cnt * 8));
      bulk_g2s_s(smem_u32(buf[b]), v + lo, static_cast<unsigned>(cnt * 8), bar);
    } else {
      mbar_arrive_s(bar);
    }
  };
  auto wait_buf = [&](int b) {
    mbar_wait_s(bar0 + 8u * b, ph[b]);
    ph[b] ^= 1u;
  };
  // Streaming refill: during pass i the slice of v_{i-1} is consumed chunk by
  // chunk (chunk m = the quads [m T, (m+1) T), 16 KB: iteration m of every
  // thread), and chunk m of v_{i+1} is copied into its place once every warp
  // has arrived on the chunk's mbarrier -- the HBM stream of the basis then
  // runs under the pass's arithmetic, not only under the grid barrier that
  // follows (whose round trips it delays: 4.2 vs ~2 us, scripts/arn_ts.py).
  // The issuing lane never sleeps on a chunk barrier inside the pass: it
  // TESTS it and issues whatever is free; the rest goes out after the pass.
  constexpr int kIssuer = T - 32;  // lane 0 of the last warp
  auto chunk_free = [&](int c, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(cbar0 + 8u * c), "r"(parity)
        : "memory");
    return ok != 0;
  };
  auto issue_chunk = [&](int c, int b, const i64* v) {
    // (no proxy fence: the chunk was only READ through the generic proxy, and
    // those reads are ordered before this point by the warps' arrivals)
    if (c == 0) {
      if (cnt > 0) mbar_arrive_expect_tx_s(bar0 + 8u * b, static_cast<unsigned>(cnt * 8));
      else mbar_arrive_s(bar0 + 8u * b);
    }
    const int q0 = c * T;
    if (q0 < nq)
      bulk_g2s_s(smem_u32(buf[b] + 4 * q0), v + lo + 4 * q0, static_cast<unsigned>(min(T, nq - q0)) * 32u,
                 bar0 + 8u * b);
  };
  if (tid == 0) {
    fetch(0, basis);
    if (j >= 1) fetch(1, basis + n);
  }
  u64 *cA = cstep + K_AXPY * OP_COUNT, *cD = cstep + K_DOT * OP_COUNT, *cN = cstep + K_NORM * OP_COUNT;
  const int post = f - sh.axpy_b1;
  auto dot_term = [&](i64 wl, i64 c, ArnAcc& A, auto ovf) {
    const i64 a = asr(wl, sh.dot_b1), b = asr(c, sh.dot_b2);
    const i64 t = wmul(a, b);
    A.sum += static_cast<u64>(t);
    if (CHECKED) {
      if (decltype(ovf)::value) A.n3 += mul_ovf(a, b);
      A.abs_add(t);
    }
  };
  auto axpy_term = [&](i64 hs, i64 vp, i64& wl, ArnAcc& A, auto ovf) {
    const i64 d = asr(wmul(hs, vp), post);
    if (CHECKED && decltype(ovf)::value) {
      A.n1 += mul_ovf(hs, vp);
      A.n2 += sub_ovf(wl, d);
    }
    wl = wsub(wl, d);
  };
  // magnitude bounds (checked mode), exactly as in k_arnoldi
  constexpr u64 kLim = 1ull << 63;
  auto absu = [](i64 v) -> u64 { return v < 0 ? u64{0} - static_cast<u64>(v) : static_cast<u64>(v); };
  auto mul_lt = [&](u64 x, u64 y2) { return __umul64hi(x, y2) == 0 && x * y2 < kLim; };
  auto shb = [](u64 v, int s2) { return (s2 >= 63 ? 0ull : (v >> (s2 < 0 ? 0 : s2))) + 1; };
  const int vst = ld + 1;
  u64* vmx_me = vmx + static_cast<size_t>(blockIdx.x) * vst;
  u64 Wb = 0, V0 = 0;
  auto cta_max2 = [&](u64 m0, u64 m1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m0 = max(m0, static_cast<u64>(__shfl_down_sync(0xffffffffu, m0, o)));
      m1 = max(m1, static_cast<u64>(__shfl_down_sync(0xffffffffu, m1, o)));
    }
    if (tid == 0) s_mx[0] = s_mx[1] = 0;
    __syncthreads();
    if ((tid & 31) == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(&s_mx[0]), static_cast<unsigned long long>(m0));
      atomicMax(reinterpret_cast<unsigned long long*>(&s_mx[1]), static_cast<unsigned long long>(m1));
    }
    __syncthreads();
  };
  auto certify = [&](u64 ahs, u64 Vp, int qs1, u64 Qb, bool has_axpy) {
    bool ok = true;
    u64 W2 = Wb;
    if (has_axpy) {
      ok = post >= 0 && mul_lt(ahs, Vp);
      const u64 dmax = ok ? ((ahs * Vp) >> post) + 1 : kLim;
      ok = ok && W2 < kLim && dmax < kLim - W2;
      W2 = ok ? W2 + dmax : kLim;
    }
    ok = ok && mul_lt(shb(W2, qs1), Qb);
    Wb = W2;
    return ok;
  };
  i64 wr[Q][4];  // this thread's rows of w: quads tid + m * T
  // ---- pass 0: w -> registers, dot_0 = <w, v_0>
  {
    ARN_TS(124)
    // w's loads go out before the wait for v_0's slice: both arrive together
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      const int q = tid + m * T;
      if (q < nq) ld_v4_nc(win + lo + 4 * q, wr[m]);
    }
    wait_buf(0);
    ARN_TS(0)
    ArnAcc A;
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      const int q = tid + m * T;
      if (q < nq) {
        i64 cq[4];
        lds_q(buf[0] + 4 * q, cq);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          dot_term(wr[m][e], cq[e], A, std::true_type{});
          if (CHECKED) {
            Wb = max(Wb, absu(wr[m][e]));
            V0 = max(V0, absu(cq[e]));
          }
        }
      }
    }
    if (CHECKED) bump(cD, OP_MUL, A.n3);
    ARN_TS(1)
    cta_reduce_post<CHECKED, T>(A.sum, A.ahi, A.alo, snapj + 0, absj + 0, red, zmask);
    ARN_TS(2)
    if (CHECKED) {
      cta_max2(Wb, V0);
      Wb = s_mx[0];
      V0 = s_mx[1];
    }
  }
  const int e0 = f - sh.dot_b1 - sh.dot_b2;
  auto h_of = [&](u64 acc) {
    const i64 a = static_cast<i64>(acc);
    const i64 h = e0 >= 0 ? asr(a, e0) : wrap_shl(a, -e0);
    return asr(h, sh.axpy_b1);
  };
  // ---- passes 1..j: axpy_{i-1} (v_{i-1} in buf[(i-1)&1]), dot_i (v_i in buf[i&1])
  for (int i = 1; i <= j; ++i) {
    const i64 hs = h_of(snap_wait(snapj + 2 * (i - 1), G, accj + i - 1, &s_word));
    ARN_TS(4 * i - 1)
    wait_buf(i & 1);
    ARN_TS(4 * i)
    const i64* vp = buf[(i - 1) & 1];
    const i64* vc = buf[i & 1];
    const bool refill = i + 1 <= j;  // v_{i+1} takes v_{i-1}'s place, chunk by chunk
    const i64* vnext = basis + static_cast<long long>(i + 1) * n;
    const unsigned cpar = static_cast<unsigned>(i - 1) & 1u;
    int issued = 0;  // (issuer lane) chunks of v_{i+1} on their way
    ArnAcc A;
    auto pass = [&](auto ovf) {
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        const int q = tid + m * T;
        if (q < nq) {
          i64 pq[4], cq[4];
          lds_q(vp + 4 * q, pq);
          lds_q(vc + 4 * q, cq);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            axpy_term(hs, pq[e], wr[m][e], A, ovf);
            dot_term(wr[m][e], cq[e], A, ovf);
          }
        }
        __syncwarp();  // the warp's reads of chunk m have been consumed
        if ((tid & 31) == 0) mbar_arrive_s(cbar0 + 8u * m);
        if (tid == kIssuer && refill)
          while (issued < m && chunk_free(issued, cpar)) issue_chunk(issued++, (i - 1) & 1, vnext);
      }
    };
    if (CHECKED && certify(absu(hs), i == 1 ? V0 : vmx_me[i - 1], sh.dot_b1, shb(vmx_me[i], sh.dot_b2), true))
      pass(std::false_type{});
    else
      pass(std::true_type{});
    if (CHECKED) {
      bump(cA, OP_MUL, A.n1);
      bump(cA, OP_SUB, A.n2);
      bump(cD, OP_MUL, A.n3);
    }
    ARN_TS(4 * i + 1)
    cta_reduce_post<CHECKED, T>(A.sum, A.ahi, A.alo, snapj + 2 * i, absj + 2 * i, red, zmask);
    ARN_TS(4 * i + 2)
    // every thread is past its reads of v_{i-1} (the reduction's CTA barrier):
    // its buffer takes v_{i+1}.  Issued by warp 1 while thread 0 runs the grid
    // barrier: the issuing thread stays blocked ~2.3 us behind the bulk copy
    // (scripts/arn_ts.py: 4.2 us per barrier with the copy issued on thread
    // 0's path against 1.5-2.1 us without one), so it must not be the thread
    // the barrier's arrival waits for.
    // The chunks still held back go out here, after the reduction's CTA
    // barrier (every chunk is free), while thread 0 runs the grid barrier.
    if (tid == kIssuer && refill)
      for (; issued < Q; ++issued) issue_chunk(issued, (i - 1) & 1, vnext);
  }
  // ---- axpy_j (v_j in buf[j&1]), then the norm sum of the orthogonalised w
  {
    const i64 hs = h_of(snap_wait(snapj + 2 * j, G, accj + j, &s_word));
    ARN_TS(4 * j + 3)
    const i64* vp = buf[j & 1];
    ArnAcc A;
    auto pass = [&](auto ovf) {
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        const int q = tid + m * T;
        if (q < nq) {
          i64 pq[4];
          lds_q(vp + 4 * q, pq);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            axpy_term(hs, pq[e], wr[m][e], A, ovf);
            const i64 sq = asr(wr[m][e], sh.norm_b1);
            const i64 t = wmul(sq, sq);
            A.sum += static_cast<u64>(t);
            if (CHECKED) {
              if (decltype(ovf)::value) A.n3 += mul_ovf(sq, sq);
              A.abs_add(t);
            }
          }
        }
      }
    };
    bool fast = false;
    if (CHECKED) {
      const u64 Vp = j == 0 ? V0 : vmx_me[j];
      fast = certify(absu(hs), Vp, 0, 1, true);
      fast = fast && mul_lt(shb(Wb, sh.norm_b1), shb(Wb, sh.norm_b1));
    }
    if (fast)
      pass(std::false_type{});
    else
      pass(std::true_type{});
    if (CHECKED) {
      bump(cA, OP_MUL, A.n1);
      bump(cA, OP_SUB, A.n2);
      bump(cN, OP_MUL, A.n3);
    }
    ARN_TS(4 * j + 5)
    cta_reduce_add<CHECKED, T>(A.sum, A.ahi, A.alo, nacc, nabs, red);
    ARN_TS(4 * j + 6)
  }
  // ---- per-step scalar work (one thread), then v_{j+1} = w / h_{j+1,j}
  grid_barrier(ctl, (++nbar) * G, nullptr, nullptr);
  ARN_TS(120)
  if (blockIdx.x == 0 && 6LL * (j + 2) > 2 * S) {  // too small a slice to stage in: straight from global memory
    if (tid == 0) {
      __threadfence();
      i64* w0 = reinterpret_cast<i64*>(&s_word);
      *w0 = nq > 0 ? wr[0][0] : 0;
      step_scalar_dev(j, f, sh, accj, 1, absj, 2, nacc, nabs, cstep + K_NORM * OP_COUNT + OP_MUL, hess, ld, g, cs,
                      sn, gabs, w0, cstep, ctl, CHECKED ? 1 : 0);
    }
  } else if (blockIdx.x == 0) {
    // the scalar step is a dependent chain of small reads and writes: stage
    // its operands (reduced accumulators, certificates, the Hessenberg
    // column, the stored rotations) in shared memory with all threads (the
    // v buffers are free now), run it on one thread there, write back
    u64* s_acc = reinterpret_cast<u64*>(buf[0]);
    u64* s_abs = s_acc + (j + 1);
    i64* s_col = reinterpret_cast<i64*>(s_abs + 2 * (j + 1));
    i64* s_cs = s_col + (j + 2);
    i64* s_sn = s_cs + (j + 1);
    i64* col = hess + static_cast<long long>(j) * ld;
    for (int q = tid; q <= j; q += T) {
      s_acc[q] = ld_cg_u64(accj + q);  // L2: the atomics' results
      s_abs[2 * q] = ld_cg_u64(absj + 2 * q);
      s_abs[2 * q + 1] = ld_cg_u64(absj + 2 * q + 1);
      s_col[q] = col[q];
      if (q < j) {
        s_cs[q] = cs[q];
        s_sn[q] = sn[q];
      }
    }
    if (tid == 0) s_col[j + 1] = col[j + 1];
    __syncthreads();
    i64* w0 = s_sn + (j + 1);
    // (no fence here: the grid barrier above acquired at gpu scope and dropped
    // the L1's lines, and the reduced words were loaded with ld.cg)
    if (tid == 0) {
      // w is only dereferenced for an error diagnostic: row 0 (this thread's first)
      *w0 = nq > 0 ? wr[0][0] : 0;
    }
    if (tid < 32) {
      __syncwarp();
      step_scalar_warp(j, f, sh, s_acc, 1, s_abs, 2, nacc, nabs, cstep + K_NORM * OP_COUNT + OP_MUL,
                       s_col - static_cast<long long>(j) * ld, ld, g, s_cs, s_sn, gabs, w0, cstep, ctl,
                       CHECKED ? 1 : 0, ts);
    }
    __syncthreads();
    for (int q = tid; q <= j + 1; q += T) col[q] = s_col[q];
    if (tid == 0) {
      cs[j] = s_cs[j];
      sn[j] = s_sn[j];
    }
  }
  ARN_TS(121)
  const u64 dm = grid_barrier(ctl, (++nbar) * G, &ctl->div_m, &s_word);
  ARN_TS(122)
  if (tid == 0) {
    volatile const int* c = &ctl->do_vecdiv;
    s_vd[0] = c[0];
    s_vd[1] = *static_cast<volatile int*>(&ctl->div_sh1);
    s_vd[2] = *static_cast<volatile int*>(&ctl->div_sh2);
    s_vd[3] = *static_cast<volatile int*>(&ctl->div_neg);
    s_vd[4] = *static_cast<volatile int*>(&ctl->div_m1);
  }
  __syncthreads();
  ARN_TS(125)
  if (!s_vd[0]) return;
  {
    SDivMagic gm;
    gm.u.m = dm;
    gm.u.sh1 = s_vd[1];
    gm.u.sh2 = s_vd[2];
    gm.den_neg = s_vd[3];
    gm.den_is_m1 = s_vd[4];
    const int b1 = sh.div_b1, ee = f - sh.div_b1 - sh.div_b2;
    i64* out = basis + static_cast<long long>(j + 1) * n + lo;
    u64 nshl = 0, ndiv = 0, vmax = 0;
    // w's registers -> this thread's own slots of the free buffer, then ONE
    // compact loop over them: this code runs once per launch, so its size
    // (instruction-cache misses), not its arithmetic, sets its time -- the
    // fully unrolled loop took 4x longer cold than warm
    i64* ws = buf[1];
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      const int q = tid + m * T;
      if (q < nq) sts_q(ws + 4 * q, wr[m]);
    }
#pragma unroll 1
    for (int m = 0; m < Q; ++m) {
      const int q = tid + m * T;
      if (q < nq) {
        i64 vq[4], wq[4];
        lds_q(ws + 4 * q, wq);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const i64 a = wq[e];
          const i64 num = wrap_shl(a, b1);
          const i64 qq = sdiv(num, gm);
          if (ee >= 0) {
            vq[e] = wrap_shl(qq, ee);
            if (CHECKED) nshl += shl_ovf(qq, ee);
          } else {
            vq[e] = asr(qq, -ee);
          }
          if (CHECKED) {
            nshl += shl_ovf(a, b1);
            ndiv += sdiv_ovf(num, gm);
            vmax = max(vmax, absu(vq[e]));
          }
        }
        st_v4(out + 4 * q, vq);
      }
    }
    ARN_TS(126)
    if (CHECKED) {
      bump(cstep + K_VEC_DIV * OP_COUNT, OP_SHL, nshl);
      bump(cstep + K_VEC_DIV * OP_COUNT, OP_DIV, ndiv);
      cta_max2(vmax, 0);
      if (tid == 0) {
        vmx_me[j + 1] = s_mx[0];
        atomicMax(reinterpret_cast<unsigned long long*>(vmx + static_cast<size_t>(kVmxRows - 1) * vst + j + 1),
                  static_cast<unsigned long long>(s_mx[0]));  // all CTAs: the SpMV's certificate
      }
    }
  }
  ARN_TS(123)
#undef ARN_TS
}


__device__ __forceinline__ int4 lds128i(unsigned a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void lds128l(unsigned a, i64& x, i64& y) {
  asm volatile("ld.shared.v2.s64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a) : "memory");
}

// yperm[p] = y[p_row[p]] (FP path: divided by gamma with one correctly rounded
// division per entry, as refine.cpp:17 forms b_k = r / gamma) -- one coalesced
// streaming pass that turns the wavefront's per-level right-hand-side
// gathers into one contiguous bulk copy
__device__ __forceinline__ u64 abs_u64(i64 v) { return v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v); }

__device__ __forceinline__ void warp_max_to(u64 m, u64* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, static_cast<u64>(__shfl_down_sync(0xffffffffu, m, o)));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(reinterpret_cast<unsigned long long*>(dst), static_cast<unsigned long long>(m));
}

template <typename T>
__global__ void __launch_bounds__(256) k_tri_gather(int n, const int* __restrict__ p_row,
                                                    const T* __restrict__ y, T* __restrict__ yperm,
                                                    const Ctl* ctl, const double* prescale, u64* ymax) {
  if (cycle_over(ctl)) return;
  u64 m = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {  // grid is capped
    T v = y[__ldg(p_row + p)];
    if constexpr (std::is_same<T, double>::value) {
      if (prescale != nullptr) v = __ddiv_rn(v, __longlong_as_double(*reinterpret_cast<const long long*>(prescale)));
    } else {
      m = max(m, abs_u64(v));
    }
    yperm[p] = v;
  }
  if (ymax != nullptr) {  // block max, then one atomic per block (a single hot word)
    __shared__ u64 sm[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, static_cast<u64>(__shfl_down_sync(0xffffffffu, m, o)));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, sm[w]);
      if (m) atomicMax(reinterpret_cast<unsigned long long*>(ymax), static_cast<unsigned long long>(m));
    }
  }
}

constexpr int kTriCompute = 256;
constexpr int kTriThreads = kTriCompute + 32;  // + bulk-loader warp

struct TriSmem {  // byte offsets of the dynamic shared-memory regions
  size_t rows, xptr, ring, bars, total;
  unsigned ring_slot;
};

// zt (tile values) | segment starts | (spare) | ring of L slots
// [records | rhs run] | mbarriers
template <int MAXD, bool COMPACT>
__host__ __device__ constexpr int tri_rec_bytes() {
  return COMPACT ? 16 + 8 * MAXD : 32 + 12 * MAXD;
}

template <int MAXD, bool COMPACT>
__host__ __device__ inline TriSmem tri_smem_layout(int tile_cap, int seg_cap, int L, int max_ext) {
  constexpr int REC = tri_rec_bytes<MAXD, COMPACT>();
  TriSmem m;
  size_t o = (static_cast<size_t>(tile_cap) * 8 + 15) & ~size_t(15);
  m.rows = o;
  o += sizeof(int) * static_cast<size_t>(seg_cap);
  m.xptr = o;
  o += sizeof(int) * static_cast<size_t>(seg_cap);
  o = (o + 127) & ~size_t(127);
  m.ring = o;
  m.ring_slot = kTriSegRows * REC + 8 * (kTriSegRows + 2);
  (void)max_ext;
  o += static_cast<size_t>(L) * m.ring_slot;
  o = (o + 15) & ~size_t(15);
  m.bars = o;
  o += 16 * static_cast<size_t>(L);  // full, empty
  m.total = o;
  return m;
}

template <typename T, bool BACKWARD, int MAXD, bool COMPACT>
__global__ void __launch_bounds__(kTriThreads) k_tri(TriArgs a, const T* __restrict__ yperm, T* out,
                                                     const Ctl* ctl, int seg_cap, int L, int pf) {
  constexpr bool FP = std::is_same<T, double>::value;
  constexpr int REC = tri_rec_bytes<MAXD, COMPACT>();
  constexpr unsigned YOFF = kTriSegRows * REC;                 // rhs run in a ring slot
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ int s_tile;
  if (cycle_over(ctl)) return;
  const TriSmem lay = tri_smem_layout<MAXD, COMPACT>(a.tile_cap, seg_cap, L, a.max_seg_ext);
  unsigned zt_s = smem_u32(smem_raw);
  asm volatile("" : "+r"(zt_s));  // kept in a register (not re-derived from %cgactaid each level)
  int* s_rows = reinterpret_cast<int*>(smem_raw + lay.rows);
  int* s_xptr = reinterpret_cast<int*>(smem_raw + lay.xptr);
  const unsigned ring_s = smem_u32(smem_raw + lay.ring);
  const unsigned full_s = smem_u32(smem_raw + lay.bars);
  const unsigned empty_s = full_s + 8u * static_cast<unsigned>(L);
  if (threadIdx.x == 0) {
    s_tile = atomicAdd(a.ticket, 1);
    for (int k = 0; k < L; ++k) {
      mbar_init_s(full_s + 8u * k, 1);  // the bulk loader's arrive (+ tx bytes)
      mbar_init_s(empty_s + 8u * k, kTriCompute / 32);
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
    for (int q = threadIdx.x; q <= nsg; q += blockDim.x) {
      s_rows[q] = __ldg(a.seg_rows + sb + q);
      s_xptr[q] = __ldg(a.seg_xptr + sb + q);
    }
  __syncthreads();
  auto seg_row = [&](int q) { return seg_in_smem ? s_rows[q] : __ldg(a.seg_rows + sb + q); };
  auto seg_xp = [&](int q) { return seg_in_smem ? s_xptr[q] : __ldg(a.seg_xptr + sb + q); };
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#ifdef IGM_TRI_TRACE
  unsigned long long* tsb = (!BACKWARD && g_tri_ts != nullptr && tile == g_tri_ts_tile) ? g_tri_ts : nullptr;
#else
  constexpr unsigned long long* tsb = nullptr;  // phase timestamps compiled out
#endif

  if (warp == kTriCompute / 32) {  // ---------------- bulk loader (one lane)
    if (lane != 0) return;
    int k = 0;
    unsigned ph = 1;  // parity of the previous use of slot k (first L levels: none)
    // records and rhs runs of levels q+L .. q+pf-1 are pulled into L2 ahead of
    // their shared-memory copy: the ring (L slots, bounded by the tile's
    // values in shared memory) then waits on an L2 hit, not on HBM latency
    auto prefetch = [&](int qq) {
      if (qq >= nsg) return;
      const int p0 = seg_row(qq), pc = seg_row(qq + 1) - p0;
      const int pa = p0 & ~1, pyc = ((p0 + pc + 1) & ~1) - pa;
      bulk_prefetch_l2(a.p_rec + static_cast<size_t>(p0) * REC, static_cast<unsigned>(pc * REC));
      bulk_prefetch_l2(yperm + pa, static_cast<unsigned>(pyc * 8));
    };
    for (int q = L; q < pf; ++q) prefetch(q);
    for (int q = 0; q < nsg; ++q) {
      if (pf > L) prefetch(q + pf);
      if (q >= L) mbar_wait_s(empty_s + 8u * k, ph);
      const int s0 = seg_row(q), c = seg_row(q + 1) - s0;
      const unsigned slot = ring_s + static_cast<unsigned>(k) * lay.ring_slot;
      const unsigned fb = full_s + 8u * k;
      // the rhs run is widened to 16-byte alignment: it lands at offset s0 & 1
      const int ya = s0 & ~1, yc = ((s0 + c + 1) & ~1) - ya;
      mbar_arrive_expect_tx_s(fb, static_cast<unsigned>(c * REC + yc * 8));
      bulk_g2s_s(slot, a.p_rec + static_cast<size_t>(s0) * REC, static_cast<unsigned>(c * REC), fb);
      bulk_g2s_s(slot + YOFF, yperm + ya, static_cast<unsigned>(yc * 8), fb);
      if (tsb && q < 2048) tsb[q * 8 + 7] = gtime();
      if (++k == L) {
        k = 0;
        ph ^= 1u;
      }
    }
    return;
  }

  // ---------------- compute warps
  // Each level's row record (dependency slots and factors, magic, rhs) is
  // read from the ring into registers and its cross-tile words are loaded
  // together with it.
  const int tid = threadIdx.x;
  const unsigned ring_end = ring_s + static_cast<unsigned>(L) * lay.ring_slot;
  const unsigned my_rec = static_cast<unsigned>(tid) * REC;
  struct Rec {
    int row, info, nd, xb;
    i64 mag, diag, y;
    int ci[MAXD];
    i64 v[MAXD];
    u64 wv[MAXD], wt[MAXD];  // cross-tile words (value, tag)
    unsigned zaddr, bar;
    bool have;
  };
  Rec R;
  unsigned f_slot = ring_s, f_bar = 0, f_ph = 0;  // ring position of the next level to fetch
  int s_f = seg_row(0);
  auto fetch = [&](int q, Rec& r) {
    r.have = false;
    r.bar = f_bar;
    if (q >= nsg) return;
    mbar_wait_s(full_s + f_bar, f_ph);
    const unsigned sl = f_slot;
    f_bar += 8;
    f_slot += lay.ring_slot;
    if (f_slot == ring_end) {
      f_slot = ring_s;
      f_bar = 0;
      f_ph ^= 1u;
    }
    const int s0 = s_f, s1 = seg_row(q + 1);
    s_f = s1;
    if (tid >= s1 - s0) return;
    const unsigned ra = sl + my_rec;
    const int4 hdr = lds128i(ra);
    if constexpr (COMPACT) {
      r.row = hdr.x;
      r.info = hdr.y & 0xffff;
      r.nd = hdr.y >> 16;
      r.mag = static_cast<i64>(static_cast<u64>(static_cast<unsigned>(hdr.z)) |
                               (static_cast<u64>(static_cast<unsigned>(hdr.w)) << 32));
      const int slot = s0 + tid;
      r.xb = r.nd > MAXD ? __ldg(a.p_xrp + slot) : 0;
      if constexpr (FP) r.diag = __ldg(a.p_diag + slot);  // used after the barrier
#pragma unroll
      for (int d = 0; d < MAXD; d += 4) {
        const int4 c4 = lds128i(ra + 16 + 4 * d);
        r.ci[d] = c4.x;
        r.ci[d + 1] = c4.y;
        r.ci[d + 2] = c4.z;
        r.ci[d + 3] = c4.w;
        const int4 v4 = lds128i(ra + 16 + 4 * MAXD + 4 * d);
        r.v[d] = v4.x;
        r.v[d + 1] = v4.y;
        r.v[d + 2] = v4.z;
        r.v[d + 3] = v4.w;
      }
    } else {
      r.row = hdr.x;
      r.nd = hdr.y;
      r.info = hdr.z;
      r.xb = hdr.w;
      lds128l(ra + 16, r.mag, r.diag);
#pragma unroll
      for (int d = 0; d < MAXD; d += 4) {
        const int4 c4 = lds128i(ra + 32 + 4 * d);
        r.ci[d] = c4.x;
        r.ci[d + 1] = c4.y;
        r.ci[d + 2] = c4.z;
        r.ci[d + 3] = c4.w;
      }
#pragma unroll
      for (int d = 0; d < MAXD; d += 2) lds128l(ra + 32 + 4 * MAXD + 8 * d, r.v[d], r.v[d + 1]);
    }
    r.y = lds64(sl + YOFF + 8u * static_cast<unsigned>(tid + (s0 & 1)));
    r.zaddr = zt_s + 8u * static_cast<unsigned>(s0 + tid - pb);
    r.have = true;
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (r.ci[d] < 0) xz_load(a.xz + ~r.ci[d], r.wv[d], r.wt[d]);
  };
  u64 zmx = 0;   // max |z| of this thread's rows (integer path)
  i64 zlast = 0;
  // one level: barrier, the row, release the level's ring slot
  auto level = [&](int q, const Rec& cur) {
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 2] = gtime();
    bar_sync(1, kTriCompute);  // level q-1 values of this tile are in shared memory
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 3] = gtime();
#ifndef IGM_TRI_SKELETON
    if (cur.have) {
      if constexpr (!FP) zmx = max(zmx, abs_u64(zlast));
      // every dependency's shared-memory load issued back to back (no
      // branch between them), then the cross-tile words selected by
      // predicate; a word not yet published when it was loaded with the
      // record is re-polled on a separate (rare) path
      i64 zb[MAXD];
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        const int c = cur.ci[d];
        zb[d] = lds64(zt_s + 8u * static_cast<unsigned>(c < 0 ? 0 : c));
      }
      unsigned stale = 0;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (cur.ci[d] < 0) {
          const bool ok = cur.wt[d] == (a.epoch ^ cur.wv[d]);
#ifdef IGM_TRI_TRACE
          if (tsb && q < 2048) {
            if (!ok) atomicAdd(tsb + q * 8 + 0, 1ull);
            atomicAdd(tsb + q * 8 + 1, 1ull);
          }
#endif
          zb[d] = ok ? static_cast<i64>(cur.wv[d]) : zb[d];
          stale |= ok ? 0u : (1u << d);
        }
      }
      if (stale) {
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
          if ((stale >> d) & 1u) zb[d] = static_cast<i64>(xz_wait(a.xz + ~cur.ci[d], a.epoch));
      }
      auto extra = [&](int d) {  // dependency beyond the record stride (rare)
        const int c = __ldg(a.p_xdep + cur.xb + d - MAXD);
        return c >= 0 ? lds64(zt_s + 8u * static_cast<unsigned>(c)) : static_cast<i64>(xz_wait(a.xz + ~c, a.epoch));
      };
      T z;
      if constexpr (FP) {
        double acc = __longlong_as_double(cur.y);
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
          if (d < cur.nd) acc = __dsub_rn(acc, __dmul_rn(__ll2double_rn(cur.v[d]), __longlong_as_double(zb[d])));
        for (int d = MAXD; d < cur.nd; ++d)
          acc = __dsub_rn(acc, __dmul_rn(__ll2double_rn(__ldg(a.p_xval + cur.xb + d - MAXD)),
                                         __longlong_as_double(extra(d))));
        z = __ddiv_rn(acc, __ll2double_rn(cur.diag));
      } else {
        // unused slots hold factor 0 at local slot 0: exact zero terms
        u64 sx = 0;
#ifndef IGM_TRI_NODEP
#pragma unroll
        for (int d = 0; d < MAXD; ++d) sx += static_cast<u64>(cur.v[d]) * static_cast<u64>(zb[d]);
#endif
        for (int d = MAXD; d < cur.nd; ++d)
          sx += static_cast<u64>(__ldg(a.p_xval + cur.xb + d - MAXD)) * static_cast<u64>(extra(d));
        const i64 acc = static_cast<i64>(static_cast<u64>(cur.y) - sx);
        SDivMagic gm;
        gm.u.m = static_cast<u64>(cur.mag);
        gm.u.sh1 = cur.info & 1;
        gm.u.sh2 = (cur.info >> 1) & 127;
        gm.den_neg = (cur.info >> 8) & 1;
        gm.den_is_m1 = 0;  // only the (separate) counting pass needs it
#ifdef IGM_TRI_NODIV
        z = acc ^ static_cast<i64>(gm.u.m);
#else
        z = sdiv(acc, gm);
#endif
      }
      i64 zbits;
      if constexpr (FP) {
        zbits = __double_as_longlong(z);
      } else {
        zbits = z;
        zlast = z;  // folded into zmx off the critical path (next level)
      }
      sts64(cur.zaddr, zbits);
#ifndef IGM_TRI_NOSTORE
#ifndef IGM_TRI_NOOUT
      out[cur.row] = z;
#endif
      if (cur.info & (1 << 10)) xz_put(a.xz + cur.row, static_cast<u64>(zbits), a.epoch);  // read by another tile
#endif
    }
#endif
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 5] = gtime();
    __syncwarp();
    if (lane == 0) mbar_arrive_s(empty_s + cur.bar);
    if (tsb && tid == 0 && q < 2048) tsb[q * 8 + 6] = gtime();
  };
  // Each level's record is read (and its cross-tile loads issued) right
  // before the level's barrier, so their latency overlaps the barrier wait.
  // Measured faster than reading records (and cross-tile words) one to four
  // levels ahead into a register ring -- also with a deliberate two-level lag
  // that waits for every word one level before its use: 1.40 vs 1.06
  // us/level at 128^3, 0.87 vs 0.68 for a single brick.
  for (int q = 0; q < nsg; ++q) {
    fetch(q, R);
    level(q, R);
  }
  if constexpr (!FP) warp_max_to(max(zmx, abs_u64(zlast)), a.zmax);
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
                                                   const Ctl* ctl, const u64* stats, double maxl, int maxd) {
  __shared__ int s_skip;
  if (cycle_over(ctl)) return;
  // every partial sum of every row is bounded by max|y| + maxd * max|l| * max|z|:
  // below 2^63 no product, subtraction or INT64_MIN / -1 can overflow, so the
  // exact count is zero (the bound is taken in FP64 with a factor-2 margin)
  if (threadIdx.x == 0) {
    const double b = __dadd_rn(static_cast<double>(stats[0]),
                               static_cast<double>(maxd) * maxl * static_cast<double>(stats[1]));
    s_skip = b < 4611686018427387904.0;  // 2^62
  }
  __syncthreads();
  if (s_skip) return;
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

// The two recounts of one preconditioner application (forward: y -> mid,
// backward: mid -> z) in ONE launch on a small grid: in a configured run both
// magnitude bounds hold and every CTA returns at once, so the cost per
// Arnoldi step is one short launch instead of two memsets and two launches
// on a full grid.  The last CTA to finish clears both factors' [max|y|,
// max|z|] words for the next application (no memset nodes).
struct TriCnt {
  int n;
  const int* rp;
  const int* ci;
  const i64* val;
  const i64* diag;
  u64* stats;  // [max|y|, max|z|, CTAs done]
  double maxl;
  int maxd;
};
__device__ __forceinline__ void tri_recount(const TriCnt& t, const i64* __restrict__ y, const i64* __restrict__ z,
                                            u64& nmul, u64& nsub, u64& ndiv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += gridDim.x * blockDim.x) {
    i64 acc = y[i];
    for (int k = t.rp[i]; k < t.rp[i + 1]; ++k) {
      const i64 l = t.val[k], zj = z[t.ci[k]];
      const i64 p = wmul(l, zj);
      nmul += mul_ovf(l, zj);
      nsub += sub_ovf(acc, p);
      acc = wsub(acc, p);
    }
    ndiv += (acc == INT64_MIN && t.diag[i] == -1);
  }
}
__global__ void __launch_bounds__(256) k_tri_count_pair(TriCnt lo, TriCnt up, const i64* __restrict__ y,
                                                        const i64* __restrict__ mid, const i64* __restrict__ z,
                                                        u64* cnt, const Ctl* ctl) {
  __shared__ int s_skip[2];
  if (threadIdx.x == 0) {
    auto holds = [](const TriCnt& t) {
      const double b = __dadd_rn(static_cast<double>(ld_cg_u64(t.stats)),
                                 static_cast<double>(t.maxd) * t.maxl * static_cast<double>(ld_cg_u64(t.stats + 1)));
      return b < 4611686018427387904.0;  // 2^62, as in k_tri_count
    };
    const bool over = cycle_over(ctl);
    s_skip[0] = over || holds(lo);
    s_skip[1] = over || holds(up);
  }
  __syncthreads();
  if (!s_skip[0] || !s_skip[1]) {
    u64 nmul = 0, nsub = 0, ndiv = 0;
    if (!s_skip[0]) tri_recount(lo, y, mid, nmul, nsub, ndiv);
    if (!s_skip[1]) tri_recount(up, mid, z, nmul, nsub, ndiv);
    bump(cnt, OP_MUL, nmul);
    bump(cnt, OP_SUB, nsub);
    bump(cnt, OP_DIV, ndiv);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned long long*>(lo.stats + 2), 1ull) == gridDim.x - 1) {
      lo.stats[0] = lo.stats[1] = lo.stats[2] = 0;
      up.stats[0] = up.stats[1] = 0;
      __threadfence();
    }
  }
}

TriArgs tri_args(const DevTri& t) {
  TriArgs a;
  a.n = t.n;
  a.ntiles = t.ntiles;
  a.tile_pbase = t.tile_pbase;
  a.tile_seg = t.tile_seg;
  a.seg_rows = t.seg_rows;
  a.seg_xptr = t.seg_xptr;
  a.seg_xrow = t.seg_xrow;
  a.p_xdep = t.p_xdep;
  a.p_xval = t.p_xval;
  a.p_rec = t.p_rec;
  a.p_xrp = t.p_xrp;
  a.p_diag = t.p_diag;
  a.tile_cap = t.tile_cap;
  a.max_seg_ext = t.max_seg_ext;
  a.xz = t.xz;
  a.zmax = t.stats + 1;
  a.epoch = 0;
  a.ticket = t.ticket;
  return a;
}

}  // namespace

// device fast paths of fx_core.cuh (isqrt, division magic, truncating and
// 128/64 division) on n input pairs: out[4i..4i+3]
__global__ void k_fx_selftest(int n, const u64* a, const u64* b, u64* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 x = a[i], y = b[i] ? b[i] : 1;
  out[4 * i + 0] = isqrt_u64(x);
  out[4 * i + 1] = make_udiv(y).m;
  const i64 sx = static_cast<i64>(x), sy = static_cast<i64>(y);
  out[4 * i + 2] = (sx == INT64_MIN && sy == -1) ? 0 : static_cast<u64>(sdiv_trunc(sx, sy));
  out[4 * i + 3] = udiv128_64_dev(x % y, ~x ^ y, y);
}

int debug_fx_selftest(int n, const u64* a, const u64* b, u64* out) {
  u64 *da, *db, *dout;
  cudaMalloc(&da, 8 * static_cast<size_t>(n) + 8);
  cudaMalloc(&db, 8 * static_cast<size_t>(n) + 8);
  cudaMalloc(&dout, 32 * static_cast<size_t>(n) + 8);
  cudaMemcpy(da, a, 8 * static_cast<size_t>(n), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, 8 * static_cast<size_t>(n), cudaMemcpyHostToDevice);
  k_fx_selftest<<<(n + 255) / 256, 256>>>(n, da, db, dout);
  const cudaError_t e = cudaMemcpy(out, dout, 32 * static_cast<size_t>(n), cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dout);
  return e == cudaSuccess ? 0 : 1;
}

// arm (out == nullptr: record step j of the following k_arnoldi2 launches) /
// read and disarm (out: cap words, CTA-major, kArnTsSlots per CTA)
int debug_arn_ts(int j, unsigned long long* out, int cap) {
  static unsigned long long* buf = nullptr;
  constexpr int kMaxCta = 1024;
  if (out == nullptr) {
    if (buf == nullptr) cudaMalloc(&buf, sizeof(unsigned long long) * kMaxCta * kArnTsSlots);
    cudaMemset(buf, 0, sizeof(unsigned long long) * kMaxCta * kArnTsSlots);
    cudaMemcpyToSymbol(g_arn_ts, &buf, sizeof(buf));
    cudaMemcpyToSymbol(g_arn_ts_j, &j, sizeof(int));
    return kArnTsSlots;
  }
  cudaDeviceSynchronize();
  const int n = cap < kMaxCta * kArnTsSlots ? cap : kMaxCta * kArnTsSlots;
  cudaMemcpy(out, buf, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  const int off = -1;
  cudaMemcpyToSymbol(g_arn_ts_j, &off, sizeof(int));
  return kArnTsSlots;
}

// ---------------------------------------------------------------------------
// FP64 engine (Engine::floating_point: refine.cpp:47-86, refsolve.cpp:9-105)
// reconstruct_fp (split.cpp:177-191): vals[k] = sum_l ldexp(double(c_l[k]), -alpha_l), from 0.0
__global__ void k_recon_vals(long long nnz, int s, const i64* __restrict__ vals, const int* __restrict__ alphas,
                             double* __restrict__ out) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int l = 0; l <= s; ++l) acc = __dadd_rn(acc, ldexp(__ll2double_rn(vals[l * nnz + k]), -alphas[l]));
    out[k] = acc;
  }
}

// MGS dot h = sum_l w_l v_l in a fixed tree order (deterministic; the
// reference's sequential sum has no cheap exact parallel form for mixed
// signs -- SURVEY.md §8(f) row 2 compares this engine by iteration counts)
constexpr int kFdotBlocks = 592;
__global__ void __launch_bounds__(256) k_fdot_partial(long long n, const double* __restrict__ w,
                                                      const double* __restrict__ v, double* part) {
  __shared__ double sh[8];
  double acc = 0.0;
  for (long long l = blockIdx.x * 256LL + threadIdx.x; l < n; l += static_cast<long long>(gridDim.x) * 256)
    acc = __dadd_rn(acc, __dmul_rn(w[l], v[l]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t = __dadd_rn(t, sh[i]);
    part[blockIdx.x] = t;
  }
}
__global__ void __launch_bounds__(256) k_fdot_final(int nb, const double* __restrict__ part, double* h) {
  __shared__ double sh[8];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += 256) acc = __dadd_rn(acc, part[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t = __dadd_rn(t, sh[i]);
    *h = t;
  }
}
// w -= h v (refsolve.cpp:58, no contraction)
__global__ void k_faxpy(long long n, double* __restrict__ w, const double* __restrict__ v, const double* h) {
  const double hv = *h;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<long long>(gridDim.x) * blockDim.x)
    w[l] = __dsub_rn(w[l], __dmul_rn(hv, v[l]));
}
// out = w / *d (refsolve.cpp:37, 69)
__global__ void k_fscale(long long n, const double* __restrict__ w, double* __restrict__ out, const double* d) {
  const double dv = *d;
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<long long>(gridDim.x) * blockDim.x)
    out[l] = __ddiv_rn(w[l], dv);
}
// x += gamma * (0.0 + sum_j wts_j v_j), j in order (refsolve.cpp:95-100, refine.cpp:87)
// mode 1: x += gamma * (0.0 + sum_j wts_j v_j) (the refinement's correction);
// mode 0: x = x0 + w_0 v_0 + w_1 v_1 + ... accumulated onto x0 (fp_cycle)
__global__ void k_fxupdate(long long n, int dim, const double* __restrict__ basis, const double* __restrict__ wts,
                           double gamma, double* __restrict__ x, int mode) {
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    double acc = mode == 0 ? x[l] : 0.0;
    for (int j = 0; j < dim; ++j) acc = __dadd_rn(acc, __dmul_rn(wts[j], basis[static_cast<long long>(j) * n + l]));
    x[l] = mode == 0 ? acc : __dadd_rn(x[l], __dmul_rn(gamma, acc));
  }
}

// ---------------------------------------------------------------------------
// launchers

// every launch is counted and checked: a launch-configuration error (not
// reported by a later synchronisation) or a sticky device fault turns into
// IGM_CUDA_ERROR at the C-ABI boundary instead of stale outputs
static void launch_check_at(int line) {
  ++g_launches;
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw LaunchFail(std::string("kernel launch (kernels.cu:") + std::to_string(line) + "): " + cudaGetErrorString(e));
  }
}
#define LAUNCH_CHECK() launch_check_at(__LINE__)

int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

bool PerDevice::first(int device) {
  const unsigned long long bit = 1ull << (device & 63);
  return (bits.fetch_or(bit) & bit) == 0;
}

// vb (checked mode, may be null): a device word that bounds |v| (the maximum
// k_arnoldi recorded over all CTAs when it wrote this basis vector)
void launch_spmv_int(cudaStream_t st, const DevSplit& m, int s, const i64* v, i64* out, u64* cnt,
                     const Ctl* ctl, bool checked, const u64* vb) {
  ProfScope prof_(st, KC_SPMV);
  // long rows (mean >= 16, max <= 32 entries: 27-point stencils): the staged kernel
  static const bool staged_on = [] {
    const char* e = std::getenv("IGM_SPMV_STAGED");
    return !(e && e[0] == '0');
  }();
  static const bool r8_on = [] {
    const char* e = std::getenv("IGM_SPMV_R8");
    return !(e && e[0] == '0');
  }();
  if (r8_on && s == 0 && m.max_row > 0 && m.max_row <= 16 && m.sell_vals == nullptr) {
    const int g = std::max(1, (m.n + 127) / 128);
    const int a0 = m.h_alphas.empty() ? 0 : m.h_alphas[0];
    if (m.max_row <= 8) {
      if (checked)
        k_spmv_int_r8<true><<<g, 128, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, a0, v, out, cnt, ctl, m.max_abs0, vb);
      else
        k_spmv_int_r8<false><<<g, 128, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, a0, v, out, cnt, ctl, 0, nullptr);
    } else {
      if (checked)
        k_spmv_int_r8<true, 16><<<g, 128, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, a0, v, out, cnt, ctl,
                                                   m.max_abs0, vb);
      else
        k_spmv_int_r8<false, 16><<<g, 128, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, a0, v, out, cnt, ctl, 0,
                                                    nullptr);
    }
    LAUNCH_CHECK();
    return;
  }
  if (s == 0 && m.sell_vals != nullptr) {
    const int g = std::max(1, ((m.n + 31) / 32 * 32 + 127) / 128);
    const int a0 = m.h_alphas.empty() ? 0 : m.h_alphas[0];
    if (checked)
      k_spmv_int_sell<true><<<g, 128, 0, st>>>(m.n, m.sell_w, m.sell_vals, m.sell_cols, a0, v, out, cnt, ctl,
                                               m.max_abs0, vb);
    else
      k_spmv_int_sell<false><<<g, 128, 0, st>>>(m.n, m.sell_w, m.sell_vals, m.sell_cols, a0, v, out, cnt, ctl, 0,
                                                nullptr);
    LAUNCH_CHECK();
    return;
  }
  if (staged_on && m.max_row > 0 && m.max_row <= kSpMaxRow && static_cast<long long>(m.nnz) >= 16LL * m.n) {
    const int tiles = (m.n + kSpRows - 1) / kSpRows;
    const int g = std::max(1, std::min((tiles + kSpWarps - 1) / kSpWarps, num_sms(cur_device()) * 12));
    if (checked)
      k_spmv_int_staged<true><<<g, kSpWarps * 32, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v,
                                                           out, cnt, ctl);
    else
      k_spmv_int_staged<false><<<g, kSpWarps * 32, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v,
                                                            out, cnt, ctl);
    LAUNCH_CHECK();
    return;
  }
  const int nt = 256;
  const int g = static_cast<int>((m.n + nt - 1) / nt > 0 ? (m.n + nt - 1) / nt : 1);
  if (checked)
    k_spmv_int<true><<<g, nt, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v, out, cnt, ctl);
  else
    k_spmv_int<false><<<g, nt, 0, st>>>(m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, s, v, out, cnt, ctl);
  LAUNCH_CHECK();
}

u64 device_max_abs(cudaStream_t st, long long n, const i64* a) {
  if (n <= 0) return 0;
  unsigned long long* d = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&d), sizeof(unsigned long long)) != cudaSuccess) return ~0ull;
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), st);
  k_max_abs<<<grid_for(n, 256), 256, 0, st>>>(n, a, d);
  LAUNCH_CHECK();
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  return h;
}

void launch_build_sell(cudaStream_t st, int n, int w, const int* rp, const int* ci, const i64* vals, i64* sv,
                       int* sc) {
  if (n <= 0) return;
  k_build_sell<<<(n + 127) / 128, 128, 0, st>>>(n, w, rp, ci, vals, sv, sc);
  LAUNCH_CHECK();
}

int device_max_row(cudaStream_t st, int n, const int* rp) {
  if (n <= 0) return 0;
  int* d = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&d), sizeof(int)) != cudaSuccess) return 0;
  cudaMemsetAsync(d, 0, sizeof(int), st);
  k_max_row<<<grid_for(n, 256), 256, 0, st>>>(n, rp, d);
  LAUNCH_CHECK();
  int h = 0;
  cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  return h;
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

size_t norm2_scratch_bytes(long long n) {
  return sizeof(N2Blk) * static_cast<size_t>(std::max<long long>(1, (n + kN2Chunk - 1) / kN2Chunk));
}

// exact norm2 chain of v (or of the decoded raw words when raw != null)
static void norm2_enqueue(cudaStream_t st, long long n, const double* v, const i64* raw, double scale,
                          double* out, Ctl* ctl, int mode, int basis_idx, void* scratch,
                          const double* start = nullptr) {
  if (norm2_serial_forced()) {
    k_norm2_serial<<<1, 256, 0, st>>>(n, v, raw, scale, out, ctl, mode, basis_idx, start);
  } else if (n <= 2 * kN2Chunk || scratch == nullptr) {
    k_norm2_exact<<<1, kN2Threads, 0, st>>>(n, v, raw, scale, out, ctl, mode, basis_idx, start);
  } else {
    const int nblk = static_cast<int>((n + kN2Chunk - 1) / kN2Chunk);
    N2Blk* blk = static_cast<N2Blk*>(scratch);
    k_n2_bsum<<<nblk, kN2BThreads, 0, st>>>(n, v, raw, scale, blk, ctl, mode, basis_idx);
    k_n2_baut<<<nblk, kN2BThreads, 0, st>>>(n, v, raw, scale, blk, ctl, mode, basis_idx, start);
    k_n2_walk<<<1, kN2Threads, 0, st>>>(n, nblk, v, raw, scale, blk, out, ctl, mode, basis_idx, start);
  }
  LAUNCH_CHECK();
}

void launch_norm2_serial(cudaStream_t st, long long n, const double* v, double* out, Ctl* ctl, int mode,
                         void* scratch, const double* start) {
  ProfScope prof_(st, KC_NORM2);
  norm2_enqueue(st, n, v, nullptr, 1.0, out, ctl, mode, 0, scratch, start);
}

void launch_basis_norms(cudaStream_t st, long long n, int nb, int f, const i64* basis, void* scratch,
                        double* out, Ctl* ctl) {
  ProfScope prof_(st, KC_NORM2);
  for (int k = 0; k < nb; ++k)
    norm2_enqueue(st, n, nullptr, basis + static_cast<long long>(k) * n, ldexp(1.0, -f), out, ctl, 4, k, scratch);
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
  const int g = static_cast<int>(std::max<long long>(1, std::min<long long>(2LL * num_sms(cur_device()), (n / 4 + nt - 1) / nt)));
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
  const int sms = num_sms(cur_device());
  const int g = grid_for(n, nt) > 2 * sms ? 2 * sms : grid_for(n, nt);
  if (checked)
    k_fx_red<true><<<g, nt, 0, st>>>(n, mode, v, w, b1, b2, acc, abs_out, cnt);
  else
    k_fx_red<false><<<g, nt, 0, st>>>(n, mode, v, w, b1, b2, acc, abs_out, cnt);
  LAUNCH_CHECK();
}

size_t exact_adds_scratch_bytes(long long n) {
  return sizeof(__int128) * static_cast<size_t>(std::max<long long>(1, (n + kAddChunk - 1) / kAddChunk));
}

void launch_exact_adds(cudaStream_t st, long long n, int mode, const i64* w, const i64* v, int b1, int b2,
                       const u64* cert, const Ctl* ctl, u64* cnt_add, void* scratch) {
  if (n <= 0) return;
  ProfScope prof_(st, KC_OTHER);
  const int nblk = static_cast<int>((n + kAddChunk - 1) / kAddChunk);
  __int128* blk = static_cast<__int128*>(scratch);
  k_adds_blk<<<nblk, kAddThreads, 0, st>>>(n, mode, w, v, b1, b2, cert, ctl, blk);
  k_adds_scan<<<1, 32, 0, st>>>(nblk, cert, ctl, blk);
  k_adds_count<<<nblk, kAddThreads, 0, st>>>(n, mode, w, v, b1, b2, cert, ctl, blk, cnt_add);
  g_launches += 3;
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
                    u64* cnt, const Ctl* ctl, bool checked, u64* vmax_out) {
  ProfScope prof_(st, KC_VEC_DIV);
  const int nt = 512;
  const int g = grid_for(n, nt);
  if (checked)
    k_vec_div<true><<<g, nt, 0, st>>>(n, w, out, f, sh.div_b1, sh.div_b2, cnt, ctl, vmax_out);
  else
    k_vec_div<false><<<g, nt, 0, st>>>(n, w, out, f, sh.div_b1, sh.div_b2, cnt, ctl, nullptr);
  LAUNCH_CHECK();
}

void launch_step_scalar(cudaStream_t st, int j, int f, ShiftsD sh, const u64* acc_col,
                        const u64* abs_col, const u64* nacc, const u64* nabs, i64* hess, int ld,
                        i64* g, i64* cs, i64* sn, i64* gabs, const i64* w, u64* cnt_step, Ctl* ctl,
                        int checked, int acc_st, int abs_st, const u64* norm_mul) {
  ProfScope prof_(st, KC_SCALAR);
  if (!norm_mul) norm_mul = cnt_step + K_NORM * OP_COUNT + OP_MUL;
  k_step_scalar<<<1, 32, 0, st>>>(j, f, sh, acc_col, acc_st, abs_col, abs_st, nacc, nabs, norm_mul, hess, ld, g,
                                 cs, sn, gabs, w, cnt_step, ctl, checked);
  LAUNCH_CHECK();
}

// rows per CTA and dynamic shared memory of the persistent step kernel; 0
// when w and one basis slice do not fit on chip (the pass kernels are used)
long long arnoldi_slice(long long n, int device) {
  static const int off = [] {
    const char* e = std::getenv("IGM_ARNOLDI");
    return e && e[0] == '0' ? 1 : 0;
  }();
  if (off || n < 4096 || n % 4 != 0) return 0;  // 32-byte aligned basis vectors
  const int G = num_sms(device);
  const long long S = ((n + G - 1) / G + 3) / 4 * 4;
  const size_t bytes = static_cast<size_t>(S) * 16;
  if (bytes > kArnSmemMax) return 0;
  return S;
}

// counted grid-barrier arrivals per CTA of one step's launch: k_arnoldi counts
// every pass barrier (j + 1) plus two; k_arnoldi2's pass barriers live in the
// snapshot slots, only the two around the scalar step use the counter
static bool arnoldi_v2(long long S) {
  static const bool v2 = [] {
    const char* e = std::getenv("IGM_ARNOLDI2");
    return e == nullptr || e[0] != '0';
  }();
  return v2 && S <= 4LL * kArn2Threads * kArn2Q;
}
int arnoldi_barriers(int j, long long S) { return arnoldi_v2(S) ? 2 : j + 3; }

void launch_arnoldi(cudaStream_t st, long long n, int j, long long S, const i64* w, i64* basis, u64* accj,
                    u64* absj, u64* nacc, u64* nabs, int f, ShiftsD sh, u64* cstep, i64* hess, int ld, i64* g,
                    i64* cs, i64* sn, i64* gabs, Ctl* ctl, unsigned gbase, bool checked, u64* vmx, u64* snapj) {
  ProfScope prof_(st, KC_MGS);
  const int dev = cur_device();
  const int G = num_sms(dev);
  const size_t smem = static_cast<size_t>(S) * 16;
  static PerDevice attr;  // the attribute is per device
  if (attr.first(dev)) {
    cudaFuncSetAttribute(k_arnoldi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kArnSmemMax));
    cudaFuncSetAttribute(k_arnoldi<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kArnSmemMax));
  }
  void* args[] = {&n, &j, &S, &w, &basis, &accj, &absj, &nacc, &nabs, &f, &sh, &cstep,
                  &hess, &ld, &g, &cs, &sn, &gabs, &ctl, &gbase, &vmx};
  static const bool v2 = [] {  // IGM_ARNOLDI2=0: the shared-memory-resident k_arnoldi (A/B timing)
    const char* e = std::getenv("IGM_ARNOLDI2");
    return e == nullptr || e[0] != '0';
  }();
  if (v2 && S <= 4LL * kArn2Threads * kArn2Q) {  // w fits the registers: k_arnoldi2
    void* args2[] = {&n, &j, &S, &w, &basis, &accj, &absj, &nacc, &nabs, &f, &sh, &cstep,
                     &hess, &ld, &g, &cs, &sn, &gabs, &ctl, &gbase, &vmx, &snapj};
    static PerDevice attr2;
    if (attr2.first(dev)) {
      cudaFuncSetAttribute(k_arnoldi2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kArnSmemMax));
      cudaFuncSetAttribute(k_arnoldi2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kArnSmemMax));
    }
    const void* fn2 =
        checked ? reinterpret_cast<const void*>(k_arnoldi2<true>) : reinterpret_cast<const void*>(k_arnoldi2<false>);
    cudaLaunchCooperativeKernel(fn2, dim3(G), dim3(kArn2Threads), args2, smem, st);
    LAUNCH_CHECK();
    return;
  }
  const void* fn = checked ? reinterpret_cast<const void*>(k_arnoldi<true>) : reinterpret_cast<const void*>(k_arnoldi<false>);
  cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kArnThreads), args, smem, st);
  LAUNCH_CHECK();
}

void launch_recon_vals(cudaStream_t st, const DevSplit& m, int s, double* out) {
  ProfScope prof_(st, KC_OTHER);
  k_recon_vals<<<grid_for(m.nnz, 256), 256, 0, st>>>(m.nnz, s, m.vals, m.alphas, out);
  LAUNCH_CHECK();
}
void launch_fdot_axpy(cudaStream_t st, long long n, double* w, const double* v, double* part, double* h) {
  ProfScope prof_(st, KC_MGS);
  k_fdot_partial<<<kFdotBlocks, 256, 0, st>>>(n, w, v, part);
  k_fdot_final<<<1, 256, 0, st>>>(kFdotBlocks, part, h);
  k_faxpy<<<grid_for(n, 256), 256, 0, st>>>(n, w, v, h);
  LAUNCH_CHECK();
  LAUNCH_CHECK();
  LAUNCH_CHECK();
}
void launch_fscale(cudaStream_t st, long long n, const double* w, double* out, const double* d) {
  ProfScope prof_(st, KC_VEC_DIV);
  k_fscale<<<grid_for(n, 256), 256, 0, st>>>(n, w, out, d);
  LAUNCH_CHECK();
}
void launch_fxupdate(cudaStream_t st, long long n, int dim, const double* basis, const double* wts, double gamma,
                     double* x, int mode) {
  ProfScope prof_(st, KC_XUPDATE);
  k_fxupdate<<<grid_for(n, 256), 256, 0, st>>>(n, dim, basis, wts, gamma, x, mode);
  LAUNCH_CHECK();
}
int fdot_blocks() { return kFdotBlocks; }

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

template <typename T, bool B, int D, bool CP>
static void tri_launch_one(cudaStream_t st, const DevTri& t, const T* y, T* out, const Ctl* ctl,
                           const double* prescale) {
  constexpr size_t kBudget = 227 * 1024 - 256;  // static smem (tile id) excluded
  static const int env_L = [] {
    const char* e = std::getenv("IGM_TRI_L");
    return e ? std::atoi(e) : 0;
  }();
  const int L0 = env_L > 0 ? env_L : 8;
  int seg_cap = t.max_tile_segs + 2, L = L0;
  TriSmem lay = tri_smem_layout<D, CP>(t.tile_cap, seg_cap, L, t.max_seg_ext);
  while (L > 1 && lay.total > kBudget) lay = tri_smem_layout<D, CP>(t.tile_cap, seg_cap, --L, t.max_seg_ext);
  if (lay.total > kBudget) {  // segment tables stay in global memory
    seg_cap = 0;
    L = L0;
    lay = tri_smem_layout<D, CP>(t.tile_cap, seg_cap, L, t.max_seg_ext);
    while (L > 1 && lay.total > kBudget) lay = tri_smem_layout<D, CP>(t.tile_cap, seg_cap, --L, t.max_seg_ext);
  }
  const size_t sm = lay.total;
  static size_t done[64] = {0};  // per device
  const int dev = cur_device() & 63;
  if (sm > done[dev]) {
    cudaFuncSetAttribute(k_tri<T, B, D, CP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    done[dev] = sm;
  }
  TriArgs args = tri_args(t);
  {  // per-launch tag: splitmix64 of a counter (never 0, the words' initial tag)
    u64 z = (++const_cast<DevTri&>(t).epoch) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    args.epoch = (z ^ (z >> 31)) | 1ull;
  }
  // right-hand side into schedule order (and the FP path's 1/gamma prescale)
  k_tri_gather<T><<<grid_full(t.n, 256), 256, 0, st>>>(t.n, t.p_row, y, static_cast<T*>(t.yperm), ctl, prescale,
                                                       std::is_same<T, double>::value ? nullptr : t.stats);
  static const int env_pf = [] {
    const char* e = std::getenv("IGM_TRI_PF");
    return e ? std::atoi(e) : 12;
  }();
  k_tri<T, B, D, CP><<<t.ntiles, kTriThreads, sm, st>>>(args, static_cast<const T*>(t.yperm), out, ctl, seg_cap,
                                                        L, env_pf);
}

template <typename T, bool B>
static void tri_dispatch(cudaStream_t st, const DevTri& t, const T* y, T* out, const Ctl* ctl,
                         const double* prescale) {
  if (t.compact) {
    if (t.stride == 4) tri_launch_one<T, B, 4, true>(st, t, y, out, ctl, prescale);
    else if (t.stride == 8) tri_launch_one<T, B, 8, true>(st, t, y, out, ctl, prescale);
    else tri_launch_one<T, B, 16, true>(st, t, y, out, ctl, prescale);
  } else {
    if (t.stride == 4) tri_launch_one<T, B, 4, false>(st, t, y, out, ctl, prescale);
    else if (t.stride == 8) tri_launch_one<T, B, 8, false>(st, t, y, out, ctl, prescale);
    else tri_launch_one<T, B, 16, false>(st, t, y, out, ctl, prescale);
  }
}

void tri_trace_setup(int tile, unsigned long long* buf) {
  cudaMemcpyToSymbol(g_tri_ts, &buf, sizeof(buf));
  cudaMemcpyToSymbol(g_tri_ts_tile, &tile, sizeof(int));
}

// Per-launch tag of the pencil wavefront: unique in the process and seeded
// per process, because its in-CTA shared-memory words may meet words left on
// the SM by an earlier kernel (of this or another factor, or process).
static u64 pen_epoch() {
  static std::atomic<u64> ctr{[] {
    std::random_device rd;
    return (static_cast<u64>(rd()) << 32) ^ rd() ^
           static_cast<u64>(std::chrono::steady_clock::now().time_since_epoch().count());
  }()};
  u64 z = ctr.fetch_add(1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (z ^ (z >> 31)) | 1ull;
}

// warp-specialised pencil wavefront (tri_pencil2.cuh), bricks coupled in
// thread-block clusters of t.pen_cy along y.  Any ticket order the stream
// builder produces is valid for every cluster size (a brick waits only on
// bricks of earlier tickets), so a cluster launch that cannot be scheduled
// (e.g. SMs taken by another context) falls back to single-brick CTAs.
template <bool CHECKED, bool FP, int CY, bool PIPE>
static bool pen2_launch_cy(cudaStream_t st, const DevTri& t, const PenArgs& a, const i64* y, i64* out,
                           const int* stop, const int* err, const double* prescale) {
  static PerDevice attr;  // the attributes are per device
  if (attr.first(cur_device())) {
    cudaFuncSetAttribute(k_tri_pencil2<CHECKED, FP, CY, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kP2Smem));
  }
  if constexpr (CY == 1) {
    k_tri_pencil2<CHECKED, FP, 1, PIPE><<<t.pen_nbricks, kP2Threads, kP2Smem, st>>>(a, y, out, stop, err, prescale);
    return true;
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(t.pen_nbricks));
    cfg.blockDim = dim3(kP2Threads);
    cfg.dynamicSmemBytes = kP2Smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CY;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_tri_pencil2<CHECKED, FP, CY, PIPE>, a, y, out, stop, err, prescale) == cudaSuccess)
      return true;
    cudaGetLastError();  // not launchable as clusters: fall back
    return false;
  }
}

template <bool CHECKED, bool FP, bool PIPE>
static void pen2_launch(cudaStream_t st, const DevTri& t, const PenArgs& a, const i64* y, i64* out, const int* stop,
                        const int* err, const double* prescale) {
  bool ok = false;
  if (t.pen_cy == 8) ok = pen2_launch_cy<CHECKED, FP, 8, PIPE>(st, t, a, y, out, stop, err, prescale);
  else if (t.pen_cy == 4) ok = pen2_launch_cy<CHECKED, FP, 4, PIPE>(st, t, a, y, out, stop, err, prescale);
  else if (t.pen_cy == 2) ok = pen2_launch_cy<CHECKED, FP, 2, PIPE>(st, t, a, y, out, stop, err, prescale);
  if (!ok) pen2_launch_cy<CHECKED, FP, 1, PIPE>(st, t, a, y, out, stop, err, prescale);
}

// pencil wavefront (tri_pencil.cuh / tri_pencil2.cuh) of a structured 7-point
// factor: integer (FP = false) or FP64 (apply_inverse_fp) substitution
template <bool FP>
static void pen_launch(cudaStream_t st, const DevTri& t, bool backward, const void* y, void* out, const Ctl* ctl,
                       bool checked, const double* prescale, const PenZ* zp = nullptr) {
  constexpr int D = 4, R = 16;
  const size_t sm = pencil_smem_bytes(R, D);
  static PerDevice attr;  // the attribute is per device
  if (attr.first(cur_device())) {
    cudaFuncSetAttribute(k_tri_pencil<D, true, FP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    cudaFuncSetAttribute(k_tri_pencil<D, false, FP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  }
  PenArgs a;
  a.gx = t.pen_gx;
  a.gy = t.pen_gy;
  a.gz = t.pen_gz;
  a.nbx = t.pen_nbx;
  a.nby = t.pen_nby;
  a.S = t.pen_S;
  a.R = R;
  a.pad = t.pen_pad;
  a.n = t.n;
  a.mirror = backward ? 1 : 0;
  a.rec = FP ? t.pen_blk_fp : t.pen_blk;
  a.brick_of_ticket = t.pen_bot;
  a.xz = t.xz;
  a.epoch = pen_epoch();
  a.ticket = t.ticket;
  a.stats = reinterpret_cast<unsigned long long*>(t.stats);
  if (zp) {
    a.zimp = zp->imp;
    a.zexp = zp->exp;
    a.kexp = zp->kexp;
    a.zepoch = zp->epoch;
  }
  const int* stop = ctl ? &ctl->stop : nullptr;
  const int* err = ctl && !zp ? &ctl->err : nullptr;  // pipelined: see k_tri_pencil2
  const i64* yi = static_cast<const i64*>(y);
  i64* oi = static_cast<i64*>(out);
  static const bool v2 = [] {  // IGM_PENCIL2=0 selects the single-warp-role kernel (A/B timing)
    const char* e = std::getenv("IGM_PENCIL2");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (v2 || zp) {
    if constexpr (!FP) {
      if (zp) {  // pipelined z-slab substitution: the PIPE instantiation
        if (checked) pen2_launch<true, false, true>(st, t, a, yi, oi, stop, err, prescale);
        else pen2_launch<false, false, true>(st, t, a, yi, oi, stop, err, prescale);
        return;
      }
    }
    if (checked && !FP) pen2_launch<true, FP, false>(st, t, a, yi, oi, stop, err, prescale);
    else pen2_launch<false, FP, false>(st, t, a, yi, oi, stop, err, prescale);
    return;
  }
  if (checked && !FP)
    k_tri_pencil<D, true, FP><<<t.pen_nbricks, kPenThreads, sm, st>>>(a, yi, oi, stop, err, prescale);
  else
    k_tri_pencil<D, false, FP><<<t.pen_nbricks, kPenThreads, sm, st>>>(a, yi, oi, stop, err, prescale);
}

int pencil27_max_resident(int device) {
  const size_t sm = pencil27_smem_bytes();
  cudaFuncSetAttribute(k_tri27<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  cudaFuncSetAttribute(k_tri27<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  cudaFuncSetAttribute(k_tri27<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  cudaFuncSetAttribute(k_tri27<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  cudaFuncSetAttribute(k_tri27<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  int a = 0, b = 0, c = 0, d = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_tri27<true>, kP27Threads, sm) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_tri27<false>, kP27Threads, sm) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_tri27<false, true>, kP27Threads, sm) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d, k_tri27<true, false, true>, kP27Threads, sm) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(std::min(a, b), std::min(c, d)) * num_sms(device);
}

// k_tri27's bricks wait on each other in both directions, so they must all
// be resident: a cooperative launch guarantees that (or fails, e.g. when
// another context's kernels occupy the SMs).  Returns false when the launch
// was refused; the caller then runs the generic wavefront.
static bool pen27_launch(cudaStream_t st, const DevTri& t, bool backward, const i64* y, i64* out, const Ctl* ctl,
                         bool checked, bool fp = false, const double* prescale = nullptr, const PenZ* zp = nullptr) {
  P27Args a;
  a.gx = t.p27_gx;
  a.gy = t.p27_gy;
  a.gz = t.p27_gz;
  a.nbx = t.p27_nbx;
  a.n = t.n;
  a.mirror = backward ? 1 : 0;
  a.rec = static_cast<const unsigned char*>(fp ? t.p27_rec_fp : t.p27_rec);
  a.xz = t.xz;
  a.epoch = pen_epoch();
  a.stats = reinterpret_cast<unsigned long long*>(t.stats);
  const int* stop = ctl ? &ctl->stop : nullptr;
  const int* err = ctl ? &ctl->err : nullptr;
  const size_t sm = pencil27_smem_bytes();
  static PerDevice attr;  // the attribute is per device
  if (attr.first(cur_device())) pencil27_max_resident(cur_device());
  const double* ps = fp ? prescale : nullptr;
  void* args[] = {&a, &y, &out, &stop, &err, &ps};
  const void* fn = fp ? reinterpret_cast<const void*>(k_tri27<false, true>)
                      : (checked ? reinterpret_cast<const void*>(k_tri27<true>)
                                 : reinterpret_cast<const void*>(k_tri27<false>));
  if (zp != nullptr && !fp) {  // z-slab hand-off: a separate instantiation
    a.zimp = zp->imp;
    a.zexp = zp->exp;
    a.kexp = zp->kexp;
    a.zepoch = zp->epoch;
    fn = checked ? reinterpret_cast<const void*>(k_tri27<true, false, true>)
                 : reinterpret_cast<const void*>(k_tri27<false, false, true>);
  }
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(t.p27_nbricks), dim3(kP27Threads), args, sm, st);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();
    return false;
  }
  return true;  // any other error is reported by LAUNCH_CHECK
}

// the rank-local substitution of a z-slab with its boundary plane streamed from
// / to the neighbour ranks (pencil wavefronts only); false when the factor is
// neither a 7-point nor a 27-point pencil factor (or the 27-point kernel's
// bricks cannot all be resident)
bool launch_tri_int_piped(cudaStream_t st, const DevTri& t, bool backward, const i64* y, i64* out, u64* cnt,
                          const Ctl* ctl, bool checked, const PenZ& z) {
  if (t.n == 0 || (!t.pen && !t.pen27)) return false;
  if (checked) cudaMemsetAsync(t.stats, 0, 2 * sizeof(u64), st);
  {
    ProfScope prof_(st, KC_TRI_INT);
    if (t.pen) pen_launch<false>(st, t, backward, y, out, ctl, checked, nullptr, &z);
    else if (!pen27_launch(st, t, backward, y, out, ctl, checked, false, nullptr, &z)) return false;
  }
  LAUNCH_CHECK();
  if (checked) {
    ProfScope prof_(st, KC_OTHER);
    k_tri_count<<<grid_for(t.n, 256), 256, 0, st>>>(t.n, t.c_rp, t.c_ci, t.c_val, t.c_diag, y, out, cnt, ctl,
                                                      t.stats, static_cast<double>(t.maxabs_l), t.maxd);
    LAUNCH_CHECK();
  }
  return true;
}

void launch_tri_count_pair(cudaStream_t st, const DevTri& lo, const DevTri& up, const i64* y, const i64* mid,
                           const i64* z, u64* cnt, const Ctl* ctl) {
  if (lo.n == 0) return;
  auto mk = [](const DevTri& t) {
    return TriCnt{t.n, t.c_rp, t.c_ci, t.c_val, t.c_diag, t.stats, static_cast<double>(t.maxabs_l), t.maxd};
  };
  ProfScope prof_(st, KC_OTHER);
  const int g = std::max(1, std::min((lo.n + 255) / 256, 2 * num_sms(cur_device())));
  k_tri_count_pair<<<g, 256, 0, st>>>(mk(lo), mk(up), y, mid, z, cnt, ctl);
  LAUNCH_CHECK();
}

// defer_count: checked mode without the stats memset and the recount launch --
// the caller runs launch_tri_count_pair after the forward / backward pair
void launch_tri_int(cudaStream_t st, const DevTri& t, bool backward, const i64* y, i64* out,
                    u64* cnt, const Ctl* ctl, bool checked, bool defer_count) {
  if (t.n == 0) return;
  if (!t.pen) cudaMemsetAsync(t.ticket, 0, sizeof(int), st);  // the pencil kernel's last CTA resets it
  if (checked && defer_count) {
    {
      ProfScope prof_(st, KC_TRI_INT);
      if (t.pen) pen_launch<false>(st, t, backward, y, out, ctl, checked, nullptr);
      else if (t.pen27 && pen27_launch(st, t, backward, y, out, ctl, checked)) {
      } else if (backward) tri_dispatch<i64, true>(st, t, y, out, ctl, nullptr);
      else tri_dispatch<i64, false>(st, t, y, out, ctl, nullptr);
    }
    LAUNCH_CHECK();
    return;
  }
  if (checked) cudaMemsetAsync(t.stats, 0, 2 * sizeof(u64), st);
  {
    ProfScope prof_(st, KC_TRI_INT);
    if (t.pen) pen_launch<false>(st, t, backward, y, out, ctl, checked, nullptr);
    else if (t.pen27 && pen27_launch(st, t, backward, y, out, ctl, checked)) {
    } else if (backward) tri_dispatch<i64, true>(st, t, y, out, ctl, nullptr);
    else tri_dispatch<i64, false>(st, t, y, out, ctl, nullptr);
  }
  LAUNCH_CHECK();
  if (checked) {
    ProfScope prof_(st, KC_OTHER);
    k_tri_count<<<grid_for(t.n, 256), 256, 0, st>>>(t.n, t.c_rp, t.c_ci, t.c_val, t.c_diag, y, out, cnt, ctl,
                                                      t.stats, static_cast<double>(t.maxabs_l), t.maxd);
    LAUNCH_CHECK();
  }
}

void launch_tri_fp(cudaStream_t st, const DevTri& t, bool backward, const double* y, double* out,
                   const Ctl* ctl, const double* prescale) {
  if (t.n == 0) return;
  if (!(t.pen && t.pen_blk_fp)) cudaMemsetAsync(t.ticket, 0, sizeof(int), st);
  ProfScope prof_(st, KC_TRI_FP);
  if (t.pen && t.pen_blk_fp) pen_launch<true>(st, t, backward, y, out, ctl, false, prescale);
  else if (t.pen27 && t.p27_rec_fp &&
           pen27_launch(st, t, backward, reinterpret_cast<const i64*>(y), reinterpret_cast<i64*>(out), ctl, false,
                        true, prescale)) {
  } else if (backward) tri_dispatch<double, true>(st, t, y, out, ctl, prescale);
  else tri_dispatch<double, false>(st, t, y, out, ctl, prescale);
  LAUNCH_CHECK();
}

}  // namespace igm
