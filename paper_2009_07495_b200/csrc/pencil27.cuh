// pencil27.cuh -- ILU(0) integer substitution for 27-point structured
// factors as a pencil wavefront (sm_100a), host stream builder + kernel.
//
// A factor qualifies when every off-diagonal entry of row (i,j,k) (solve
// order; mirrored for U) is one of the 13 "lower" neighbours of the 27-point
// stencil: the 9 of plane k-1 and (i-1,j-1,k), (i,j-1,k), (i+1,j-1,k),
// (i-1,j,k).  The level function i + 2j + 4k orders them (every dependency is
// 1..7 levels earlier), so a thread owning the z-pencil (i,j) of a 16 x 16
// brick handles row k at brick step (i mod 16) + 2 (j mod 16) + 4k: a lane is
// active every fourth step and each warp step has 8 active lanes.
//
// Unlike the 7-point case the bricks depend on each other in both directions
// (row (i,j,k) reads (i+1,j+1,k-1) of the +x / +y brick), so every brick of a
// launch must be resident at once: the launcher uses a cooperative launch
// (co-residency guaranteed or the launch fails) and falls back to the generic
// wavefront when it fails.  Inside a brick every row
// value goes through a shared-memory ring of R planes; brick-boundary rows are
// also exported as tagged words (value, tag ^ value) in global memory, which
// the neighbour bricks read.  A word of another launch / plane or a torn word
// fails its tag and is re-polled; every dependency is of an earlier step, so
// no lane ever waits on a value its own warp has still to compute.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

#include "fx_core.cuh"

namespace igm {

constexpr int kP27B = 16;                 // brick: 16 x 16 pencils
constexpr int kP27Threads = kP27B * kP27B;  // one per pencil (8 warps of 16 x 2)
constexpr int kP27R = 8;                  // ring planes
constexpr int kP27Rec = 64;               // stream bytes per row: 13 x int32 factor, int32 info, u64 reciprocal
constexpr int kP27Lag = 24;               // max steps a warp may lead its neighbour warps (ring of kP27R planes)

// the 13 dependency offsets (di, dj, dk)
__host__ __device__ constexpr int p27_di(int q) { return q < 9 ? q % 3 - 1 : (q < 12 ? q - 10 : -1); }
__host__ __device__ constexpr int p27_dj(int q) { return q < 9 ? q / 3 - 1 : (q < 12 ? -1 : 0); }
__host__ __device__ constexpr int p27_dk(int q) { return q < 9 ? -1 : 0; }

struct Pencil27Stream {
  bool ok = false;
  int gx = 0, gy = 0, gz = 0, nbx = 0, nby = 0, nbricks = 0;
  std::vector<unsigned char> rec;  // [brick][thread][k] x 64 B
};

// info: sh1 | sh2 << 1 | den_neg << 8 | presence of dependency q << (9 + q)
inline Pencil27Stream build_pencil27_stream(int n, const int* rp, const int* ci, const std::int64_t* vals,
                                            const int* dpos, bool upper, int gx, int gy, int gz, bool fp = false) {
  Pencil27Stream P;
  if (gx < 2 || gy < 2 || gz < 1 || static_cast<long long>(gx) * gy * gz != n) return P;
  const long long plane = static_cast<long long>(gx) * gy;
  P.gx = gx;
  P.gy = gy;
  P.gz = gz;
  P.nbx = (gx + kP27B - 1) / kP27B;
  P.nby = (gy + kP27B - 1) / kP27B;
  P.nbricks = P.nbx * P.nby;
  P.rec.assign(static_cast<size_t>(P.nbricks) * kP27Threads * gz * kP27Rec, 0);
  for (int r = 0; r < n; ++r) {
    const long long rs = upper ? n - 1 - r : r;
    const long long i = rs % gx, j = (rs / gx) % gy, k = rs / plane;
    std::int32_t f[13] = {0};
    int mask = 0;
    for (int q2 = rp[r]; q2 < rp[r + 1]; ++q2) {
      if (q2 == dpos[r]) continue;
      const int c = ci[q2];
      if (c < 0 || c >= n) return Pencil27Stream{};
      if (upper ? c < r : c > r) continue;  // outside the triangle: never read (ilu.cpp:126-135)
      if (c == r) return Pencil27Stream{};
      const long long cs = upper ? n - 1 - c : c;
      const long long di = cs % gx - i, dj = (cs / gx) % gy - j, dk = cs / plane - k;
      int q = -1;
      if (dk == -1 && di >= -1 && di <= 1 && dj >= -1 && dj <= 1) q = static_cast<int>((dj + 1) * 3 + di + 1);
      else if (dk == 0 && dj == -1 && di >= -1 && di <= 1) q = static_cast<int>(10 + di);
      else if (dk == 0 && dj == 0 && di == -1) q = 12;
      if (q < 0 || (mask >> q) & 1) return Pencil27Stream{};
      const std::int64_t v = vals[q2];
      if (v < INT32_MIN || v > INT32_MAX) return Pencil27Stream{};
      f[q] = static_cast<std::int32_t>(v);
      mask |= 1 << q;
    }
    if (dpos[r] < rp[r] || dpos[r] >= rp[r + 1] || ci[dpos[r]] != r || vals[dpos[r]] == 0) return Pencil27Stream{};
    const SDivMagic g = make_sdiv(vals[dpos[r]]);
    const std::int32_t info = (g.u.sh1 & 1) | ((g.u.sh2 & 127) << 1) | (g.den_neg << 8) | (mask << 9);
    const long long bx = i / kP27B, by = j / kP27B, xl = i % kP27B, jl = j % kP27B;
    const long long t = (jl >> 1) * 32 + (jl & 1) * 16 + xl;  // thread of the pencil
    unsigned char* e = &P.rec[((static_cast<size_t>(by * P.nbx + bx) * kP27Threads + t) * gz + k) * kP27Rec];
    std::memcpy(e, f, 52);
    std::memcpy(e + 52, &info, 4);
    if (fp) {
      const double dd = static_cast<double>(vals[dpos[r]]);
      std::memcpy(e + 56, &dd, 8);
    } else {
      std::memcpy(e + 56, &g.u.m, 8);
    }
  }
  P.ok = true;
  return P;
}

struct P27Args {
  int gx, gy, gz, nbx;
  long long n;
  int mirror;
  const unsigned char* rec;
  ulonglong2* xz;           // exported boundary values by solve-order row
  unsigned long long epoch;
  unsigned long long* stats;  // [max|y|, max|z|] bounds (checked mode)
  // z-slab pipelining (PIPE instantiation; igm_dc_tri_piped, dist.ZPipe):
  // plane 0's values arrive as (value, zepoch + natural idx) words in zimp,
  // plane kexp's leave the same way into the neighbour rank's buffer zexp
  const ulonglong2* zimp = nullptr;
  ulonglong2* zexp = nullptr;
  int kexp = -1;
  unsigned long long zepoch = 0;
};

__device__ __forceinline__ void p27_ldg16(const ulonglong2* p, u64& v, u64& t) {
  asm volatile("{ .reg .b128 x; ld.global.relaxed.gpu.b128 x, [%2]; mov.b128 {%0, %1}, x; }"
               : "=l"(v), "=l"(t)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void p27_lds16(unsigned a, u64& v, u64& t) {
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v), "=l"(t) : "r"(a) : "memory");
}

// FP = true: the FP64 substitution on the integer factors (apply_inverse_fp,
// ilu.cpp:157-180): acc = y (or y / gamma), acc -= L_rd * z_d over the row's
// entries in CSR order -- dependencies 0..12 for the lower factor, 12..0 for
// the mirrored upper one -- every operation rounded on its own, absent
// entries skipped, then acc / diag (the stream holds the diagonal as a double)
template <bool CHECKED, bool FP = false, bool PIPE = false>
__global__ void __launch_bounds__(kP27Threads, 2) k_tri27(P27Args a, const i64* __restrict__ y, i64* __restrict__ out,
                                                          const int* stop, const int* err,
                                                          const double* prescale = nullptr) {
  extern __shared__ __align__(16) unsigned char p27_smem[];
  __shared__ volatile int s_prog[kP27Threads / 32];  // steps completed per warp (ring back-pressure)
  if (stop != nullptr && (*stop | *err) != 0) return;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, xl = lane & 15, jl = 2 * w + (lane >> 4);
  if (lane == 0) s_prog[w] = 0;
  const int bx = blockIdx.x % a.nbx, by = blockIdx.x / a.nbx;
  const int i = bx * kP27B + xl, j = by * kP27B + jl;
  const bool ing = i < a.gx && j < a.gy;
  const int gz = a.gz;
  const long long plane = static_cast<long long>(a.gx) * a.gy;
  // ring [pencil (jl,xl)][plane slot] x 16 B, then the lane-private record
  // slots [2][thread] x 80 B (64 B record + 8 B rhs + pad)
  const unsigned ring0 = static_cast<unsigned>(__cvta_generic_to_shared(p27_smem));
  const unsigned pre0 = ring0 + kP27Threads * kP27R * 16 + tid * 80u;
  {
    uint4* rz = reinterpret_cast<uint4*>(p27_smem);
    for (int q = tid; q < kP27Threads * kP27R; q += kP27Threads) rz[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const unsigned char* rp = a.rec + (static_cast<size_t>(blockIdx.x) * kP27Threads + tid) * gz * kP27Rec;
  const long long rb = static_cast<long long>(j) * a.gx + i;  // solve-order row at k = 0
  auto issue = [&](int k) {  // this lane's record and rhs of row k into slot k & 1
    const unsigned d = pre0 + static_cast<unsigned>(k & 1) * (kP27Threads * 80u);
    const unsigned char* src = rp + static_cast<size_t>(k) * kP27Rec;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * c), "l"(src + 16 * c) : "memory");
    const long long r = rb + k * plane;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 64), "l"(y + (a.mirror ? a.n - 1 - r : r))
                 : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (ing) issue(0);
  // per dependency: in this brick (shared ring) or a neighbour's (global word)
  int inb = 0;
#pragma unroll
  for (int q = 0; q < 13; ++q) {
    const int nx = xl + p27_di(q), ny = jl + p27_dj(q);
    if (nx >= 0 && nx < kP27B && ny >= 0 && ny < kP27B) inb |= 1 << q;
  }
  const bool bnd = xl == 0 || xl == kP27B - 1 || jl == 0 || jl == kP27B - 1;  // exported (read by neighbours)
  const int off = xl + 2 * jl;  // row k at brick step off + 4k
  const unsigned my_ring = ring0 + static_cast<unsigned>((jl * kP27B + xl) * kP27R) * 16u;
  constexpr u64 C = 0x9E3779B97F4A7C15ull;
  const u64 epoch = a.epoch;
  u64 ymx = 0, zmx = 0;
  // step-synchronous: at step s the lanes with (s - off) % 4 == 0 handle row
  // (s - off) / 4 (8 lanes per warp); the warp reconverges every step
  const int Smax = kP27B - 1 + 2 * (kP27B - 1) + 4 * gz;
  int seen = 0;  // min progress of warps w-1 / w+1 last observed
#pragma unroll 1
  for (int s = 0; s < Smax; ++s) {
    __syncwarp();
    if (lane == 0) s_prog[w] = s;
    // Step s overwrites ring slot k & 7, which held plane k - 8; its last
    // readers (warps w-1, w, w+1: dependency offsets |dj| <= 1) read it at
    // their step s - 25 at the latest (plane k - 7 with a dk = -1 entry,
    // lane offset <= off + 3).  A factor with the full 27-point pattern keeps
    // the warps within a step of each other; a subset pattern (no coupling
    // back to warp w+1) could otherwise let warp w lap its consumers.
    if (s - kP27Lag > seen) {
      do {
        const int a0 = w > 0 ? s_prog[w - 1] : 0x3fffffff;
        const int a1 = w + 1 < kP27Threads / 32 ? s_prog[w + 1] : 0x3fffffff;
        seen = a0 < a1 ? a0 : a1;
      } while (s - kP27Lag > seen);
    }
    const int dd = s - off;
    if (!ing || dd < 0 || (dd & 3) != 0 || (dd >> 2) >= gz) continue;
    const int k = dd >> 2;
    {
      asm volatile("cp.async.wait_all;" ::: "memory");
      const unsigned d = pre0 + static_cast<unsigned>(k & 1) * (kP27Threads * 80u);
      int f[13];
      int info;
      u64 mg, yv;
      {
        int4 q0, q1, q2, q3;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w) : "r"(d) : "memory");
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w) : "r"(d + 16) : "memory");
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(q2.x), "=r"(q2.y), "=r"(q2.z), "=r"(q2.w) : "r"(d + 32) : "memory");
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(q3.x), "=r"(q3.y), "=r"(q3.z), "=r"(q3.w) : "r"(d + 48) : "memory");
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(mg) : "r"(d + 56) : "memory");
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(yv) : "r"(d + 64) : "memory");
        f[0] = q0.x; f[1] = q0.y; f[2] = q0.z; f[3] = q0.w;
        f[4] = q1.x; f[5] = q1.y; f[6] = q1.z; f[7] = q1.w;
        f[8] = q2.x; f[9] = q2.y; f[10] = q2.z; f[11] = q2.w;
        f[12] = q3.x; info = q3.y;
      }
      if (k + 1 < gz) issue(k + 1);
      if (PIPE && k == 0 && a.zimp != nullptr) {  // a unit halo row: its value is the neighbour rank's
        const long long idx = a.mirror ? static_cast<long long>(a.gy - 1 - j) * a.gx + (a.gx - 1 - i)
                                       : static_cast<long long>(j) * a.gx + i;
        u64 zt;
        do {
          asm volatile("{ .reg .b128 x; ld.relaxed.sys.global.b128 x, [%2]; mov.b128 {%0, %1}, x; }"
                       : "=l"(yv), "=l"(zt)
                       : "l"(a.zimp + idx)
                       : "memory");
        } while (zt != a.zepoch + static_cast<u64>(idx));
      }
      const u64 w0 = epoch ^ (static_cast<u64>(k + 1) * C), w1 = epoch ^ (static_cast<u64>(k) * C);  // tags of planes k, k-1
      const long long r = rb + k * plane;
      const int mask = info >> 9;
      // every dependency's word loaded back to back, checked afterwards
      u64 v[13], t[13];
#pragma unroll
      for (int q = 0; q < 13; ++q) {
        v[q] = 0;
        t[q] = (p27_dk(q) ? w1 : w0);  // an absent entry reads as fresh 0
        if (!((mask >> q) & 1)) continue;
        if ((inb >> q) & 1)
          p27_lds16(ring0 + static_cast<unsigned>(((jl + p27_dj(q)) * kP27B + xl + p27_di(q)) * kP27R +
                                                  ((k + p27_dk(q)) & (kP27R - 1))) * 16u, v[q], t[q]);
        else
          p27_ldg16(a.xz + (r + p27_di(q) + static_cast<long long>(p27_dj(q)) * a.gx + p27_dk(q) * plane), v[q], t[q]);
      }
#pragma unroll
      for (int q = 0; q < 13; ++q) {
        const u64 want = p27_dk(q) ? w1 : w0;
        if (t[q] != (want ^ v[q])) {  // not there yet: re-poll (rare off the critical path)
          if ((inb >> q) & 1) {
            const unsigned ad = ring0 + static_cast<unsigned>(((jl + p27_dj(q)) * kP27B + xl + p27_di(q)) * kP27R +
                                                             ((k + p27_dk(q)) & (kP27R - 1))) * 16u;
            do {
              p27_lds16(ad, v[q], t[q]);
            } while (t[q] != (want ^ v[q]));
          } else {
            const ulonglong2* gp = a.xz + (r + p27_di(q) + static_cast<long long>(p27_dj(q)) * a.gx + p27_dk(q) * plane);
            do {
              p27_ldg16(gp, v[q], t[q]);
            } while (t[q] != (want ^ v[q]));
          }
        }
      }
      i64 z;
      if constexpr (FP) {
        double acc = __longlong_as_double(static_cast<long long>(yv));
        if (prescale != nullptr) acc = __ddiv_rn(acc, *prescale);
#pragma unroll
        for (int u = 0; u < 13; ++u) {
          const int q = a.mirror ? 12 - u : u;
          if ((mask >> q) & 1)
            acc = __dsub_rn(acc, __dmul_rn(static_cast<double>(f[q]), __longlong_as_double(static_cast<long long>(v[q]))));
        }
        z = __double_as_longlong(__ddiv_rn(acc, __longlong_as_double(static_cast<long long>(mg))));
      } else {
        u64 sx = 0;
#pragma unroll
        for (int q = 0; q < 13; ++q) sx += static_cast<u64>(static_cast<i64>(f[q])) * v[q];
        SDivMagic gm;
        gm.u.m = mg;
        gm.u.sh1 = info & 1;
        gm.u.sh2 = (info >> 1) & 127;
        gm.den_neg = (info >> 8) & 1;
        gm.den_is_m1 = 0;
        z = sdiv(static_cast<i64>(yv - sx), gm);
      }
      const u64 tg = w0 ^ static_cast<u64>(z);
      asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(my_ring + static_cast<unsigned>(k & (kP27R - 1)) * 16u),
                   "l"(z), "l"(tg)
                   : "memory");
      if (bnd)
        asm volatile("{ .reg .b128 x; mov.b128 x, {%0, %1}; st.global.relaxed.gpu.b128 [%2], x; }" ::"l"(z), "l"(tg),
                     "l"(a.xz + r)
                     : "memory");
      out[a.mirror ? a.n - 1 - r : r] = z;
      if (PIPE && k == a.kexp && a.zexp != nullptr) {  // the next rank's plane-0 value
        const long long idx = a.mirror ? static_cast<long long>(a.gy - 1 - j) * a.gx + (a.gx - 1 - i)
                                       : static_cast<long long>(j) * a.gx + i;
        asm volatile("{ .reg .b128 x; mov.b128 x, {%1, %2}; st.relaxed.sys.global.b128 [%0], x; }" ::"l"(a.zexp + idx),
                     "l"(static_cast<u64>(z)), "l"(a.zepoch + static_cast<u64>(idx))
                     : "memory");
      }
      if (CHECKED && !FP) {
        ymx |= yv ^ static_cast<u64>(static_cast<i64>(yv) >> 63);
        zmx |= static_cast<u64>(z ^ (z >> 63));
      }
    }
  }
  __syncwarp();
  if (lane == 0) s_prog[w] = 0x3fffffff;  // done: never a consumer again
  if (CHECKED && !FP && a.stats != nullptr) {
    if (ymx) atomicMax(a.stats, static_cast<unsigned long long>(ymx + 1));
    if (zmx) atomicMax(a.stats + 1, static_cast<unsigned long long>(zmx + 1));
  }
}

inline size_t pencil27_smem_bytes() { return static_cast<size_t>(kP27Threads) * kP27R * 16 + 2ull * kP27Threads * 80; }

}  // namespace igm
