// tri_pencil2.cuh -- warp-specialised pencil wavefront for structured 7-point
// ILU(0) factors (sm_100a).  Same substitution, stream and brick geometry as
// tri_pencil.cuh (k_tri_pencil); what changes is who waits for what.
//
// Integer path of apply_inverse (ilu.cpp:122-155) and FP64 path of
// apply_inverse_fp (ilu.cpp:157-180), bit-identical to k_tri_pencil.
//
// One CTA = one 16 x (2 kPenWarps) brick of z-pencils:
//   * kPenWarps COMPUTE warps, lane (xl, jj) of warp w walks pencil
//     (16 bx + xl, 2 kPenWarps by + 2 w + jj) one row per step (row k at step
//     k + xl + jj).  Every dependency of a step is in shared memory or a
//     register: -x from lane xl-1 (__shfl_up), -y from lane (xl, 0)
//     (__shfl_xor 16) or from a tagged ring slot, -z the lane's own previous
//     row.  A compute warp never touches global memory except to store.
//   * one LOADER warp: per stage of G steps and per compute warp, one
//     cp.async.bulk of the G record blocks (768 B each, the same stream as
//     k_tri_pencil) and a per-lane cp.async gather of the G right-hand-side
//     words, both completing on the stage's mbarrier; NS stages in flight.
//   * one IMPORTER warp: polls the tagged (value, epoch ^ kc(k) ^ value)
//     words the -x and -y neighbour bricks export to global memory, up to PI
//     rows ahead per face lane, and copies each valid word into the shared
//     ring the consuming compute lane reads.  The global round trip of a
//     brick-to-brick hand-off is thus paid by a warp that is off the
//     critical path, instead of by a compute warp re-polling a stale
//     prefetched word (ncu on k_tri_pencil: the re-poll loop held ~40 % of
//     all warp stall samples).
// Deadlock freedom: bricks wait only on bricks of earlier tickets (resident);
// compute warp w waits only on warp w-1, the importer and the loader; the
// importer never blocks (a word whose ring slot is still in use stays in
// global memory until the next round); the loader waits for a stage slot to
// be released, and a warp can run at most R <= NS*G steps ahead of the next.
#pragma once

#include "tri_pencil.cuh"

namespace igm {

constexpr int kP2G = 8;    // steps per stage
constexpr int kP2NS = 4;   // stages per compute warp
constexpr int kP2R = 32;   // ring slots (rows); kP2R <= kP2NS * kP2G
constexpr int kP2PI = 8;   // importer: outstanding polls per face lane
#ifdef P2_WATCH
constexpr int kP2Threads = 32 * (kPenWarps + 3);  // + a watchdog warp (diagnostics build)
__device__ volatile unsigned long long* g_p2_watch;
#else
constexpr int kP2Threads = 32 * (kPenWarps + 2);
#endif
static_assert(kP2R <= kP2NS * kP2G, "ring lead must not exceed the staged window");
static_assert(2 * kPenWarps + 16 <= 32, "importer lanes");

// dynamic shared memory layout (bytes)
constexpr unsigned kP2RingBytes = kPenWarps * kP2R * 16 * 16;  // [warp][slot][xl] (v, tag): y-values
constexpr unsigned kP2XrBytes = kPenWarps * 2 * kP2R * 16;     // [warp][jj][slot] (v, tag): x-imports
constexpr unsigned kP2RecBytes = kPenWarps * kP2NS * kP2G * 768;
constexpr unsigned kP2RhsBytes = kPenWarps * kP2NS * kP2G * 256;
constexpr unsigned kP2OffXr = kP2RingBytes;
constexpr unsigned kP2OffRec = kP2OffXr + kP2XrBytes;
constexpr unsigned kP2OffRhs = kP2OffRec + kP2RecBytes;
constexpr unsigned kP2OffBar = kP2OffRhs + kP2RhsBytes;  // full[w][NS], empty[w][NS]
constexpr unsigned kP2OffProg = kP2OffBar + 2 * kPenWarps * kP2NS * 8;
constexpr unsigned kP2Smem = kP2OffProg + 128;

__device__ __forceinline__ void p2_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void p2_mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool p2_mbar_try(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2; selp.u32 %0, 1, 0, P1; }"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
#if defined(P2_DBG) && !defined(P2_GUARDS)
#define P2_GUARDS
#endif
#ifdef P2_GUARDS  // diagnostics build (scripts/pencil2_proto.cu): spin guards that report and break
__device__ unsigned long long g_p2_rep[64 * 4];
__device__ unsigned g_p2_nrep;
__device__ unsigned g_p2_idc[8];
__device__ __noinline__ void p2_report(int id, int x, int y) {
  atomicAdd(&g_p2_nrep, 1u);
  const unsigned q = atomicAdd(&g_p2_idc[id & 7], 1u) == 0 ? static_cast<unsigned>(id & 7) : 64u;
  if (q < 64) {
    g_p2_rep[q * 4] = blockIdx.x;
    g_p2_rep[q * 4 + 1] = threadIdx.x;
    g_p2_rep[q * 4 + 2] = static_cast<unsigned long long>(id);
    g_p2_rep[q * 4 + 3] = (static_cast<unsigned long long>(static_cast<unsigned>(x)) << 32) | static_cast<unsigned>(y);
  }
}
__device__ unsigned long long g_p2_blk[256 * 16];
#define P2_GUARD(id_, xa_, ya_)                                                                   \
  if (++spins > (1u << 22)) {                                                                \
    p2_report(id_, xa_, ya_);                                                                     \
    unsigned long long* sn = g_p2_blk + blockIdx.x * 16;                                     \
    sn[0] = t; sn[1] = bx; sn[2] = by;                                                       \
    for (int qq = 0; qq < 4; ++qq) sn[3 + qq] = prog[qq];                                    \
    for (int qq = 0; qq < 8; ++qq) sn[7 + qq] = reinterpret_cast<volatile int*>(p2_smem + kP2OffProg)[8 + qq]; \
    sn[15] = 1;                                                                              \
    break;                                                                                   \
  }
#else
#define P2_GUARD(id, x, y)
#endif
#ifdef P2_DBG  // per-step timestamps of brick P2_DBG
__device__ unsigned long long g_p2_ts[8 * 4096];
#define P2_TS(slot, val) \
  if (t == P2_DBG && (slot) < 8 * 4096) g_p2_ts[slot] = (val);
__device__ __forceinline__ long long p2_clk(u64 dep) {
  long long c;
  asm volatile("{ .reg .u64 d; mov.u64 d, %1; mov.u64 %0, %%clock64; }" : "=l"(c) : "l"(dep) : "memory");
  return c;
}
#define P2_PH(q, dep)                    \
  {                                      \
    const long long c_ = p2_clk(dep);    \
    ph[q] += c_ - pc;                    \
    pc = c_;                             \
  }
#else
#define P2_TS(slot, val) {}
#define P2_PH(q, dep)
#endif
#ifdef P2_STAGETS
__device__ long long g_p2_sts[8 * 1024];
__device__ unsigned long long g_p2_bt[64 * 64 * 16];
#endif
#ifndef P2_NS
#define P2_NS 0
#endif
#ifndef P2_KNOB  // timing experiments only: bits switch pieces of the compute step off
#define P2_KNOB 0
#endif
#if P2_NS > 0
#define P2_SLEEP() __nanosleep(P2_NS)
#else
#define P2_SLEEP()
#endif
// shared-memory hand-off word: {z, k + 1} (16 B; the tag k + 1 is never 0,
// the rings are cleared at kernel start and a slot holds rows k, k + R, ...)
__device__ __forceinline__ void p2_sts_word(unsigned a, u64 z, int k) {
  asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(static_cast<unsigned>(z)),
               "r"(static_cast<unsigned>(z >> 32)), "r"(k + 1), "r"(0));
}
__device__ __forceinline__ void p2_lds_word(unsigned a, u64& z, int& t) {
  unsigned lo, hi, pad;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(lo), "=r"(hi), "=r"(t), "=r"(pad) : "r"(a));
  z = (static_cast<u64>(hi) << 32) | lo;
}
__device__ __forceinline__ void p2_lds2(unsigned a, u64& v, u64& tg) {
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v), "=l"(tg) : "r"(a) : "memory");
}

template <bool CHECKED, bool FP>
__global__ void __launch_bounds__(kP2Threads, 1)
    k_tri_pencil2(PenArgs a, const i64* __restrict__ y, i64* __restrict__ out, const int* stop, const int* err,
                  const double* prescale) {
  extern __shared__ __align__(128) unsigned char p2_smem[];
  __shared__ int s_t;
  if (stop != nullptr && (*stop | *err) != 0) return;  // the cycle already ended (Ctl::stop / Ctl::err)
  constexpr int W = kPenWarps, G = kP2G, NS = kP2NS, R = kP2R;
  constexpr unsigned RM = R - 1;
  constexpr u64 C = 0x9E3779B97F4A7C15ull;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(p2_smem));
  const unsigned bar_full = sbase + kP2OffBar, bar_empty = bar_full + W * NS * 8;
  volatile int* prog = reinterpret_cast<volatile int*>(p2_smem + kP2OffProg);
  if (tid == 0) {
    s_t = atomicAdd(a.ticket, 1);
    for (int q = 0; q < W * NS; ++q) {
      p2_mbar_init(bar_full + q * 8, 33);  // 32 gathering lanes (noinc) + the bulk copy's expect_tx
      p2_mbar_init(bar_empty + q * 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) prog[tid] = 0;
  {  // clear the rings: shared memory keeps words of earlier kernels
    uint4* rz = reinterpret_cast<uint4*>(p2_smem);
    for (int q = tid; q < static_cast<int>((kP2RingBytes + kP2XrBytes) / 16); q += kP2Threads)
      rz[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const int t = s_t;
  const int code = __ldg(a.brick_of_ticket + t);
  const int bx = code & 0xffff, by = code >> 16;
  const int gz = a.gz, S = a.S;
  const long long plane = static_cast<long long>(a.gx) * a.gy;
  const long long gxl = a.gx;
  const u64 epoch = a.epoch;
  const long long ystride = a.mirror ? -plane : plane;

  if (w == W) {
    // ------------------------------------------------------------ loader
    const int xl = lane & 15, jj = lane >> 4, kb = xl + jj;
    const int i = bx * kPenX + xl;
    const unsigned char* src0 = reinterpret_cast<const unsigned char*>(a.rec) +
                                static_cast<size_t>(t) * W * static_cast<size_t>(S + a.pad) * 768;
    // per compute warp: this lane's rhs pointer at step 0 and activity window
    const i64* yp[W];
    int sa[W];
#pragma unroll
    for (int v = 0; v < W; ++v) {
      const int j = by * kPenY + 2 * v + jj;
      const long long r0 = static_cast<long long>(j) * a.gx + i - static_cast<long long>(kb) * plane;
      yp[v] = y + (a.mirror ? a.n - 1 - r0 : r0);
      sa[v] = (i < a.gx && j < a.gy) ? kb : 0x3fffffff;
    }
    const int nst = (S + G - 1) / G;
#pragma unroll 1
    for (int g = 0; g < nst; ++g) {
      const int slot = g % NS;
#pragma unroll
      for (int v = 0; v < W; ++v) {
        const unsigned fb = bar_full + (v * NS + slot) * 8;
#ifdef P2_WATCH
        if (lane == 0) {
          prog[16] = g;
          prog[17] = v;
        }
#endif
        if (g >= NS) {
          unsigned spins = 0;
          (void)spins;
          while (!p2_mbar_try(bar_empty + (v * NS + slot) * 8, static_cast<unsigned>((g / NS) - 1) & 1u)) {
            P2_GUARD(1, g, v)
            P2_SLEEP();
          }
        }
        if (lane == 0) P2_TS(4 * 4096 + g * 4 + v, clock64())
        const unsigned drec = sbase + kP2OffRec + static_cast<unsigned>((v * NS + slot) * G) * 768u;
        const unsigned drhs = sbase + kP2OffRhs + static_cast<unsigned>((v * NS + slot) * G) * 256u + lane * 8u;
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(G * 768) : "memory");
          const unsigned char* src = src0 + (static_cast<size_t>(v) * (S + a.pad) + static_cast<size_t>(g) * G) * 768;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(drec),
              "l"(src), "r"(G * 768), "r"(fb)
              : "memory");
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
          const int s = g * G + q;
          const bool act = static_cast<unsigned>(s - sa[v]) < static_cast<unsigned>(gz);
          const i64* p = act ? yp[v] + static_cast<long long>(s) * ystride : y;
          if (P2_KNOB & 32) p = y + ((static_cast<long long>(t) * 64 * 1024 + static_cast<long long>(s) * 256 + v * 64 + lane) & (a.n - 1));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(drhs + q * 256u), "l"(p),
                       "r"(act ? 8 : 0)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fb) : "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef P2_WATCH
  } else if (w == W + 2) {
    if (lane == 0) {
      const long long t0 = clock64();
      while (clock64() - t0 < 4000000000ll) {
        if (reinterpret_cast<volatile int*>(p2_smem + kP2OffProg)[20] == W) break;  // compute warps done
      }
      if (reinterpret_cast<volatile int*>(p2_smem + kP2OffProg)[20] != W) {
        volatile unsigned long long* o = g_p2_watch + blockIdx.x * 16;
        o[0] = t; o[1] = bx; o[2] = by;
        for (int qq = 0; qq < 4; ++qq) o[3 + qq] = prog[qq];
        o[7] = prog[16]; o[8] = prog[17];
        for (int qq = 0; qq < 2 * W * NS; ++qq) {  // mbarrier phase parity bits: test_wait.parity 0
          unsigned ok;
          asm volatile("{ .reg .pred P1; mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], 0; selp.u32 %0, 1, 0, P1; }"
                       : "=r"(ok) : "r"(bar_full + qq * 8) : "memory");
          o[9] |= static_cast<unsigned long long>(ok) << qq;
        }
        o[15] = 1;
        __threadfence_system();
      }
    }
#endif
  } else if (w == W + 1) {
    // ------------------------------------------------------------ importer
    // lanes 0..15: -y face (column xl of warp 0's jj = 0 row, from brick by-1);
    // lanes 16..16+2W-1: -x face (row 2v + jj of the brick, from brick bx-1)
    bool on = false;
    const ulonglong2* src = nullptr;
    unsigned dst = 0, dstride = 0;
    int cw = 0, coff = 0;  // consumer warp and lane offset: row k is read at its step k + coff
    if (lane < 16) {
      const int i = bx * kPenX + lane, j = by * kPenY;
      on = by > 0 && i < a.gx;
      src = a.xz + (static_cast<long long>(j - 1) * a.gx + i);
      dst = sbase + static_cast<unsigned>(lane) * 16u;  // ring 0, lane xl
      dstride = 256u;
      cw = 0;
      coff = lane;
    } else if (lane < 16 + 2 * W) {
      const int v = (lane - 16) >> 1, jj = (lane - 16) & 1;
      const int i = bx * kPenX, j = by * kPenY + 2 * v + jj;
      on = bx > 0 && j < a.gy;
      src = a.xz + (static_cast<long long>(j) * a.gx + i - 1);
      dst = sbase + kP2OffXr + static_cast<unsigned>((v * 2 + jj) * R) * 16u;
      dstride = 16u;
      cw = v;
      coff = jj;
    }
    int k = 0;
    const int kend = on ? gz : 0;
    int seen = 0;  // last observed progress of the consumer warp
#pragma unroll 1
    unsigned spins = 0;
    (void)spins;
    while (__any_sync(0xffffffffu, k < kend)) {
      P2_GUARD(2, k, kend)
      u64 v[kP2PI], tg[kP2PI];
#pragma unroll
      for (int q = 0; q < kP2PI; ++q) {
        v[q] = 0;
        tg[q] = 1;
        if (k + q < kend) pen_xz_load(src + static_cast<long long>(k + q) * plane, v[q], tg[q]);
      }
      // deliver the valid prefix whose ring slots the consumer has released
      int dcount = 0;
      bool run = true;
#pragma unroll
      for (int q = 0; q < kP2PI; ++q) {
        const int kk = k + q;
        run = run && kk < kend && tg[q] == epoch + static_cast<u64>(kk);
        if (run && kk - R + coff + 1 > seen) {
          seen = prog[cw];  // slot of row kk - R must have been read
          run = kk - R + coff + 1 <= seen;
        }
        if (run) {
          const unsigned d = dst + (static_cast<unsigned>(kk) & RM) * dstride;
          p2_sts_word(d, v[q], kk);
          if (lane == 0 || lane == 16) P2_TS((lane == 0 ? 5 : 6) * 4096 + kk, clock64())
          ++dcount;
        }
      }
      k += dcount;
#ifdef P2_GUARDS
      if (lane >= 16 && lane < 24) prog[8 + lane - 16] = k;
#endif
    }
  } else {
    // ------------------------------------------------------------ compute
    // One stage (G steps) per outer iteration, the steps unrolled: the
    // operands of a step are plain shared-memory loads the compiler may
    // schedule early, the row is computed speculatively from the ring / import
    // words as loaded and only then are their tags checked (a stale word,
    // rare, sends the whole warp through the re-poll path and recomputes), so
    // the dependent chain of a step is shuffle -> products -> division.
    const int xl = lane & 15, jj = lane >> 4;
    const int i = bx * kPenX + xl, j = by * kPenY + 2 * w + jj;
    const bool ing = i < a.gx && j < a.gy;
    const int kb = xl + jj;
    const int sa = ing ? kb : 0x3fffffff;
    const bool xin = xl == 0 && bx > 0;                 // -x value imported (importer -> xr ring)
    const bool yin = !(P2_KNOB & 128) && jj == 0 && (w > 0 || by > 0);  // -y value from ring w (warp w-1 or importer)
    const bool pprod = w + 1 < W && jj == 1;            // feeds warp w+1 through ring w+1
    const bool yprod = w + 1 < W;
    const bool exp_ = (xl == kPenX - 1 && bx + 1 < a.nbx) || (w == W - 1 && jj == 1 && by + 1 < a.nby);
    const unsigned ring_cons = sbase + (static_cast<unsigned>(w) * R * 16 + xl) * 16u;
    const unsigned ring_prod = sbase + (static_cast<unsigned>(w + 1) * R * 16 + xl) * 16u;
    const unsigned xr_cons = sbase + kP2OffXr + static_cast<unsigned>((w * 2 + jj) * R) * 16u;
    const unsigned char* rec0 = p2_smem + kP2OffRec + static_cast<size_t>(w * NS * G) * 768u;
    const unsigned char* rhs0 = p2_smem + kP2OffRhs + static_cast<size_t>(w * NS * G) * 256u;
    const unsigned fb0 = bar_full + w * NS * 8, eb0 = bar_empty + w * NS * 8;
    u64 ek = epoch - static_cast<u64>(kb);  // global export tag of the step's row: epoch + k
    const long long r0 = static_cast<long long>(j) * a.gx + i - static_cast<long long>(kb) * plane;
    const long long nat0 = a.mirror ? a.n - 1 - r0 : r0;
    i64* op = out + nat0;
    ulonglong2* ep = a.xz + r0;
    i64 zc = 0, zxs = 0, zys = 0;  // own previous row; lane xl-1's and lane (xl, 0)'s previous rows
    u64 ymx = 0, zmx = 0;
    const double gam = prescale != nullptr ? *prescale : 1.0;
    const bool mirror = a.mirror != 0;
    const int nst = (S + G - 1) / G;
#pragma unroll 1
    for (int g = 0; g < nst; ++g) {
      const int slot = g & (NS - 1);
#ifdef P2_STAGETS
      if (lane == 0 && t == 0) g_p2_sts[4096 + w * 1024 + g] = clock64();
#endif
      {  // this stage's records and right-hand sides have landed
        unsigned spins = 0;
        (void)spins;
        while (!p2_mbar_try(fb0 + slot * 8, static_cast<unsigned>(g / NS) & 1u)) {
          P2_GUARD(3, g, slot)
        }
      }
      if (yprod) {  // ring back-pressure, once per stage: warp w+1 must have read row k - R
        const int need = (g + 1) * G - 1 - R;
        unsigned spins = 0;
        (void)spins;
        while (prog[w + 1] < need) {
          P2_GUARD(6, g, need)
          P2_SLEEP();
        }
      }
#ifdef P2_STAGETS
      if (lane == 0 && t == 0) g_p2_sts[w * 1024 + g] = clock64();
      if (lane == 0 && (g == 2 || g == 6)) {  // per brick: global time warp w enters stage 2 / 6
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g_p2_bt[(bx * 64 + by) * 16 + w * 2 + (g == 6)] = gt;
      }
#endif
      const unsigned char* recg = rec0 + static_cast<size_t>(slot * G) * 768u;
      const unsigned char* rhsg = rhs0 + static_cast<size_t>(slot * G) * 256u;
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int s = g * G + q;
        const int k = s - kb;
        const bool act = static_cast<unsigned>(s - sa) < static_cast<unsigned>(gz);
        const unsigned rs = static_cast<unsigned>(k) & RM;
        const int4 rc = *reinterpret_cast<const int4*>(recg + q * 768 + lane * 16);
        const u64 mg = *reinterpret_cast<const u64*>(recg + q * 768 + 512 + lane * 8);
        const u64 yv = *reinterpret_cast<const u64*>(rhsg + q * 256 + lane * 8);
        const bool pys = yin && act, pxs = xin && act;
        const unsigned ysa = ring_cons + rs * 256u, xsa = xr_cons + rs * 16u;
        // unconditional loads: a lane without that neighbour has a zero factor
        // (integer) or a clear presence bit (FP) for it, so any word is harmless
        u64 vv, xv;
        int vt, xt;
        p2_lds_word(ysa, vv, vt);
        p2_lds_word(xsa, xv, xt);
        auto row = [&](i64 zx, i64 zy) -> i64 {
          if constexpr (FP) {
            double acc = __longlong_as_double(static_cast<long long>(yv));
            if (prescale != nullptr) acc = __ddiv_rn(acc, gam);
            auto term = [&](double c, int f, i64 zb, int bit) {
              const double tt = __dsub_rn(c, __dmul_rn(static_cast<double>(f), __longlong_as_double(zb)));
              return (rc.w >> bit) & 1 ? tt : c;
            };
            if (mirror) {  // upper factor: +x, +y, +z columns ascending
              acc = term(acc, rc.x, zx, 10);
              acc = term(acc, rc.y, zy, 11);
              acc = term(acc, rc.z, zc, 12);
            } else {       // lower factor: -z, -y, -x columns ascending
              acc = term(acc, rc.z, zc, 12);
              acc = term(acc, rc.y, zy, 11);
              acc = term(acc, rc.x, zx, 10);
            }
            return __double_as_longlong(__ddiv_rn(acc, __longlong_as_double(static_cast<long long>(mg))));
          } else {
            const u64 sx = static_cast<u64>(static_cast<i64>(rc.z)) * static_cast<u64>(zc) +
                           static_cast<u64>(static_cast<i64>(rc.y)) * static_cast<u64>(zy) +
                           static_cast<u64>(static_cast<i64>(rc.x)) * static_cast<u64>(zx);
            SDivMagic gm;
            gm.u.m = mg;
            gm.u.sh1 = rc.w & 1;
            gm.u.sh2 = (rc.w >> 1) & 127;
            gm.den_neg = (rc.w >> 8) & 1;
            gm.den_is_m1 = 0;
            return sdiv(static_cast<i64>(yv - sx), gm);
          }
        };
        i64 z = row(xl == 0 ? static_cast<i64>(xv) : zxs, jj == 0 ? static_cast<i64>(vv) : zys);
        bool stx = pxs && xt != k + 1, sty = pys && vt != k + 1;
        if (__any_sync(0xffffffffu, stx || sty)) {  // a word not delivered yet (rare): re-poll, recompute
          unsigned spins = 0;
          (void)spins;
          do {
            if (stx) p2_lds_word(xsa, xv, xt);
            if (sty) p2_lds_word(ysa, vv, vt);
            stx = stx && xt != k + 1;
            sty = sty && vt != k + 1;
            P2_GUARD(4, s, k)
            P2_SLEEP();
          } while (__any_sync(0xffffffffu, stx || sty));
          z = row(xl == 0 ? static_cast<i64>(xv) : zxs, jj == 0 ? static_cast<i64>(vv) : zys);
        }
        // the next step's x and y neighbours at once: the shuffle is the next link of the chain
        const i64 zxn = __shfl_up_sync(0xffffffffu, z, 1);
        const i64 zyn = __shfl_xor_sync(0xffffffffu, z, 16);
        if (act && pprod) p2_sts_word(ring_prod + rs * 256u, static_cast<u64>(z), k);
        if (P2_KNOB & 64) {
          if (act) out[(static_cast<long long>(t) * 64 * 1024 + static_cast<long long>(s) * 256 + w * 64 + lane) & (a.n - 1)] = z;
        } else if (act) {
          *op = z;
        }
        asm volatile(
            "{ .reg .pred p; .reg .b128 t; setp.ne.b32 p, %3, 0; mov.b128 t, {%1, %2};\n"
            "@p st.global.relaxed.gpu.b128 [%0], t; }" ::"l"(ep),
            "l"(z), "l"(ek), "r"((int)(act && exp_)));
        if constexpr (CHECKED && !FP) {
          ymx |= yv ^ static_cast<u64>(static_cast<i64>(yv) >> 63);
          zmx |= static_cast<u64>(z ^ (z >> 63));
        }
        zc = z;
        zxs = zxn;
        zys = zyn;
        if (lane == 0) prog[w] = s + 1;
        op += ystride;
        ep += plane;
        ++ek;
      }
      __syncwarp();  // release the stage slot to the loader
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(eb0 + slot * 8) : "memory");
    }
#ifdef P2_WATCH
    if (lane == 0) atomicAdd(const_cast<int*>(&prog[20]), 1);
#endif
    if constexpr (CHECKED && !FP) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ymx |= static_cast<u64>(__shfl_down_sync(0xffffffffu, ymx, o));
        zmx |= static_cast<u64>(__shfl_down_sync(0xffffffffu, zmx, o));
      }
      if (lane == 0) {
        atomicMax(a.stats, static_cast<unsigned long long>(ymx + 1));
        atomicMax(a.stats + 1, static_cast<unsigned long long>(zmx + 1));
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.ticket + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      a.ticket[0] = 0;
      a.ticket[1] = 0;
      __threadfence();
    }
  }
}

}  // namespace igm
