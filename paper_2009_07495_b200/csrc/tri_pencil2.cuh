// tri_pencil2.cuh -- warp-specialised, cluster-coupled pencil wavefront for
// structured 7-point ILU(0) factors (sm_100a).  Same substitution, record
// stream and brick geometry as tri_pencil.cuh (k_tri_pencil); what changes is
// who waits for what, and where the brick-to-brick hand-offs travel.
//
// Integer path of apply_inverse (ilu.cpp:122-155) and FP64 path of
// apply_inverse_fp (ilu.cpp:157-180), bit-identical to k_tri_pencil.
//
// One CTA = one 16 x (2 kPenWarps) brick of z-pencils; CY CTAs stacked along y
// form a thread-block cluster (CY = 1: no cluster):
//   * kPenWarps COMPUTE warps: lane (xl, jj) of warp w walks pencil
//     (16 bx + xl, 2 kPenWarps by + 2 w + jj), row k at step k + xl + jj.
//     Every input of a step is in a register or shared memory: -x from lane
//     xl-1 (__shfl_up), -y from lane (xl, 0) (__shfl_xor 16) or a ring slot,
//     -z the lane's previous row.  The row is computed speculatively from the
//     ring / import words as loaded and their tags are checked afterwards (a
//     stale word, rare, sends the whole warp, kept converged, through a
//     re-poll and a recompute), so a step's dependent chain is shuffle ->
//     three wrapping products -> exact reciprocal division.
//   * one LOADER warp: per stage of G steps and compute warp, one
//     cp.async.bulk of the G record blocks (768 B each, the stream of
//     pencil.hpp) and a per-lane cp.async gather of the G right-hand sides,
//     completing on the stage's mbarrier; NS stages in flight per warp.
//   * one IMPORTER warp: polls, PI rows ahead per face lane, the tagged
//     (value, epoch + k) words that neighbour bricks OUTSIDE the cluster
//     export to global memory, and copies each valid word into the shared
//     ring its consumer lane reads.  The global round trip of those
//     hand-offs is thus paid off the critical path.
//   * inside a cluster the last warp of brick (bx, by) writes its jj = 1 rows
//     straight into ring 0 of brick (bx, by+1) with st.shared::cluster
//     (DSMEM, ~0.2 us instead of ~2 us through L2 and the importer).
// Shared-memory hand-off words are {z, k + 1} (16 B; the rings are cleared
// before the cluster barrier that precedes any remote write, and a slot holds
// rows k, k + R, ..., so k + 1 identifies the word).
// Deadlock freedom: clusters are taken in wavefront ticket order (a cluster
// waits only on clusters of earlier tickets, which are resident); inside a
// cluster brick by+1 waits only on brick by; compute warp w waits only on
// warp w-1, the importer and the loader; the importer never blocks (a word
// whose ring slot is still in use stays in global memory until the next
// round); the loader waits for a stage slot to be released, and a warp can
// run at most R <= NS*G steps ahead of its consumer (checked once per stage).
#pragma once

#include "tri_pencil.cuh"

namespace igm {

constexpr int kP2G = 8;    // steps per stage
constexpr int kP2NS = 4;   // stages per compute warp
constexpr int kP2R = 32;   // ring slots (rows); kP2R <= kP2NS * kP2G
constexpr int kP2PI = 8;   // importer: outstanding polls per face lane
constexpr int kP2Threads = 32 * (kPenWarps + 2);
static_assert(kP2R <= kP2NS * kP2G, "ring lead must not exceed the staged window");
static_assert(2 * kPenWarps + 16 <= 32, "importer lanes");

// dynamic shared memory layout (bytes)
constexpr unsigned kP2RingBytes = kPenWarps * kP2R * 16 * 16;  // [warp][slot][xl] {z, k+1}: y-values
constexpr unsigned kP2XrBytes = kPenWarps * 2 * kP2R * 16;     // [warp][jj][slot] {z, k+1}: x-imports
constexpr unsigned kP2RecBytes = kPenWarps * kP2NS * kP2G * 768;
constexpr unsigned kP2RhsBytes = kPenWarps * kP2NS * kP2G * 256;
constexpr unsigned kP2OffXr = kP2RingBytes;
constexpr unsigned kP2OffRec = kP2OffXr + kP2XrBytes;
constexpr unsigned kP2OffRhs = kP2OffRec + kP2RecBytes;
constexpr unsigned kP2OffBar = kP2OffRhs + kP2RhsBytes;  // full[w][NS], empty[w][NS]
constexpr unsigned kP2OffProg = kP2OffBar + 2 * kPenWarps * kP2NS * 8;  // [w] steps done; [8] ticket
constexpr unsigned kP2Smem = kP2OffProg + 128;

__device__ __forceinline__ void p2_mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
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
__device__ __forceinline__ void p2_sts_word(unsigned a, u64 z, int k) {
  asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(static_cast<unsigned>(z)),
               "r"(static_cast<unsigned>(z >> 32)), "r"(k + 1), "r"(0));
}
__device__ __forceinline__ void p2_sts_word_remote(unsigned a, u64 z, int k) {  // a: shared::cluster address
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(static_cast<unsigned>(z)),
               "r"(static_cast<unsigned>(z >> 32)), "r"(k + 1), "r"(0)
               : "memory");
}
__device__ __forceinline__ void p2_lds_word(unsigned a, u64& z, int& t) {
  unsigned lo, hi, pad;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(lo), "=r"(hi), "=r"(t), "=r"(pad) : "r"(a));
  z = (static_cast<u64>(hi) << 32) | lo;
}
__device__ __forceinline__ unsigned p2_mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ int p2_ld_remote(unsigned a) {
  int v;
  asm volatile("ld.relaxed.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void p2_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned p2_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

#ifdef P2_GUARDS  // diagnostics build (scripts/pencil2_proto.cu): spin guards that report and break
__device__ unsigned long long g_p2_rep[8 * 4];
__device__ unsigned g_p2_nrep;
__device__ __noinline__ void p2_report(int id, int x, int y) {
  atomicAdd(&g_p2_nrep, 1u);
  if (id >= 0 && id < 8 && atomicCAS(reinterpret_cast<unsigned long long*>(&g_p2_rep[id * 4]), 0ull, 1ull) == 0ull) {
    g_p2_rep[id * 4 + 1] = blockIdx.x;
    g_p2_rep[id * 4 + 2] = threadIdx.x;
    g_p2_rep[id * 4 + 3] = (static_cast<unsigned long long>(static_cast<unsigned>(x)) << 32) | static_cast<unsigned>(y);
  }
}
#define P2_GUARD(id_, xa_, ya_)     \
  if (++spins > (1u << 22)) {       \
    p2_report(id_, xa_, ya_);       \
    break;                          \
  }
#else
#define P2_GUARD(id_, xa_, ya_)
#endif
#ifdef P2_STAGETS  // per-brick global times of stage entries (scripts/pencil2_proto.cu)
__device__ unsigned long long g_p2_bt[64 * 64 * 16];
#endif

// PIPE: the z-slab hand-off of a pipelined row partition (PenArgs::zimp /
// zexp); a separate instantiation so the single-GPU kernel carries none of it
template <bool CHECKED, bool FP, int CY, bool PIPE = false>
__global__ void __launch_bounds__(kP2Threads, 1)
    k_tri_pencil2(PenArgs a, const i64* __restrict__ y, i64* __restrict__ out, const int* stop, const int* err,
                  const double* prescale) {
  extern __shared__ __align__(128) unsigned char p2_smem[];
  // the cycle already ended (Ctl::stop / Ctl::err): uniform over the grid, so
  // every CTA of a cluster returns before any cluster barrier.  Pipelined
  // slabs pass err = nullptr: an error can be rank-local (encode), and the
  // neighbours' wavefronts wait on this one's words -- only the replicated
  // stop ends all of them together
  if (stop != nullptr && (*stop | (err != nullptr ? *err : 0)) != 0) return;
  constexpr int W = kPenWarps, G = kP2G, NS = kP2NS, R = kP2R;
  constexpr unsigned RM = R - 1;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(p2_smem));
  const unsigned bar_full = sbase + kP2OffBar, bar_empty = bar_full + W * NS * 8;
  volatile int* prog = reinterpret_cast<volatile int*>(p2_smem + kP2OffProg);
  const unsigned rank = CY > 1 ? p2_cluster_rank() : 0u;
  if (tid == 0) {
    if (rank == 0) prog[8] = atomicAdd(a.ticket, 1);  // one ticket per cluster
    for (int q = 0; q < W * NS; ++q) {
      p2_mbar_init(bar_full + q * 8, 33);  // 32 gathering lanes (noinc) + the bulk copy's expect_tx
      p2_mbar_init(bar_empty + q * 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 8) prog[tid] = 0;
  {  // clear the rings: shared memory keeps words of earlier kernels
    uint4* rz = reinterpret_cast<uint4*>(p2_smem);
    for (int q = tid; q < static_cast<int>((kP2RingBytes + kP2XrBytes) / 16); q += kP2Threads)
      rz[q] = make_uint4(0, 0, 0, 0);
  }
  if constexpr (CY > 1) p2_cluster_sync();  // rings cleared cluster-wide before any remote write
  else __syncthreads();
  const int t = (CY > 1 ? p2_ld_remote(p2_mapa(sbase + kP2OffProg + 32, 0)) : prog[8]) * CY + static_cast<int>(rank);
  const int code = __ldg(a.brick_of_ticket + t);
  const int bx = code & 0xffff, by = code >> 16;
  const int gz = a.gz, S = a.S;
  const long long plane = static_cast<long long>(a.gx) * a.gy;
  const u64 epoch = a.epoch;
  const long long ystride = a.mirror ? -plane : plane;
  const bool ynext_remote = CY > 1 && static_cast<int>(rank) + 1 < CY && by + 1 < a.nby;  // brick by+1 in this cluster
  const bool yprev_global = by > 0 && (CY == 1 || rank == 0);                            // brick by-1 in another

  if (w == W) {
    // ------------------------------------------------------------ loader
    const int xl = lane & 15, jj = lane >> 4, kb = xl + jj;
    const int i = bx * kPenX + xl;
    const unsigned char* src0 = reinterpret_cast<const unsigned char*>(a.rec) +
                                static_cast<size_t>(t) * W * static_cast<size_t>(S + a.pad) * 768;
    const i64* yp[W];  // this lane's rhs pointer at step 0, per compute warp
    int sa[W];         // and its activity window [sa, sa + gz)
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
        if (g >= NS) {
          unsigned spins = 0;
          (void)spins;
          while (!p2_mbar_try(bar_empty + (v * NS + slot) * 8, static_cast<unsigned>((g / NS) - 1) & 1u)) {
            P2_GUARD(1, g, v)
          }
        }
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
          if (PIPE && a.zimp != nullptr && act && s == sa[v]) {  // plane 0: the neighbour rank's value (pipelined slabs)
            const int j = by * kPenY + 2 * v + jj;
            const long long idx = a.mirror ? static_cast<long long>(a.gy - 1 - j) * a.gx + (a.gx - 1 - i)
                                           : static_cast<long long>(j) * a.gx + i;
            u64 zv, zt;
            unsigned spins = 0;
            (void)spins;
            do {
              asm volatile("{ .reg .b128 t; ld.relaxed.sys.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                           : "=l"(zv), "=l"(zt)
                           : "l"(a.zimp + idx)
                           : "memory");
              P2_GUARD(7, s, v)
            } while (zt != a.zepoch + static_cast<u64>(idx));
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(drhs + q * 256u), "l"(zv) : "memory");
            continue;
          }
          const i64* p = act ? yp[v] + static_cast<long long>(s) * ystride : y;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(drhs + q * 256u), "l"(p),
                       "r"(act ? 8 : 0)
                       : "memory");
        }
        if (PIPE && a.zimp != nullptr) asm volatile("fence.acq_rel.cta;" ::: "memory");  // imported words stored above
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(fb) : "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (w == W + 1) {
    // ------------------------------------------------------------ importer
    // lanes 0..15: -y face (column xl of warp 0's jj = 0 row, from brick by-1,
    // only when that brick is in another cluster); lanes 16..16+2W-1: -x face
    // (row 2v + jj of the brick, from brick bx-1)
    bool on = false;
    const ulonglong2* src = nullptr;
    unsigned dst = 0, dstride = 0;
    int cw = 0, coff = 0;  // consumer warp and lane offset: row k is read at its step k + coff
    if (lane < 16) {
      const int i = bx * kPenX + lane, j = by * kPenY;
      on = yprev_global && i < a.gx;
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
    unsigned spins = 0;
    (void)spins;
#pragma unroll 1
    while (__any_sync(0xffffffffu, k < kend)) {
      P2_GUARD(2, k, kend)
      u64 v[kP2PI], tg[kP2PI];
#pragma unroll
      for (int q = 0; q < kP2PI; ++q) {
        v[q] = 0;
        tg[q] = ~0ull;
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
          p2_sts_word(dst + (static_cast<unsigned>(kk) & RM) * dstride, v[q], kk);
          ++dcount;
        }
      }
      k += dcount;
    }
  } else {
    // ------------------------------------------------------------ compute
    const int xl = lane & 15, jj = lane >> 4;
    const int i = bx * kPenX + xl, j = by * kPenY + 2 * w + jj;
    const bool ing = i < a.gx && j < a.gy;
    const int kb = xl + jj;
    const int sa = ing ? kb : 0x3fffffff;
    const bool xin = xl == 0 && bx > 0;                 // -x value imported (importer -> xr ring)
    const bool yin = jj == 0 && (w > 0 || by > 0);      // -y value from ring w (warp w-1, brick by-1 or importer)
    const bool last = w == W - 1;
    const bool pprod = jj == 1 && (!last || ynext_remote);  // feeds ring w+1 (or the next brick's ring 0)
    const bool yprod = !last || ynext_remote;
    const bool exp_ = (xl == kPenX - 1 && bx + 1 < a.nbx) || (last && jj == 1 && by + 1 < a.nby && !ynext_remote);
    const unsigned ring_cons = sbase + (static_cast<unsigned>(w) * R * 16 + xl) * 16u;
    // the consumer's ring: ring w+1 here, or ring 0 of the cluster's next CTA
    const unsigned ring_prod_l = sbase + (static_cast<unsigned>(last ? 0 : w + 1) * R * 16 + xl) * 16u;
    const unsigned ring_prod = (CY > 1 && last && ynext_remote) ? p2_mapa(ring_prod_l, rank + 1) : ring_prod_l;
    const unsigned prog_cons = (CY > 1 && last && ynext_remote)
                                   ? p2_mapa(sbase + kP2OffProg, rank + 1)
                                   : sbase + kP2OffProg + static_cast<unsigned>(w + 1) * 4u;
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
      if (lane == 0 && (g == 2 || g == 6)) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        g_p2_bt[(bx * 64 + by) * 16 + w * 2 + (g == 6)] = gt;
      }
#endif
      {  // this stage's records and right-hand sides have landed
        unsigned spins = 0;
        (void)spins;
        while (!p2_mbar_try(fb0 + slot * 8, static_cast<unsigned>(g / NS) & 1u)) {
          P2_GUARD(3, g, slot)
        }
      }
      if (yprod) {  // ring back-pressure, once per stage: the consumer must have read row k - R
        const int need = (g + 1) * G - 1 - R;
        unsigned spins = 0;
        (void)spins;
        while ((CY > 1 && last) ? p2_ld_remote(prog_cons) < need : prog[w + 1] < need) {
          P2_GUARD(6, g, need)
        }
      }
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
          } while (__any_sync(0xffffffffu, stx || sty));
          z = row(xl == 0 ? static_cast<i64>(xv) : zxs, jj == 0 ? static_cast<i64>(vv) : zys);
        }
        // the next step's x and y neighbours at once: the shuffle is the next link of the chain
        const i64 zxn = __shfl_up_sync(0xffffffffu, z, 1);
        const i64 zyn = __shfl_xor_sync(0xffffffffu, z, 16);
        if (act && pprod) {
          if (CY > 1 && last) p2_sts_word_remote(ring_prod + rs * 256u, static_cast<u64>(z), k);
          else p2_sts_word(ring_prod + rs * 256u, static_cast<u64>(z), k);
        }
        if (act) *op = z;
        if (PIPE && a.zexp != nullptr && act && k == a.kexp) {  // the next rank's plane-0 value (pipelined slabs)
          const long long idx = a.mirror ? static_cast<long long>(a.gy - 1 - j) * a.gx + (a.gx - 1 - i)
                                         : static_cast<long long>(j) * a.gx + i;
          const u64 tz = a.zepoch + static_cast<u64>(idx);
          asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.sys.global.b128 [%0], t; }" ::"l"(a.zexp + idx),
                       "l"(static_cast<u64>(z)), "l"(tz)
                       : "memory");
        }
        asm volatile(
            "{ .reg .pred p; .reg .b128 t; setp.ne.b32 p, %3, 0; mov.b128 t, {%1, %2};\n"
            "@p st.global.relaxed.gpu.b128 [%0], t; }" ::"l"(ep),
            "l"(z), "l"(ek), "r"((int)(act && exp_)));
        if constexpr (CHECKED && !FP) {  // magnitude bounds: OR of v ^ (v >> 63) (idle lanes contribute 0)
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
    if constexpr (CHECKED && !FP) {  // |v| <= (v ^ (v >> 63)) + 1
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
  // no CTA may leave while a cluster peer can still touch its shared memory;
  // the last CTA to finish resets the ticket counters for the next launch
  if constexpr (CY > 1) p2_cluster_sync();
  else __syncthreads();
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
