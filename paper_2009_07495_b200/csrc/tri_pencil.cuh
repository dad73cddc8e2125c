// tri_pencil.cuh -- structured-grid ILU(0) substitution as a warp-synchronous
// pencil wavefront (sm_100a).  Stream layout and applicability: pencil.hpp.
//
// Integer path of apply_inverse (ilu.cpp:122-155): z_r = trunc((y_r - sum_d
// L_rd z_d) / diag_r), products and the sum wrapping mod 2^64 (any summation
// order gives the same word), the division by the raw diagonal through its
// exact reciprocal (fx_core.cuh sdiv, INT64_MIN / -1 -> INT64_MIN).
//
// One CTA = one 16 x 16 brick of z-pencils, one pencil per thread, 8 warps of
// 16 x 2 pencils.  Lane (xl, jj) of warp w handles row (i, j, k) at warp step
// s = k + xl + jj, so per step:
//   -x value : lane xl-1's row of the previous step     (__shfl_up)
//   -y value : jj = 1: lane (xl, 0) of the previous step (__shfl_xor 16)
//              jj = 0: warp w-1's jj = 1 lanes, handed over through a
//              shared-memory ring of tagged (value, tag) words, the warp
//              running >= 2 steps behind its producer warp
//   -z value : the lane's own previous row (a register)
// so a step costs two shuffles, three wrapping products, the reciprocal
// division -- no CTA barrier per level.  Brick faces: lanes xl = 0 and warp
// 0's jj = 0 lanes read the neighbour brick's exported values as tagged
// 128-bit words (value, epoch ^ value) from global memory, loaded P steps
// ahead with the row's record and right-hand side; the exporting lanes
// (xl = 15, warp 7's jj = 1) store them with one strong 128-bit store.  A
// brick only waits on bricks of an earlier ticket (wavefront order bx+by),
// every brick below it is already resident: no deadlock for any grid.
#pragma once

#include "fx_core.cuh"
#include "pencil.hpp"

namespace igm {

constexpr int kPenThreads = 32 * kPenWarps;

// dynamic shared memory: the in-CTA y rings, then the D-step prefetch ring
__host__ __device__ inline size_t pencil_ring_bytes(int R) { return static_cast<size_t>(kPenWarps - 1) * R * 16 * 16; }
__host__ __device__ inline size_t pencil_smem_bytes(int R, int D) {
  return pencil_ring_bytes(R) + static_cast<size_t>(D) * 16384;
}

struct PenArgs {
  int gx, gy, gz, nbx, nby, S, R, pad;  // R: shared-memory ring depth (steps, power of 2); pad: idle blocks per warp
  long long n;
  int mirror;                       // backward solve: natural row = n - 1 - solve-order row
  const void* rec;                  // [ticket][warp][step] blocks of 768 B: 32 x int4 record, 32 x u64 reciprocal
  const int* brick_of_ticket;
  ulonglong2* xz;                   // exported values by solve-order row (tagged)
  unsigned long long epoch;         // per launch, hashed, non-zero
  int* ticket;
  unsigned long long* stats;        // [max|y|, max|z|] of this apply (checked mode's bound)
  // z-slab pipelining (k_tri_pencil2 only; dist.py's row-partitioned solve):
  // the right-hand sides of solve-order plane 0 come from tagged words
  // zimp[idx] = (value, zepoch + idx) written by the neighbour rank (idx =
  // natural j * gx + i), and plane kexp's results go to zexp[idx] likewise
  const ulonglong2* zimp = nullptr;
  ulonglong2* zexp = nullptr;
  int kexp = -1;
  unsigned long long zepoch = 0;
};

__device__ __forceinline__ void pen_xz_load(const ulonglong2* p, u64& v, u64& tg) {
  asm volatile("{ .reg .b128 t; ld.global.relaxed.gpu.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(v), "=l"(tg)
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ u64 pen_xz_wait(const ulonglong2* p, u64 epoch) {
  u64 v, tg;
  do {
    pen_xz_load(p, v, tg);
  } while (tg != (epoch ^ v));
  return v;
}
__device__ __forceinline__ void pen_xz_put(ulonglong2* p, u64 v, u64 epoch) {
  asm volatile("{ .reg .b128 t; mov.b128 t, {%0, %1}; st.global.relaxed.gpu.b128 [%2], t; }" ::"l"(v),
               "l"(epoch ^ v), "l"(p)
               : "memory");
}
__device__ __forceinline__ void pen_lds2(unsigned a, u64& v, u64& tg) {
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v), "=l"(tg) : "r"(a) : "memory");
}
__device__ __forceinline__ void pen_sts2(unsigned a, u64 v, u64 tg) {
  asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(v), "l"(tg) : "memory");
}
__device__ __forceinline__ u64 pen_tag(u64 epoch, int k) {
  return epoch ^ (static_cast<u64>(k + 1) * 0x9E3779B97F4A7C15ull);
}
__device__ __forceinline__ u64 pen_abs(i64 v) { return v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v); }

#ifdef PEN_TRACE
__device__ unsigned long long g_pen_ts[kPenWarps * 4096];
__device__ unsigned long long g_pen_ph[kPenWarps * 512 * 8];
__device__ unsigned long long g_pen_cnt[kPenWarps * 4];
#define PEN_PH(q) if (t == 0 && lane == 0 && s < 512) g_pen_ph[(w * 512 + s) * 8 + (q)] = clock64();
#else
#define PEN_PH(q)
#endif
#ifndef PEN_RING_LD
#define PEN_RING_LD "ld.volatile.shared.v2.u64"
#endif

// prefetch ring: per step D slot of 16 KB = four 16-byte fields x 256 lanes
constexpr unsigned kPenFRec = 0, kPenFMy = 4096, kPenFXi = 8192, kPenFYi = 12288, kPenStep = 16384;

// FP: the same substitutions in FP64 on the integer factors (apply_inverse_fp,
// ilu.cpp:157-180): acc = y (optionally / gamma, refine.cpp:17), acc -= L_rd
// * z_d over the row's entries in CSR order (-z, -y, -x for the lower factor;
// +x, +y, +z for the upper), then acc / diag, every operation rounded on its
// own (no contraction); absent entries are skipped, not subtracted as zero
// (a -0 rhs must stay -0).  The stream's reciprocal field holds the diagonal
// as a double.
template <int D, bool CHECKED, bool FP>
__global__ void __launch_bounds__(kPenThreads, 1)
    k_tri_pencil(PenArgs a, const i64* __restrict__ y, i64* __restrict__ out, const int* stop, const int* err,
                 const double* prescale) {
  extern __shared__ __align__(16) unsigned char pen_smem[];
  __shared__ int s_t;
  __shared__ volatile int s_prog[kPenWarps];
  if (stop != nullptr && (*stop | *err) != 0) return;  // the cycle already ended (Ctl::stop / Ctl::err)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, xl = lane & 15, jj = lane >> 4;
  if (tid == 0) s_t = atomicAdd(a.ticket, 1);
  if (tid < kPenWarps) s_prog[tid] = 0;
  {  // clear the in-CTA rings: shared memory keeps words of earlier kernels
    uint4* rz = reinterpret_cast<uint4*>(pen_smem);
    for (int q = tid; q < static_cast<int>(pencil_ring_bytes(a.R) / 16); q += kPenThreads) rz[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const int t = s_t;
  const int code = __ldg(a.brick_of_ticket + t);
  const int bx = code & 0xffff, by = code >> 16;
  const int i = bx * kPenX + xl, j = by * kPenY + 2 * w + jj;
  const bool ing = i < a.gx && j < a.gy;
  const int gz = a.gz, S = a.S;
  const long long plane = static_cast<long long>(a.gx) * a.gy;
  const int kb = xl + jj;                  // k = s - kb
  const int sa = ing ? kb : 0x3fffffff;    // active iff (unsigned)(s - sa) < gz
  const bool xin = xl == 0 && bx > 0;                // -x value from the neighbour brick
  const bool yin = w == 0 && jj == 0 && by > 0;      // -y value from the neighbour brick
  const bool ycons = w > 0 && jj == 0;               // -y value from warp w-1 (shared-memory ring)
  const bool yprod = w + 1 < kPenWarps;              // this warp feeds warp w+1
  const bool pprod = yprod && jj == 1;
  const bool plead = w > 0 && lane == 0;
  const bool exp_ = (xl == kPenX - 1 && bx + 1 < a.nbx) || (w == kPenWarps - 1 && jj == 1 && by + 1 < a.nby);
  const unsigned Rm = static_cast<unsigned>(a.R - 1);
  const unsigned ring0 = static_cast<unsigned>(__cvta_generic_to_shared(pen_smem));
  const unsigned ring_prod = ring0 + (static_cast<unsigned>(w) * a.R * 16 + xl) * 16u;       // ring w
  const unsigned ring_cons = ring0 + (static_cast<unsigned>(w - 1) * a.R * 16 + xl) * 16u;   // ring w-1
  const unsigned pre0 = ring0 + static_cast<unsigned>(pencil_ring_bytes(a.R)) + static_cast<unsigned>(tid) * 16u;
  const unsigned prog_me = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(&s_prog[w])));
  const u64 epoch = a.epoch;
  // every handed-over word (shared ring or global export) is (z, epoch ^ kc(k) ^ z),
  // kc(k) = (k + 1) * C: a word of another launch, another row of the ring
  // slot or a torn word fails the check
  constexpr u64 C = 0x9E3779B97F4A7C15ull;
  u64 kc = static_cast<u64>(1 - kb) * C;
  const long long r0 = static_cast<long long>(j) * a.gx + i - static_cast<long long>(kb) * plane;  // row at s = 0
  const long long ystride = a.mirror ? -plane : plane;
  const long long nat0 = a.mirror ? a.n - 1 - r0 : r0;

  // ---- prefetch side (step sp = s + D - 1): record block, reciprocal, rhs, face words.
  // The stream is padded with idle blocks per warp, so the record copies never
  // need a bound check; rhs and face copies are predicated on the row being
  // active (the rhs zero-filled otherwise: idle lanes then compute 0 / 1 = 0).
  const unsigned char* bp = reinterpret_cast<const unsigned char*>(a.rec) +
                            (static_cast<size_t>(t) * kPenWarps + w) * static_cast<size_t>(S + a.pad) * 768 + lane * 16;
  const i64* yp = y + nat0;
  const ulonglong2* xpf = a.xz + r0;
  unsigned pslot = 0;
  int sp = 0;
  const long long gxl = a.gx;
  auto issue = [&]() {
    const unsigned d = pre0 + pslot;
    const bool act = static_cast<unsigned>(sp - sa) < static_cast<unsigned>(gz);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + kPenFRec), "l"(bp) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + kPenFMy), "l"(bp + 512 - lane * 8) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d + kPenFMy + 8), "l"(act ? yp : y),
                 "r"(act ? 8 : 0)
                 : "memory");
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %2, 0;\n"
        "@p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(d + kPenFXi), "l"(xpf - 1), "r"((int)(xin && act))
        : "memory");
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %2, 0;\n"
        "@p cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(d + kPenFYi), "l"(xpf - gxl), "r"((int)(yin && act))
        : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    ++sp;
    bp += 768;
    yp += ystride;
    xpf += plane;
    pslot = pslot + kPenStep == D * kPenStep ? 0 : pslot + kPenStep;
  };
#pragma unroll 1
  for (int q = 0; q < D - 1; ++q) issue();

  // ---- current side (step s)
  i64* op = out + nat0;
  ulonglong2* ep = a.xz + r0;
  unsigned cslot = 0;
  i64 zc = 0;
  u64 ymx = 0, zmx = 0;
  const double gam = prescale != nullptr ? *prescale : 1.0;
  int cons_seen = 0;  // last observed progress of warp w+1 (ring back-pressure)
#pragma unroll 1
  for (int s = 0; s < S; ++s) {
#ifdef PEN_TRACE
    if (t == 0 && lane == 0 && s < 4096) g_pen_ts[w * 4096 + s] = clock64();
#endif
    const int k = s - kb;
    const bool act = static_cast<unsigned>(s - sa) < static_cast<unsigned>(gz);
    const unsigned rs = (static_cast<unsigned>(k) & Rm) * 256u;
    const u64 want = epoch ^ kc;
    __syncwarp();  // reconverge after a (rare) divergent stale path: the shuffles' fast path
    const i64 zxs = __shfl_up_sync(0xffffffffu, zc, 1);
    const i64 zys = __shfl_xor_sync(0xffffffffu, zc, 16);
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");  // this step's group (the newest is s + D - 2)
    const unsigned d = pre0 + cslot;
    // the lane's -y source: warp w-1's ring slot or the prefetched import word
    const bool pys = (ycons || yin) && act, pxs = xin && act;
    const unsigned ysa = ycons ? ring_cons + rs : d + kPenFYi;
    int4 rc;
    u64 mg, yv, xv, xt, vv, vt;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(rc.x), "=r"(rc.y), "=r"(rc.z), "=r"(rc.w)
                 : "r"(d + kPenFRec)
                 : "memory");
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(mg), "=l"(yv) : "r"(d + kPenFMy) : "memory");
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %3, 0; mov.b64 %0, 0; mov.b64 %1, 0;\n"
        "@p ld.volatile.shared.v2.u64 {%0, %1}, [%2]; }"
        : "=l"(vv), "=l"(vt)
        : "r"(ysa), "r"((int)pys)
        : "memory");
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %3, 0; mov.b64 %0, 0; mov.b64 %1, 0;\n"
        "@p ld.shared.v2.u64 {%0, %1}, [%2]; }"
        : "=l"(xv), "=l"(xt)
        : "r"(d + kPenFXi), "r"((int)pxs)
        : "memory");
    issue();  // the prefetch of step s + D - 1: its slot was read last step
    if ((pys && vt != (want ^ vv)) || (pxs && xt != (want ^ xv))) {  // not there yet when fetched (rare)
      if (pxs)
        while (xt != (want ^ xv)) pen_xz_load(ep - 1, xv, xt);
      if (pys) {
        if (ycons)
          while (vt != (want ^ vv)) pen_lds2(ysa, vv, vt);
        else
          while (vt != (want ^ vv)) pen_xz_load(ep - gxl, vv, vt);
      }
    }
    const i64 zx = xl == 0 ? static_cast<i64>(xv) : zxs;
    const i64 zy = jj == 0 ? static_cast<i64>(vv) : zys;
    i64 z;
    if constexpr (FP) {
      double acc = __longlong_as_double(static_cast<long long>(yv));
      if (prescale != nullptr) acc = __ddiv_rn(acc, gam);
      auto term = [&](double c, int f, i64 zb, int bit) {
        const double t = __dsub_rn(c, __dmul_rn(static_cast<double>(f), __longlong_as_double(zb)));
        return (rc.w >> bit) & 1 ? t : c;
      };
      if (a.mirror) {  // upper factor: +x, +y, +z columns ascending
        acc = term(acc, rc.x, zx, 10);
        acc = term(acc, rc.y, zy, 11);
        acc = term(acc, rc.z, zc, 12);
      } else {         // lower factor: -z, -y, -x columns ascending
        acc = term(acc, rc.z, zc, 12);
        acc = term(acc, rc.y, zy, 11);
        acc = term(acc, rc.x, zx, 10);
      }
      z = __double_as_longlong(__ddiv_rn(acc, __longlong_as_double(static_cast<long long>(mg))));
    } else {
      const u64 sx = static_cast<u64>(static_cast<i64>(rc.x)) * static_cast<u64>(zx) +
                     static_cast<u64>(static_cast<i64>(rc.y)) * static_cast<u64>(zy) +
                     static_cast<u64>(static_cast<i64>(rc.z)) * static_cast<u64>(zc);
      const i64 acc = static_cast<i64>(yv - sx);
      SDivMagic gm;
      gm.u.m = mg;
      gm.u.sh1 = rc.w & 1;
      gm.u.sh2 = (rc.w >> 1) & 127;
      gm.den_neg = (rc.w >> 8) & 1;
      gm.den_is_m1 = 0;
      z = sdiv(acc, gm);
    }
    if (yprod && s - a.R > cons_seen) {  // ring slot of row k - R must have been read by warp w+1
      do {
        cons_seen = s_prog[w + 1];
      } while (cons_seen < s - a.R);
    }
    const u64 tg = want ^ static_cast<u64>(z);
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %3, 0;\n"
        "@p st.volatile.shared.v2.u64 [%0], {%1, %2}; }" ::"r"(ring_prod + rs),
        "l"(z), "l"(tg), "r"((int)(act && pprod))
        : "memory");
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0;\n@p st.global.b64 [%0], %1; }" ::"l"(op), "l"(z),
                 "r"((int)act)
                 : "memory");
    asm volatile(
        "{ .reg .pred p; .reg .b128 t; setp.ne.b32 p, %3, 0; mov.b128 t, {%1, %2};\n"
        "@p st.global.relaxed.gpu.b128 [%0], t; }" ::"l"(ep),
        "l"(z), "l"(tg), "r"((int)(act && exp_))
        : "memory");

    if constexpr (CHECKED && !FP) {  // magnitude bounds: OR of v ^ (v >> 63) (idle lanes contribute 0)
      ymx |= yv ^ static_cast<u64>(static_cast<i64>(yv) >> 63);
      zmx |= static_cast<u64>(z ^ (z >> 63));
    }
    zc = z;
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0;\n@p st.volatile.shared.u32 [%0], %1; }" ::"r"(prog_me),
                 "r"(s + 1), "r"((int)plead)
                 : "memory");
    op += ystride;
    ep += plane;
    kc += C;
    cslot = cslot + kPenStep == D * kPenStep ? 0 : cslot + kPenStep;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
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
  // the last CTA to finish resets the ticket counters for the next launch
  // (ticket[1] counts finished CTAs), so no memset precedes a launch
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
