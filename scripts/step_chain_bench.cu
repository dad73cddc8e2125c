// Microbenchmark: cycles per step of the pencil wavefront's dependent chain
// (shuffles -> three wrapping products -> exact reciprocal division) with
// and without the per-step shared/global memory operations around it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -Ipaper_2009_07495_b200/csrc scripts/step_chain_bench.cu -o scripts/step_chain_bench
#include <cstdio>
#include <vector>

#include "fx_core.cuh"

using namespace igm;

template <int V>
__global__ void k_chain(int steps, const int4* rec, const u64* mag, const i64* rhs, i64* out, long long* cyc,
                        i64* sink, int ncomp, int spin, const i64* rhsg) {
  __shared__ __align__(8) unsigned long long sbar;
  __shared__ volatile int sdone;
  __shared__ int4 srec[32 * 32];
  __shared__ u64 smag[32 * 32], srhs[32 * 32];
  __shared__ ulonglong2 sring[32 * 16];
  __shared__ volatile int sprog[32];
  const int lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
    srec[q] = rec[q];
    smag[q] = mag[q];
    srhs[q] = rhs[q];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&sbar))));
    sdone = 0;
  }
  __syncthreads();
  if (static_cast<int>(threadIdx.x >> 5) >= ncomp) {  // spinner warp
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&sbar));
    while (sdone == 0) {
      if (spin == 1) {
        unsigned ok;
        asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0; selp.u32 %0, 1, 0, P1; }"
                     : "=r"(ok) : "r"(b) : "memory");
      } else if (spin == 2) {
        __nanosleep(200);
      }
    }
    return;
  }
  i64 zc = lane;
  int4 rc = srec[lane];
  u64 mg = smag[lane];
  u64 yv = srhs[lane];
  i64* op = out + threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 1
  for (int s = 0; s < steps; ++s) {
    if (V >= 1) {  // per-step operands from shared memory
      const int q = (s & 31) * 32 + lane;
      rc = srec[q];
      mg = smag[q];
      yv = srhs[q];
    }
    const i64 zxs = __shfl_up_sync(0xffffffffu, zc, 1);
    const i64 zys = __shfl_xor_sync(0xffffffffu, zc, 16);
    const u64 sx = static_cast<u64>(static_cast<i64>(rc.z)) * static_cast<u64>(zc) +
                   static_cast<u64>(static_cast<i64>(rc.y)) * static_cast<u64>(zys) +
                   static_cast<u64>(static_cast<i64>(rc.x)) * static_cast<u64>(zxs);
    const i64 acc = static_cast<i64>(yv - sx);
    SDivMagic gm;
    gm.u.m = mg;
    gm.u.sh1 = rc.w & 1;
    gm.u.sh2 = (rc.w >> 1) & 127;
    gm.den_neg = (rc.w >> 8) & 1;
    gm.den_is_m1 = 0;
    const i64 z = sdiv(acc, gm);
    if (V >= 2 && V != 6) {
      *op = z;
      op += 4096;
      if (op > out + (1 << 22)) op = out + threadIdx.x;
    }
    if (V == 7) {  // scattered rhs gather (one 8-B load per lane, every lane another plane) + scattered store
      const int kk = (s - (lane & 15) - (lane >> 4)) & 255;
      const i64 g = __ldcg(rhsg + static_cast<long long>((kk + 7) & 255) * 16384 + (threadIdx.x >> 5) * 32 + lane);
      yv ^= static_cast<u64>(g);
      out[static_cast<long long>(kk) * 16384 + (threadIdx.x >> 5) * 32 + lane] = z;
    }
    if (V == 6) {  // scattered output store: every lane a different plane (pencil layout)
      const int kk = (s - (lane & 15) - (lane >> 4)) & 255;
      out[static_cast<long long>(kk) * 16384 + (threadIdx.x >> 5) * 32 + lane] = z;
    }
    if (V == 3 || V == 5) {  // + a strong 128-bit export store on two lanes
      if ((lane & 15) == 15)
        asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.global.relaxed.gpu.b128 [%0], t; }" ::"l"(reinterpret_cast<ulonglong2*>(out) + (s & 1023) * 32 + lane),
                     "l"(z), "l"(z ^ 77)
                     : "memory");
    }
    if (V == 4 || V == 5) {  // + __syncwarp, volatile progress word, tagged ring store
      __syncwarp();
      sprog[threadIdx.x >> 5] = s;
      asm volatile("st.volatile.shared.v2.u64 [%0], {%1, %2};" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&sring[(s & 15) * 32 + lane]))),
                   "l"(z), "l"(z ^ 5)
                   : "memory");
    }
    zc = z;
  }
  const long long t1 = clock64();
  sdone = 1;
  if (lane == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = zc;
}

int main() {
  std::vector<int4> rec(32 * 32);
  std::vector<u64> mag(32 * 32);
  std::vector<i64> rhs(32 * 32);
  for (int q = 0; q < 32 * 32; ++q) {
    const i64 d = 65536 + 37 * q;
    const SDivMagic m = make_sdiv(d);
    rec[q] = make_int4(1000 + q, -2000 + q, 3000 - q, (m.u.sh1 & 1) | ((m.u.sh2 & 127) << 1) | (m.den_neg << 8));
    mag[q] = m.u.m;
    rhs[q] = static_cast<i64>(q) << 40;
  }
  int4* d_rec;
  u64* d_mag;
  i64 *d_rhs, *d_out, *d_sink;
  long long* d_cyc;
  cudaMalloc(&d_rec, rec.size() * 16);
  cudaMalloc(&d_mag, mag.size() * 8);
  cudaMalloc(&d_rhs, rhs.size() * 8);
  cudaMalloc(&d_out, (256ll * 16384 + 4096) * 8);
  cudaMalloc(&d_sink, 148 * 1024 * 8);
  cudaMalloc(&d_cyc, 148 * 32 * 8);
  cudaMemcpy(d_rec, rec.data(), rec.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(d_mag, mag.data(), mag.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_rhs, rhs.data(), rhs.size() * 8, cudaMemcpyHostToDevice);
  const int steps = 10000;
  for (int spin = 0; spin < 3; ++spin)
  for (int warps : {1, 4}) {
    for (int v = 0; v < 8; ++v) {
      if (spin && v != 5) continue;
      const int nthr = 32 * warps + (spin ? 64 : 0);
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) k_chain<0><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 1) k_chain<1><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 2) k_chain<2><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 3) k_chain<3><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 4) k_chain<4><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 7) k_chain<7><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out + 4096);
        if (v == 6) k_chain<6><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
        if (v == 5) k_chain<5><<<1, nthr>>>(steps, d_rec, d_mag, d_rhs, d_out, d_cyc, d_sink, warps, spin, d_out);
      }
      cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
      std::printf("spin %d warps %d variant %d (%s): %.1f cycles/step\n", spin, warps, v,
                  v == 0 ? "registers only" : v == 1 ? "+ smem operands" : v == 2 ? "+ global store" : v == 3 ? "+ strong b128 export" : v == 4 ? "+ syncwarp/prog/ring (no export)" : v == 5 ? "+ all" : v == 6 ? "smem operands + scattered store" : "+ scattered rhs gather (LDG) + scattered store", double(c) / steps);
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
