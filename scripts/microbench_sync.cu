// Microbenchmarks for the ILU wavefront's communication primitives (dev tool).
//   1. cross-SM ping-pong over tagged 128-bit words (st/ld.relaxed.gpu.b128)
//   2. cost of an mbarrier arrive (release / relaxed), bar.sync and
//      fence.acq_rel.cta issued while the thread has K global loads in flight
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_sync.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ void st128(ulonglong2* p, u64 v, u64 t) {
  asm volatile("{ .reg .b128 q; mov.b128 q, {%0, %1}; st.global.relaxed.gpu.b128 [%2], q; }" ::"l"(v), "l"(t),
               "l"(p)
               : "memory");
}
__device__ __forceinline__ void ld128(const ulonglong2* p, u64& v, u64& t) {
  asm volatile("{ .reg .b128 q; ld.global.relaxed.gpu.b128 q, [%2]; mov.b128 {%0, %1}, q; }"
               : "=l"(v), "=l"(t)
               : "l"(p)
               : "memory");
}

// two CTAs bounce a counter: CTA 0 writes word[0] = i, CTA 1 waits for it and
// writes word[1] = i, CTA 0 waits ... ; cycles per round trip
__global__ void pingpong(ulonglong2* w, int iters, u64* out) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;
  u64 t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (me == 0) {
      st128(w + 0, i, ~(u64)i);
      u64 v, t;
      do ld128(w + 16, v, t); while (t != ~(u64)i || v != (u64)i);
    } else {
      u64 v, t;
      do ld128(w + 0, v, t); while (t != ~(u64)i || v != (u64)i);
      st128(w + 16, i, ~(u64)i);
    }
  }
  u64 t1 = clock64();
  if (me == 0) out[0] = (t1 - t0) / iters;
}

// plain load latency of a cold-ish strong b128 load (L2 hit), one lane
__global__ void ldlat(const ulonglong2* w, int iters, u64* out) {
  if (threadIdx.x != 0) return;
  u64 acc = 0;
  u64 t0 = clock64();
  int idx = 0;
  for (int i = 0; i < iters; ++i) {
    u64 v, t;
    ld128(w + (idx & 4095) * 8, v, t);
    idx += (int)(v & 1) + 97;  // dependent chain
    acc += t;
  }
  u64 t1 = clock64();
  out[0] = (t1 - t0) / iters;
  out[1] = acc;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// cost of a sync op while K independent global loads are in flight
template <int MODE>
__global__ void drain(const ulonglong2* w, int iters, int K, u64* out) {
  __shared__ alignas(8) unsigned long long bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1000000));
  __syncthreads();
  if (threadIdx.x != 0) return;
  u64 acc = 0, tot = 0;
  for (int i = 0; i < iters; ++i) {
    u64 v[8], t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < K) ld128(w + ((i * 8 + k) * 37 & 65535) * 8, v[k], t[k]);
    u64 t0 = clock64();
    if (MODE == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (MODE == 1) asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (MODE == 2) asm volatile("fence.acq_rel.cta;" ::: "memory");
    if (MODE == 3) asm volatile("bar.sync 1, 32;" ::: "memory");
    if (MODE == 4) {}
    u64 t1 = clock64();
    tot += t1 - t0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < K) acc += v[k] ^ t[k];
  }
  out[0] = tot / iters;
  out[1] = acc;
}

// throughput test: per iteration issue K loads whose results are consumed one
// iteration LATER, then do the sync op; if the op waits for loads in flight
// the iteration costs ~ one load latency
template <int MODE>
__global__ void overlap(const ulonglong2* w, int iters, u64* out) {
  __shared__ alignas(8) unsigned long long bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1000000));
  __syncthreads();
  if (threadIdx.x >= 32) return;
  u64 acc = 0;
  u64 pv[4] = {0, 0, 0, 0}, pt[4] = {0, 0, 0, 0};
  u64 t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    u64 v[4], t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) ld128(w + (((i * 4 + k) * 37 + threadIdx.x * 131) & 65535) * 8, v[k], t[k]);
    if (MODE == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (MODE == 1) asm volatile("fence.acq_rel.cta;" ::: "memory");
    if (MODE == 2) asm volatile("bar.sync 1, 32;" ::: "memory");
    if (MODE == 3) __syncwarp();
    if (MODE == 4) asm volatile("st.global.relaxed.gpu.b64 [%0], %1;" ::"l"(out + 8 + threadIdx.x), "l"(acc) : "memory");
    // consume the previous iteration's loads
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += pv[k] ^ pt[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pv[k] = v[k];
      pt[k] = t[k];
    }
    // ~200 cycles of independent ALU work
#pragma unroll 1
    for (int z = 0; z < 40; ++z) acc = acc * 3 + z;
  }
  u64 t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = acc;
  }
}

// cost of a CTA barrier right after this warp issued a global store
template <int MODE>
__global__ void store_then_bar(ulonglong2* w, int iters, u64* out) {
  u64 acc = 0;
  u64 t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    ulonglong2* p = w + ((i * 97 + threadIdx.x * 131) & 65535) * 8;
    if (MODE == 1) st128(p, acc, acc ^ 5);                                  // strong .gpu 128-bit
    if (MODE == 2) *reinterpret_cast<u64*>(p) = acc;                         // weak 64-bit
    if (MODE == 3) asm volatile("st.global.relaxed.gpu.b64 [%0], %1;" ::"l"(p), "l"(acc) : "memory");
    if (MODE == 4) asm volatile("st.global.wt.b64 [%0], %1;" ::"l"(p), "l"(acc) : "memory");
    asm volatile("bar.sync 1, 256;" ::: "memory");
    acc = acc * 3 + i;
  }
  u64 t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = acc;
  }
}

// weak-load consumer: CTA 0 publishes (value_i, tag_i = e ^ value_i) for a
// stream of rows, CTA 1 polls them with .cg loads and checks every accepted
// value against the expected one
__device__ __forceinline__ void ld128_cg(const ulonglong2* p, u64& v, u64& t) {
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(v), "=l"(t) : "l"(p) : "memory");
}
__global__ void weak_consumer(ulonglong2* w, int rows, u64 e, u64* out) {
  const int lane = threadIdx.x;
  if (blockIdx.x == 0) {
    for (int r = lane; r < rows; r += 32) {
      const u64 v = 0x1234567ull * (r + 1) + e;
      st128(w + r, v, e ^ v);
      for (int z = 0; z < 50; ++z) asm volatile("nanosleep.u32 20;");
    }
  } else {
    u64 bad = 0, polls = 0;
    for (int r = lane; r < rows; r += 32) {
      u64 v, t;
      do {
        ld128_cg(w + r, v, t);
        ++polls;
      } while (t != (e ^ v));
      if (v != 0x1234567ull * (r + 1) + e) ++bad;
    }
    atomicAdd(out, bad);
    atomicAdd(out + 1, polls);
  }
}

// wavefront-like iteration: 3 loads issued per thread, consumed two
// iterations later; some shared-memory work and a CTA barrier per iteration
template <int STRONG>
__global__ void pipelined_loads(const ulonglong2* w, int iters, u64* out) {
  __shared__ u64 sh[256];
  u64 V[2][3], T[2][3];
  u64 acc = threadIdx.x;
  auto issue = [&](int it, int b) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const ulonglong2* p = w + (((it * 3 + d) * 389 + threadIdx.x * 131 + blockIdx.x * 7919) & 65535) * 8;
      if (STRONG) ld128(p, V[b][d], T[b][d]);
      else asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(V[b][d]), "=l"(T[b][d]) : "l"(p) : "memory");
    }
  };
  issue(0, 0);
  issue(1, 1);
  u64 t0 = clock64();
  for (int it = 0; it < iters; it += 2) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      u64 s = 0;
#pragma unroll
      for (int d = 0; d < 3; ++d) s += V[b][d] ^ T[b][d];
      acc = acc * 3 + s;
      sh[threadIdx.x] = acc;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      acc += sh[(threadIdx.x + 1) & 255];
      issue(it + b + 2, b);
    }
  }
  u64 t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = acc;
  }
}

int main(int argc, char** argv) {
  ulonglong2* w;
  u64* out;
  cudaMalloc(&w, sizeof(ulonglong2) * 65536 * 8);
  cudaMemset(w, 0, sizeof(ulonglong2) * 65536 * 8);
  cudaMallocManaged(&out, 64);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(w, 0, 4096);
    pingpong<<<2, 32>>>(w, 2000, out);
    cudaDeviceSynchronize();
    printf("pingpong round trip: %llu cycles (%s)\n", out[0], cudaGetErrorString(cudaGetLastError()));
  }
  ldlat<<<1, 32>>>(w, 4000, out);
  cudaDeviceSynchronize();
  printf("dependent strong b128 load latency: %llu cycles\n", out[0]);
  const char* names[] = {"mbarrier.arrive (release)", "mbarrier.arrive.relaxed", "fence.acq_rel.cta", "bar.sync (1 warp)",
                         "nothing"};
  for (int K : {0, 1, 4, 8}) {
    u64 r[5];
    drain<0><<<1, 32>>>(w, 2000, K, out); cudaDeviceSynchronize(); r[0] = out[0];
    drain<1><<<1, 32>>>(w, 2000, K, out); cudaDeviceSynchronize(); r[1] = out[0];
    drain<2><<<1, 32>>>(w, 2000, K, out); cudaDeviceSynchronize(); r[2] = out[0];
    drain<3><<<1, 32>>>(w, 2000, K, out); cudaDeviceSynchronize(); r[3] = out[0];
    drain<4><<<1, 32>>>(w, 2000, K, out); cudaDeviceSynchronize(); r[4] = out[0];
    for (int m = 0; m < 5; ++m) printf("K=%d loads in flight: %-28s %llu cycles\n", K, names[m], r[m]);
  }
  const char* on[] = {"mbarrier.arrive", "fence.acq_rel.cta", "bar.sync", "__syncwarp", "st.relaxed.gpu", "none"};
  for (int m = 0; m < 6; ++m) {
    if (m == 0) overlap<0><<<1, 32>>>(w, 2000, out);
    if (m == 1) overlap<1><<<1, 32>>>(w, 2000, out);
    if (m == 2) overlap<2><<<1, 32>>>(w, 2000, out);
    if (m == 3) overlap<3><<<1, 32>>>(w, 2000, out);
    if (m == 4) overlap<4><<<1, 32>>>(w, 2000, out);
    if (m == 5) overlap<5><<<1, 32>>>(w, 2000, out);
    cudaDeviceSynchronize();
    printf("overlap: loads consumed next iteration, op=%-18s %llu cycles/iter\n", on[m], out[0]);
  }
  for (int rep = 0; rep < (argc > 1 && argv[1][0] == 'w' ? 3 : 0); ++rep) {  // "w": hangs on B200
    out[0] = out[1] = 0;
    weak_consumer<<<2, 32>>>(w, 4096, 0x9E3779B97F4A7C15ull * (rep + 1) | 1, out);
    cudaDeviceSynchronize();
    printf("weak .cg consumer rep %d: wrong accepted %llu, polls %llu (%s)\n", rep, out[0], out[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int grid : {1, 148}) {
    pipelined_loads<1><<<grid, 256>>>(w, 4000, out);
    cudaDeviceSynchronize();
    const u64 a = out[0];
    pipelined_loads<0><<<grid, 256>>>(w, 4000, out);
    cudaDeviceSynchronize();
    printf("pipelined loads (3/thread, used 2 iterations later) grid %d: strong %llu, weak %llu cycles/iter\n", grid,
           a, out[0]);
  }
  const char* sn[] = {"no store", "st.relaxed.gpu.b128", "weak st.b64", "st.relaxed.gpu.b64", "st.wt.b64"};
  for (int m = 0; m < 5; ++m) {
    if (m == 0) store_then_bar<0><<<1, 256>>>(w, 2000, out);
    if (m == 1) store_then_bar<1><<<1, 256>>>(w, 2000, out);
    if (m == 2) store_then_bar<2><<<1, 256>>>(w, 2000, out);
    if (m == 3) store_then_bar<3><<<1, 256>>>(w, 2000, out);
    if (m == 4) store_then_bar<4><<<1, 256>>>(w, 2000, out);
    cudaDeviceSynchronize();
    printf("store then bar.sync(256): %-22s %llu cycles/iter\n", sn[m], out[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
