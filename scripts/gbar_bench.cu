// Microbenchmark: latency of one MGS pass's grid-wide reduction + barrier in
// a persistent 148-CTA kernel (k_arnoldi2's handshake), two protocols:
//   0: atomics into one accumulator, red.release counter, ld.acquire spin,
//      then a fetch of the accumulator (the round-2 k_arnoldi2 handshake)
//   1: all-gather of tagged words: each CTA stores its partial(s) as
//      (value, tag) 128-bit words into slot[pass & 1][cta]; threads t < G of
//      every CTA poll slot t until its tag matches and the CTA sums the G
//      words (wrapping u64 adds: any order) -- no fences, no atomics, one
//      L2 round trip
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/gbar_bench.cu -o scripts/gbar_bench
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef unsigned long long u64;

struct Ctl {
  unsigned gbar;
  u64 acc[3 * 512];
};

constexpr int T = 512;

__device__ __forceinline__ void st_word(ulonglong2* p, u64 v, u64 tag) {
  asm volatile("{ .reg .b128 t; mov.b128 t, {%0, %1}; st.relaxed.gpu.global.b128 [%2], t; }" ::"l"(v), "l"(tag),
               "l"(p)
               : "memory");
}
__device__ __forceinline__ void ld_word(const ulonglong2* p, u64& v, u64& tag) {
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(v), "=l"(tag)
               : "l"(p)
               : "memory");
}

template <int NW>
__device__ __forceinline__ void cta_sum(u64 (&s)[NW], u64 (*red)[32]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < NW; ++k) s[k] += __shfl_down_sync(0xffffffffu, s[k], o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NW; ++k) red[k][wid] = s[k];
  __syncthreads();
}

template <int MODE, int NW>
__global__ void __launch_bounds__(T, 1) k_bench(Ctl* ctl, ulonglong2* slots, int passes, u64 epoch, u64* out,
                                                long long* cyc, int work) {
  __shared__ u64 red[NW][32];
  __shared__ u64 s_tot[NW];
  const unsigned G = gridDim.x;
  u64 x = threadIdx.x + 1000 * blockIdx.x, chk = 0;
  long long t0 = clock64();
  for (int p = 0; p < passes; ++p) {
    // a little per-thread work (stands for the pass's rows)
    for (int r = 0; r < work; ++r) x = x * 6364136223846793005ull + 1442695040888963407ull;
    u64 s[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) s[k] = x + k;
    cta_sum<NW>(s, red);
    if (MODE == 0) {
      if (threadIdx.x == 0) {
        u64 a[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          a[k] = 0;
          for (int i = 0; i < T / 32; ++i) a[k] += red[k][i];
          atomicAdd(&ctl->acc[NW * p + k], a[k]);
        }
        unsigned* c = &ctl->gbar;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
        const unsigned target = (p + 1) * G;
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        } while (v < target);
#pragma unroll
        for (int k = 0; k < NW; ++k) s_tot[k] = *reinterpret_cast<volatile u64*>(&ctl->acc[NW * p + k]);
      }
      __syncthreads();
    } else {
      ulonglong2* base = slots + static_cast<size_t>(p & 1) * G * NW;
      const u64 tag = epoch + p;
      if (threadIdx.x < NW) {
        const int k = threadIdx.x;
        u64 a = 0;
        for (int i = 0; i < T / 32; ++i) a += red[k][i];
        st_word(base + blockIdx.x * NW + k, a, tag);
      }
      // threads t < G*NW poll word t
      u64 v[NW];
#pragma unroll
      for (int k = 0; k < NW; ++k) v[k] = 0;
      if (threadIdx.x < G) {
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          u64 tg;
          do {
            ld_word(base + threadIdx.x * NW + k, v[k], tg);
          } while (tg != tag);
        }
      }
      __syncthreads();  // red[] reads above are done before it is reused
      cta_sum<NW>(v, red);
      if (threadIdx.x < NW) {
        u64 a = 0;
        for (int i = 0; i < T / 32; ++i) a += red[threadIdx.x][i];
        s_tot[threadIdx.x] = a;
      }
      __syncthreads();
    }
    chk += s_tot[0];
    x ^= s_tot[NW - 1];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[blockIdx.x] = chk;
    cyc[blockIdx.x] = t1 - t0;
  }
}

template <int MODE, int NW>
static void run(int G, int passes, int work, const char* name) {
  Ctl* ctl;
  ulonglong2* slots;
  u64* out;
  long long* cyc;
  cudaMalloc(&ctl, sizeof(Ctl));
  cudaMalloc(&slots, 2 * G * NW * sizeof(ulonglong2));
  cudaMalloc(&out, G * sizeof(u64));
  cudaMalloc(&cyc, G * sizeof(long long));
  cudaMemset(slots, 0, 2 * G * NW * sizeof(ulonglong2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  std::vector<u64> h0(G);
  for (int rep = 0; rep < 6; ++rep) {
    cudaMemset(ctl, 0, sizeof(Ctl));
    const u64 epoch = (static_cast<u64>(rep) + 1) << 32;
    void* args[] = {&ctl, &slots, &passes, (void*)&epoch, &out, &cyc, &work};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((const void*)k_bench<MODE, NW>, dim3(G), dim3(T), args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
    cudaMemcpy(h0.data(), out, G * sizeof(u64), cudaMemcpyDeviceToHost);
  }
  cudaError_t e = cudaGetLastError();
  bool same = true;
  for (int i = 1; i < G; ++i) same = same && h0[i] == h0[0];
  std::printf("%-28s words=%d work=%d: %.3f us/pass  (agree=%d, %s)\n", name, NW, work, 1e3 * best / passes, same,
              cudaGetErrorString(e));
  cudaFree(ctl);
  cudaFree(slots);
  cudaFree(out);
  cudaFree(cyc);
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int passes = 400;
  for (int work : {0, 200}) {
    run<0, 1>(sms, passes, work, "atomic+counter");
    run<1, 1>(sms, passes, work, "tagged all-gather");
    run<0, 3>(sms, passes, work, "atomic+counter");
    run<1, 3>(sms, passes, work, "tagged all-gather");
  }
  return 0;
}
