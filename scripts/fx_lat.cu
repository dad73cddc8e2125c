// One-thread latency of the scalar fixed-point helpers (cycles per call on a
// dependent chain): isqrt_u64, make_udiv, sdiv_trunc, and a plain 64-bit '/'
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -Ipaper_2009_07495_b200/csrc scripts/fx_lat.cu -o scripts/fx_lat
#include <cstdio>
#include "fx_core.cuh"
using namespace igm;

__global__ void k_lat(u64 seed, u64* out, long long* cyc) {
  u64 x = seed | 1;
  long long t0 = clock64();
  for (int i = 0; i < 64; ++i) x = isqrt_u64(x * 0x9e3779b97f4a7c15ull) + x;
  long long t1 = clock64();
  for (int i = 0; i < 64; ++i) x += make_udiv((x >> 3) | 1).m;
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) x += static_cast<u64>(sdiv_trunc(static_cast<i64>(x), static_cast<i64>((x >> 17) | 3)));
  long long t3 = clock64();
  for (int i = 0; i < 64; ++i) x += static_cast<u64>(static_cast<i64>(x) / static_cast<i64>((x >> 17) | 3));
  long long t4 = clock64();
  double d = static_cast<double>(x);
  for (int i = 0; i < 64; ++i) d = __dmul_rn(d, 1.0000001) + 1.0;
  long long t5 = clock64();
  for (int i = 0; i < 64; ++i) x = static_cast<u64>(__ull2double_rn(x)) + 3;
  long long t6 = clock64();
  out[0] = x + static_cast<u64>(d);
  cyc[0] = (t1 - t0) / 64;
  cyc[1] = (t2 - t1) / 64;
  cyc[2] = (t3 - t2) / 64;
  cyc[3] = (t4 - t3) / 64;
  cyc[4] = (t5 - t4) / 64;
  cyc[5] = (t6 - t5) / 64;
}

int main() {
  u64* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 64);
  for (int r = 0; r < 2; ++r) k_lat<<<1, 1>>>(12345 + r, o, c);
  long long h[6];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("cycles/call: isqrt %lld  make_udiv %lld  sdiv_trunc %lld  i64 '/' %lld  dmul+add %lld  u64->f64->u64 %lld\n",
              h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
