// Standalone check + timing of the 27-point pencil wavefront
// (csrc/pencil27.cuh) on random 27-point lower/upper factors against a
// sequential CPU substitution.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -Ipaper_2009_07495_b200/csrc scripts/pencil27_proto.cu -o scripts/pencil27_proto
// Run: scripts/pencil27_proto gx gy gz [iters]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pencil27.cuh"

using namespace igm;

static u64 sm64(u64& s) {
  u64 z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);       \
      std::exit(1);                                                                         \
    }                                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const int gx = argc > 1 ? std::atoi(argv[1]) : 64, gy = argc > 2 ? std::atoi(argv[2]) : gx,
            gz = argc > 3 ? std::atoi(argv[3]) : gx, iters = argc > 4 ? std::atoi(argv[4]) : 10;
  const long long plane = static_cast<long long>(gx) * gy;
  const int n = static_cast<int>(plane * gz);
  u64 seed = 7;
  for (int upper = 0; upper < 2; ++upper) {
    std::vector<int> rp(n + 1, 0), ci, dpos(n);
    std::vector<i64> v;
    ci.reserve(static_cast<size_t>(n) * 14);
    v.reserve(static_cast<size_t>(n) * 14);
    for (int r = 0; r < n; ++r) {
      const long long i = r % gx, j = (r / gx) % gy, k = r / plane;
      auto off = [&]() { return static_cast<i64>(sm64(seed) % (1ull << 18)) - (1ll << 17); };
      // natural-order columns ascending: dk, dj, di from -1..1
      for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            const long long ii = i + di, jj = j + dj, kk = k + dk;
            if (ii < 0 || ii >= gx || jj < 0 || jj >= gy || kk < 0 || kk >= gz) continue;
            const long long c = kk * plane + jj * gx + ii;
            if (c == r) {
              dpos[r] = static_cast<int>(ci.size());
              i64 d = static_cast<i64>((1ull << 16) + sm64(seed) % (1ull << 16));
              ci.push_back(r);
              v.push_back((sm64(seed) & 1) ? -d : d);
            } else if (upper ? c > r : c < r) {
              ci.push_back(static_cast<int>(c));
              v.push_back(off());
            }
          }
      rp[r + 1] = static_cast<int>(ci.size());
    }
    std::vector<i64> y(n), zr(n, 0);
    for (auto& e : y) e = static_cast<i64>(sm64(seed)) >> (sm64(seed) % 40);
    for (int q = 0; q < n; ++q) {
      const int r = upper ? n - 1 - q : q;
      u64 acc = static_cast<u64>(y[r]);
      for (int p = rp[r]; p < rp[r + 1]; ++p)
        if (p != dpos[r]) acc -= static_cast<u64>(v[p]) * static_cast<u64>(zr[ci[p]]);
      zr[r] = sdiv(static_cast<i64>(acc), make_sdiv(v[dpos[r]]));
    }
    Pencil27Stream PS = build_pencil27_stream(n, rp.data(), ci.data(), v.data(), dpos.data(), upper, gx, gy, gz);
    if (!PS.ok) {
      std::printf("stream build failed\n");
      return 1;
    }
    const size_t sm = pencil27_smem_bytes();
    CK(cudaFuncSetAttribute(k_tri27<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    int per = 0, nsm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tri27<true>, kP27Threads, sm));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    std::printf("%s %dx%dx%d: %d bricks, resident %d x %d, stream %.1f MB, levels %d\n", upper ? "upper" : "lower", gx,
                gy, gz, PS.nbricks, per, nsm, PS.rec.size() / 1e6, (gx - 1) + 2 * (gy - 1) + 4 * (gz - 1) + 1);
    if (per * nsm < PS.nbricks) {
      std::printf("not co-resident\n");
      continue;
    }
    unsigned char* d_rec;
    ulonglong2* d_xz;
    i64 *d_y, *d_z;
    unsigned long long* d_st;
    CK(cudaMalloc(&d_rec, PS.rec.size()));
    CK(cudaMalloc(&d_xz, static_cast<size_t>(n) * 16));
    CK(cudaMalloc(&d_y, static_cast<size_t>(n) * 8));
    CK(cudaMalloc(&d_z, static_cast<size_t>(n) * 8));
    CK(cudaMalloc(&d_st, 16));
    CK(cudaMemcpy(d_rec, PS.rec.data(), PS.rec.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_y, y.data(), static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_xz, 0, static_cast<size_t>(n) * 16));
    P27Args a;
    a.gx = gx;
    a.gy = gy;
    a.gz = gz;
    a.nbx = PS.nbx;
    a.n = n;
    a.mirror = upper;
    a.rec = d_rec;
    a.xz = d_xz;
    a.stats = d_st;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f, tot = 0;
    for (int it = -3; it < iters; ++it) {
      a.epoch = (0x51ull + it) * 0x9E3779B97F4A7C15ull | 1ull;
      CK(cudaMemset(d_z, 0x5a, static_cast<size_t>(n) * 8));
      cudaEventRecord(e0);
      k_tri27<true><<<PS.nbricks, kP27Threads, sm>>>(a, d_y, d_z, nullptr, nullptr);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 0) {
        best = std::min(best, ms);
        tot += ms;
      }
    }
    std::vector<i64> z(n);
    CK(cudaMemcpy(z.data(), d_z, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int r = 0; r < n; ++r) bad += z[r] != zr[r];
    const int lev = (gx - 1) + 2 * (gy - 1) + 4 * (gz - 1) + 1;
    std::printf("  best %.1f us, mean %.1f us, %.3f us/level, mismatches %lld / %d\n", best * 1e3, tot / iters * 1e3,
                best * 1e3 / lev, bad, n);
    cudaFree(d_rec);
    cudaFree(d_xz);
    cudaFree(d_y);
    cudaFree(d_z);
    cudaFree(d_st);
  }
  return 0;
}
