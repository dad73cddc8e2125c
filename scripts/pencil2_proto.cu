// Standalone check + timing of the pencil wavefronts (csrc/tri_pencil.cuh and
// the warp-specialised / cluster-coupled csrc/tri_pencil2.cuh) on random
// 7-point lower/upper factors of a gx x gy x gz grid, against a sequential
// CPU substitution.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -Ipaper_2009_07495_b200/csrc scripts/pencil2_proto.cu -o scripts/pencil2_proto
//   (-DP2_GUARDS: spin guards that report instead of hanging; -DP2_STAGETS:
//   per-brick stage-entry times)
// Run: scripts/pencil2_proto gx gy gz [iters] [warmup] [cy]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tri_pencil2.cuh"

using namespace igm;

static u64 sm64(u64& s) {
  u64 z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

static int g_warm = 20;

template <int CY>
static void launch2(const PencilStream& PS, const PenArgs& a, const i64* y, i64* z, size_t sm) {
  if constexpr (CY == 1) {
    k_tri_pencil2<true, false, 1><<<PS.nbricks, kP2Threads, sm>>>(a, y, z, nullptr, nullptr, nullptr);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PS.nbricks);
    cfg.blockDim = dim3(kP2Threads);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CY;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_tri_pencil2<true, false, CY>, a, y, z, static_cast<const int*>(nullptr),
                          static_cast<const int*>(nullptr), static_cast<const double*>(nullptr)));
  }
}

// variant: 0 = k_tri_pencil (D = 4, R = 16), else k_tri_pencil2 with cluster size `variant`
template <int CY>
static float run(int variant, const PencilStream& PS, int n, bool upper, const std::vector<i64>& y,
                 std::vector<i64>& z, int iters) {
  void* d_rec;
  unsigned long long* d_stats;
  int *d_bot, *d_ticket;
  ulonglong2* d_xz;
  i64 *d_y, *d_z;
  CK(cudaMalloc(&d_rec, PS.blk.size() * 8));
  CK(cudaMalloc(&d_bot, PS.brick_of_ticket.size() * 4));
  CK(cudaMalloc(&d_ticket, 8));
  CK(cudaMemset(d_ticket, 0, 8));
  CK(cudaMalloc(&d_stats, 16));
  CK(cudaMalloc(&d_xz, static_cast<size_t>(n) * 16));
  CK(cudaMalloc(&d_y, static_cast<size_t>(n) * 8));
  CK(cudaMalloc(&d_z, static_cast<size_t>(n) * 8));
  CK(cudaMemcpy(d_rec, PS.blk.data(), PS.blk.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_bot, PS.brick_of_ticket.data(), PS.brick_of_ticket.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_y, y.data(), static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_xz, 0, static_cast<size_t>(n) * 16));
  const int R = 16;
  const size_t sm = variant ? kP2Smem : pencil_smem_bytes(R, 4);
  if (variant) {
    CK(cudaFuncSetAttribute(k_tri_pencil2<true, false, CY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(sm)));
    if (CY > 8)
      CK(cudaFuncSetAttribute(k_tri_pencil2<true, false, CY>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  } else {
    CK(cudaFuncSetAttribute(k_tri_pencil<4, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(sm)));
  }
  PenArgs a;
  a.gx = PS.gx;
  a.gy = PS.gy;
  a.gz = PS.gz;
  a.nbx = PS.nbx;
  a.nby = PS.nby;
  a.S = PS.S;
  a.R = R;
  a.pad = PS.pad;
  a.n = n;
  a.mirror = upper;
  a.rec = d_rec;
  a.brick_of_ticket = d_bot;
  a.xz = d_xz;
  a.ticket = d_ticket;
  a.stats = d_stats;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, tot = 0;
  for (int it = -g_warm; it < iters; ++it) {
    a.epoch = (0x1234567ull + it + 1000 * variant) * 0x9E3779B97F4A7C15ull | 1ull;
    CK(cudaMemset(d_z, 0x5a, static_cast<size_t>(n) * 8));
    cudaEventRecord(e0);
    if (variant) launch2<CY>(PS, a, d_y, d_z, sm);
    else k_tri_pencil<4, true, false><<<PS.nbricks, kPenThreads, sm>>>(a, d_y, d_z, nullptr, nullptr, nullptr);
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
#ifdef P2_GUARDS
  if (variant) {
    unsigned nrep = 0;
    CK(cudaMemcpyFromSymbol(&nrep, g_p2_nrep, 4));
    std::vector<unsigned long long> rep(8 * 4);
    CK(cudaMemcpyFromSymbol(rep.data(), g_p2_rep, rep.size() * 8));
    std::printf("  guard reports: %u\n", nrep);
    for (int q = 0; q < 8; ++q)
      if (rep[q * 4])
        std::printf("    first id %d: blk %llu tid %llu x %d y %d\n", q, rep[q * 4 + 1], rep[q * 4 + 2],
                    (int)(rep[q * 4 + 3] >> 32), (int)(rep[q * 4 + 3] & 0xffffffffu));
  }
#endif
#ifdef P2_STAGETS
  if (variant) {
    std::vector<unsigned long long> bt(64 * 64 * 16);
    CK(cudaMemcpyFromSymbol(bt.data(), g_p2_bt, bt.size() * 8));
    auto T = [&](int bx, int by, int w, int e) { return (long long)bt[(bx * 64 + by) * 16 + w * 2 + e]; };
    const long long t00 = T(0, 0, 0, 0);
    std::printf("    warp0 stage-2 entry (ns from brick 0,0) by row:\n");
    for (int by = 0; by < std::min(PS.nby, 4); ++by) {
      std::printf("     by=%d:", by);
      for (int bx = 0; bx < std::min(PS.nbx, 64); ++bx) std::printf(" %lld", T(bx, by, 0, 0) - t00);
      std::printf("\n");
    }
    std::printf("     bx=0 down y:");
    for (int by = 0; by < std::min(PS.nby, 64); ++by) std::printf(" %lld", T(0, by, 0, 0) - t00);
    std::printf("\n     brick (1,1) warp lags at stage 2: %lld %lld %lld ns; warp 0 stage 2->6: %lld ns\n",
                T(1, 1, 1, 0) - T(1, 1, 0, 0), T(1, 1, 2, 0) - T(1, 1, 0, 0), T(1, 1, 3, 0) - T(1, 1, 0, 0),
                T(1, 1, 0, 1) - T(1, 1, 0, 0));
  }
#endif
  z.resize(n);
  CK(cudaMemcpy(z.data(), d_z, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  std::printf("  %-14s: best %.1f us, mean %.1f us\n",
              variant == 0 ? "pencil" : (variant == 1 ? "pencil2 cy=1" : (variant == 8 ? "pencil2 cy=8" : "pencil2 cy=16")),
              best * 1e3, tot / iters * 1e3);
  cudaFree(d_rec);
  cudaFree(d_bot);
  cudaFree(d_ticket);
  cudaFree(d_stats);
  cudaFree(d_xz);
  cudaFree(d_y);
  cudaFree(d_z);
  return best;
}

int main(int argc, char** argv) {
  const int gx = argc > 1 ? std::atoi(argv[1]) : 128, gy = argc > 2 ? std::atoi(argv[2]) : gx,
            gz = argc > 3 ? std::atoi(argv[3]) : gx, iters = argc > 4 ? std::atoi(argv[4]) : 20;
  if (argc > 5) g_warm = std::atoi(argv[5]);
  const int cyv = argc > 6 ? std::atoi(argv[6]) : 8;
  const long long plane = static_cast<long long>(gx) * gy;
  const int n = static_cast<int>(plane * gz);
  u64 seed = 42;
  for (int upper = 0; upper < 2; ++upper) {
    std::vector<int> rp(n + 1, 0), ci, dpos(n);
    std::vector<i64> v;
    for (int r = 0; r < n; ++r) {
      const long long i = r % gx, j = (r / gx) % gy, k = r / plane;
      auto add = [&](long long c, i64 val) {
        ci.push_back(static_cast<int>(c));
        v.push_back(val);
      };
      auto off = [&]() { return static_cast<i64>(sm64(seed) % (1ull << 18)) - (1ll << 17); };
      auto dia = [&]() {
        i64 d = static_cast<i64>((1ull << 16) + sm64(seed) % (1ull << 16));
        return (sm64(seed) & 1) ? -d : d;
      };
      if (!upper) {
        if (k > 0) add(r - plane, off());
        if (j > 0) add(r - gx, off());
        if (i > 0) add(r - 1, off());
        dpos[r] = static_cast<int>(ci.size());
        add(r, dia());
      } else {
        dpos[r] = static_cast<int>(ci.size());
        add(r, dia());
        if (i < gx - 1) add(r + 1, off());
        if (j < gy - 1) add(r + gx, off());
        if (k < gz - 1) add(r + plane, off());
      }
      rp[r + 1] = static_cast<int>(ci.size());
    }
    std::vector<i64> y(n), zr(n, 0);
    for (auto& e : y) e = static_cast<i64>(sm64(seed)) >> (sm64(seed) % 40);
    // sequential reference (ilu.cpp:126-153): wrapping sum, truncating division
    for (int q = 0; q < n; ++q) {
      const int r = upper ? n - 1 - q : q;
      u64 acc = static_cast<u64>(y[r]);
      for (int p = rp[r]; p < rp[r + 1]; ++p)
        if (p != dpos[r]) acc -= static_cast<u64>(v[p]) * static_cast<u64>(zr[ci[p]]);
      zr[r] = sdiv(static_cast<i64>(acc), make_sdiv(v[dpos[r]]));
    }
    std::printf("%s %dx%dx%d: %d levels\n", upper ? "upper" : "lower", gx, gy, gz, gx + gy + gz - 2);
    for (int variant : {0, 1, cyv}) {
      if (variant > 1 && variant != 8 && variant != 16) continue;
      const int cy = variant > 1 ? variant : 1;
      PencilStream PS = build_pencil_stream(n, rp.data(), ci.data(), v.data(), dpos.data(), upper, gx, gy, gz, 16,
                                            false, cy);
      if (!PS.ok) {
        std::printf("stream build failed\n");
        return 1;
      }
      std::vector<i64> z;
      const float ms = variant == 8    ? run<8>(variant, PS, n, upper, y, z, iters)
                       : variant == 16 ? run<16>(variant, PS, n, upper, y, z, iters)
                                       : run<1>(variant, PS, n, upper, y, z, iters);
      long long bad = 0;
      for (int r = 0; r < n; ++r) bad += z[r] != zr[r];
      std::printf("    %d bricks, mismatches %lld / %d  (%.3f us/level)\n", PS.nbricks, bad, n,
                  ms * 1e3 / (gx + gy + gz - 2));
      std::fflush(stdout);
    }
  }
  return 0;
}
