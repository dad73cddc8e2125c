// Standalone check + timing of the pencil wavefronts (csrc/tri_pencil.cuh, csrc/tri_pencil2.cuh) on
// random 7-point lower/upper factors of a gx x gy x gz grid, against a
// sequential CPU substitution.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -Ipaper_2009_07495_b200/csrc scripts/pencil2_proto.cu -o scripts/pencil2_proto
// Run: scripts/pencil_proto gx gy gz [iters]
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

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

static int g_warm = 50;
#ifdef P2_WATCH
#include <thread>
#include <chrono>
static volatile unsigned long long* g_watch_host = nullptr;
static void watch_setup() {
  void* h;
  CK(cudaHostAlloc(&h, 256 * 16 * 8, cudaHostAllocMapped));
  std::memset(h, 0, 256 * 16 * 8);
  g_watch_host = static_cast<volatile unsigned long long*>(h);
  void* d;
  CK(cudaHostGetDevicePointer(&d, h, 0));
  CK(cudaMemcpyToSymbol(g_p2_watch, &d, sizeof(d)));
}
static void watch_wait(cudaEvent_t ev) {
  for (int it = 0; it < 600; ++it) {
    if (cudaEventQuery(ev) == cudaSuccess) return;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  std::printf("HANG: watchdog snapshots\n");
  for (int b = 0; b < 256; ++b)
    if (g_watch_host[b * 16 + 15])
      std::printf("  blk %d ticket %llu brick (%llu,%llu) prog %lld %lld %lld %lld loader g %lld v %lld full/empty parity0-done bits %llx\n", b,
                  g_watch_host[b * 16], g_watch_host[b * 16 + 1], g_watch_host[b * 16 + 2], (long long)g_watch_host[b * 16 + 3],
                  (long long)g_watch_host[b * 16 + 4], (long long)g_watch_host[b * 16 + 5], (long long)g_watch_host[b * 16 + 6],
                  (long long)g_watch_host[b * 16 + 7], (long long)g_watch_host[b * 16 + 8], g_watch_host[b * 16 + 9]);
  std::fflush(stdout);
  std::_Exit(3);
}
#endif
template <int P, bool V2>
static float run(const PencilStream& PS, int n, bool upper, const std::vector<i64>& y, std::vector<i64>& z,
                 int iters, int R) {
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
  const size_t sm = V2 ? kP2Smem : pencil_smem_bytes(R, P);
  if (V2) CK(cudaFuncSetAttribute(k_tri_pencil2<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  else CK(cudaFuncSetAttribute(k_tri_pencil<P, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
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
  const int warm = g_warm;
  for (int it = -warm; it < iters + 2; ++it) {
    a.epoch = (0x1234567ull + it) * 0x9E3779B97F4A7C15ull | 1ull;

    CK(cudaMemset(d_z, 0x5a, static_cast<size_t>(n) * 8));
    cudaEventRecord(e0);
    if (V2) k_tri_pencil2<true, false><<<PS.nbricks, kP2Threads, sm>>>(a, d_y, d_z, nullptr, nullptr, nullptr);
    else k_tri_pencil<P, true, false><<<PS.nbricks, kPenThreads, sm>>>(a, d_y, d_z, nullptr, nullptr, nullptr);
    cudaEventRecord(e1);
#ifdef P2_WATCH
    if (V2) watch_wait(e1);
#endif
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2) {
      best = std::min(best, ms);
      tot += ms;
    }
  }
#ifdef PEN_TRACE
  {
    std::vector<unsigned long long> ts(kPenWarps * 4096);
    CK(cudaMemcpyFromSymbol(ts.data(), g_pen_ts, ts.size() * 8));
    for (int w = 0; w < kPenWarps; ++w) {
      const unsigned long long* q = &ts[w * 4096];
      const int S = PS.S;
      {
        std::vector<unsigned long long> cn(kPenWarps * 4);
        CK(cudaMemcpyFromSymbol(cn.data(), g_pen_cnt, cn.size() * 8));
        std::printf("    warp %d: stale lane-steps %llu, ring spins %llu (cumulative)\n", w, cn[w * 4], cn[w * 4 + 1]);
        std::vector<unsigned long long> ph(kPenWarps * 512 * 8);
        CK(cudaMemcpyFromSymbol(ph.data(), g_pen_ph, ph.size() * 8));
        double acc[6] = {0, 0, 0, 0, 0, 0};
        int cnt = 0;
        for (int s = 20; s < std::min(PS.S - 1, 100); ++s, ++cnt) {
          const unsigned long long* e = &ph[(w * 512 + s) * 8];
          const unsigned long long nx = ph[(w * 512 + s + 1) * 8];
          for (int q = 0; q < 5; ++q) acc[q] += double(e[q + 1] - e[q]);
          acc[5] += double(nx - e[5]);
        }
        std::printf("    warp %d phases (cyc): ring+pre %.0f | wait %.0f | lds+stale %.0f | math %.0f | bp %.0f | tail+issue %.0f\n", w,
                    acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt);
      }
      std::printf("    warp %d: start +%lld cyc, steps 1-16 %.0f cyc/step, 16-%d %.0f cyc/step\n", w,
                  (long long)(q[0] - ts[0]), (q[16] - q[1]) / 15.0, S - 1, (q[S - 1] - q[16]) / double(S - 17));
    }
  }
#endif
#ifdef P2_GUARDS
  if (V2) {
    unsigned nrep = 0;
    CK(cudaMemcpyFromSymbol(&nrep, g_p2_nrep, 4));
    std::vector<unsigned long long> rep(64 * 4);
    CK(cudaMemcpyFromSymbol(rep.data(), g_p2_rep, rep.size() * 8));
    std::printf("  guard reports: %u\n", nrep);
    std::vector<unsigned long long> sn(256 * 16);
    CK(cudaMemcpyFromSymbol(sn.data(), g_p2_blk, sn.size() * 8));
    int shown = 0;
    for (int b = 0; b < 256 && shown < 40; ++b)
      if (sn[b * 16 + 15]) {
        ++shown;
        std::printf("    blk %d: ticket %llu brick (%llu,%llu) prog %lld %lld %lld %lld | ximp k:", b, sn[b * 16], sn[b * 16 + 1], sn[b * 16 + 2],
                    (long long)sn[b * 16 + 3], (long long)sn[b * 16 + 4], (long long)sn[b * 16 + 5], (long long)sn[b * 16 + 6]);
        for (int q = 0; q < 8; ++q) std::printf(" %lld", (long long)(int)sn[b * 16 + 7 + q]);
        std::printf("\n");
      }
    std::vector<unsigned> idc(8);
    CK(cudaMemcpyFromSymbol(idc.data(), g_p2_idc, 32));
    for (int q = 0; q < 8; ++q) if (idc[q]) std::printf("    id %d: %u reports\n", q, idc[q]);
    for (unsigned q = 0; q < 8; ++q)
      if (idc[q])
      std::printf("    blk %llu tid %llu id %llu x %lld y %lld\n", rep[q * 4], rep[q * 4 + 1], rep[q * 4 + 2],
                  (long long)(int)(rep[q * 4 + 3] >> 32), (long long)(int)(rep[q * 4 + 3] & 0xffffffffu));
  }
#endif
#ifdef P2_DBG
  if (V2) {
    std::vector<unsigned long long> ts(8 * 4096);
    CK(cudaMemcpyFromSymbol(ts.data(), g_p2_ts, ts.size() * 8));
    const unsigned long long t0 = ts[0];
    for (int w = 0; w < kPenWarps; ++w) {
      const unsigned long long* q = &ts[w * 4096];
      const int S = PS.S;
      std::printf("    warp %d: start +%lld, mean %.0f cyc/step over 8..S-8; steps:", w, (long long)(q[0] - t0),
                  double(q[S - 8] - q[8]) / (S - 16));
      for (int s2 = 0; s2 < std::min(S, 40); s2 += 4) std::printf(" %lld", (long long)(q[s2] - t0));
      std::printf("\n");
    }
    for (int w = 0; w < kPenWarps; ++w) {
      std::printf("    warp %d phases cyc/step: stage %.0f | lds+shfl+wait %.0f | math %.0f | bp %.0f | stores %.0f | loop %.0f\n", w,
                  ts[7 * 4096 + w * 8] / double(PS.S), ts[7 * 4096 + w * 8 + 1] / double(PS.S), ts[7 * 4096 + w * 8 + 2] / double(PS.S),
                  ts[7 * 4096 + w * 8 + 3] / double(PS.S), ts[7 * 4096 + w * 8 + 4] / double(PS.S), ts[7 * 4096 + w * 8 + 5] / double(PS.S));
    }
    std::printf("    loader issue (g, v=0):");
    for (int g = 0; g < std::min((PS.S + 7) / 8, 12); ++g) std::printf(" %lld", (long long)(ts[4 * 4096 + g * 4] - t0));
    std::printf("\n    importer y lane0 deliver k:");
    for (int k2 = 0; k2 < 40; k2 += 4) std::printf(" %lld", (long long)(ts[5 * 4096 + k2] - t0));
    std::printf("\n    importer x lane16 deliver k:");
    for (int k2 = 0; k2 < 40; k2 += 4) std::printf(" %lld", (long long)(ts[6 * 4096 + k2] - t0));
    std::printf("\n");
  }
#endif
#ifdef P2_STAGETS
  if (V2) {
    std::vector<long long> st(8 * 1024);
    CK(cudaMemcpyFromSymbol(st.data(), g_p2_sts, st.size() * 8));
    const int nst = (PS.S + 7) / 8;
    for (int w = 0; w < kPenWarps; ++w) {
      std::printf("    warp %d stage starts (cyc from warp0 stage0):", w);
      for (int g = 0; g < nst; g += 2) std::printf(" %lld", st[w * 1024 + g] - st[0]);
      long long wt = 0;
      for (int g = 1; g < nst; ++g) wt += st[w * 1024 + g] - st[4096 + w * 1024 + g];
      std::printf("  | stage+bp wait total %lld cyc\n", wt);
    }
    std::vector<unsigned long long> bt(64 * 64 * 16);
    CK(cudaMemcpyFromSymbol(bt.data(), g_p2_bt, bt.size() * 8));
    auto T = [&](int bx, int by, int w, int e) { return (long long)bt[(bx * 64 + by) * 16 + w * 2 + e]; };
    const long long t00 = T(0, 0, 0, 0);
    std::printf("    brick warp0 stage-2 entry (ns from brick 0,0), x along row by=0..3 / y along column bx=0:\n");
    for (int by = 0; by < std::min(PS.nby, 4); ++by) {
      std::printf("     by=%d:", by);
      for (int bx = 0; bx < PS.nbx; ++bx) std::printf(" %lld", T(bx, by, 0, 0) - t00);
      std::printf("\n");
    }
    std::printf("     bx=0 down y:");
    for (int by = 0; by < PS.nby; ++by) std::printf(" %lld", T(0, by, 0, 0) - t00);
    std::printf("\n     warp lag within brick (1,1) w0..3 at stage 2: %lld %lld %lld %lld ns; stage 2->6 of warp0: %lld ns\n",
                T(1, 1, 0, 0) - T(1, 1, 0, 0), T(1, 1, 1, 0) - T(1, 1, 0, 0), T(1, 1, 2, 0) - T(1, 1, 0, 0),
                T(1, 1, 3, 0) - T(1, 1, 0, 0), T(1, 1, 0, 1) - T(1, 1, 0, 0));
  }
#endif
  z.resize(n);
  CK(cudaMemcpy(z.data(), d_z, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  std::fflush(stdout);
  std::printf("  %s: best %.1f us, mean %.1f us\n", V2 ? "pencil2" : "pencil ", best * 1e3, tot / iters * 1e3);
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
#ifdef P2_WATCH
  watch_setup();
#endif
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
    PencilStream PS = build_pencil_stream(n, rp.data(), ci.data(), v.data(), dpos.data(), upper, gx, gy, gz);
    if (!PS.ok) {
      std::printf("stream build failed\n");
      return 1;
    }
    std::printf("%s %dx%dx%d: %d bricks, %d steps/warp, stream %.1f MB, %d levels\n", upper ? "upper" : "lower", gx,
                gy, gz, PS.nbricks, PS.S, PS.blk.size() * 8 / 1e6, gx + gy + gz - 2);
    std::vector<i64> z;
    for (int R : {16}) {
      for (int Pv : {0, 1}) {
        const float ms = Pv == 0 ? run<4, false>(PS, n, upper, y, z, iters, R) : run<4, true>(PS, n, upper, y, z, iters, R);
        long long bad = 0;
        for (int r = 0; r < n; ++r) bad += z[r] != zr[r];
        std::printf("    mismatches %lld / %d  (%.3f us/level)\n", bad, n, ms * 1e3 / (gx + gy + gz - 2));
      }
    }
  }
  return 0;
}
