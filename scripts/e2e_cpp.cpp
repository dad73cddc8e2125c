// e2e_cpp -- the drop-in boundary timed the way a reference user calls it:
// a C++ program written against the reference's API (include/intgmres/),
// linked against libigm_b200.so, that runs intgmres::solve (refine.hpp:67-70)
// on config 2 with host std::vector containers in and out.  bench.py writes
// the config-2 inputs (workloads/gen.py) as raw files and parses this
// program's JSON line.  Host setup (row_scale, build_split, factorize_ilu0,
// split_cast) uses the drop-in API too and is not timed; every timed call
// uploads b, downloads x and reuses the operators through the verified
// operator cache (shim.cpp: same arrays, same content fingerprint).
//
//   e2e_cpp <dir with rp.bin ci.bin v.bin bh.bin> <steps> <warmup> <x_out.bin>
#include <intgmres/csr.hpp>
#include <intgmres/ilu.hpp>
#include <intgmres/refine.hpp>
#include <intgmres/split.hpp>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

using namespace intgmres;

template <class T>
static std::vector<T> read_all(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("cannot open " + path);
  const std::streamsize bytes = f.tellg();
  f.seekg(0);
  std::vector<T> v(static_cast<std::size_t>(bytes) / sizeof(T));
  f.read(reinterpret_cast<char*>(v.data()), bytes);
  return v;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: e2e_cpp dir steps warmup x_out\n");
    return 2;
  }
  const std::string dir = argv[1];
  const int steps = std::atoi(argv[2]), warmup = std::atoi(argv[3]);
  try {
    CsrMatrixF a;
    a.row_ptr = read_all<int>(dir + "/rp.bin");
    a.col_idx = read_all<int>(dir + "/ci.bin");
    a.vals = read_all<double>(dir + "/v.bin");
    a.n = static_cast<int>(a.row_ptr.size()) - 1;
    const std::vector<double> bh = read_all<double>(dir + "/bh.bin");
    const auto s0 = std::chrono::steady_clock::now();
    const RowScaled rs = row_scale(a, 32);
    const std::vector<double> b = scale_rhs(bh, rs.scale);
    const SplitMatrix sp = build_split(rs.a, 32, 1);
    const IluFactors il = split_cast(factorize_ilu0(rs.a));
    const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
    RefineConfig cfg;
    cfg.tol = 1e-10;
    cfg.max_refinements = 1000;
    cfg.m = 30;
    cfg.shifts = ShiftPlan::default_preconditioned(QFormat{30});
    cfg.s = sp.depth();
    SolveResult r;
    double first = 0;
    for (int i = 0; i < warmup; ++i) {
      const auto t = std::chrono::steady_clock::now();
      r = solve(sp, rs.a, b, cfg, &il);
      if (i == 0) first = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
    }
    long iters = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) {
      r = solve(sp, rs.a, b, cfg, &il);
      iters += r.report.total_inner_iterations;
    }
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::ofstream xo(argv[4], std::ios::binary);
    xo.write(reinterpret_cast<const char*>(r.x.data()), static_cast<std::streamsize>(r.x.size() * sizeof(double)));
    std::printf(
        "{\"iters_per_s\": %.3f, \"ms_per_solve\": %.4f, \"iterations\": %ld, \"steps\": %d, \"warmup\": %d, "
        "\"first_call_s\": %.4f, \"host_setup_s\": %.3f, \"converged\": %d, \"final_relres\": %.6e, "
        "\"refinements\": %d}\n",
        iters / dt, 1e3 * dt / steps, iters, steps, warmup, first, setup_s, r.report.converged ? 1 : 0,
        r.report.relres_history.back(), r.report.refinements);
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
