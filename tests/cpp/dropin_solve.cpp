// A C++ program written against the reference's own API (intgmres::, the
// headers in include/intgmres/), linked against libigm_b200.so instead of the
// reference library: the drop-in boundary of SURVEY.md §8(b) exercised the way
// an existing user would.  It builds config 1's matrix (2D 5-point upwind
// convection-diffusion, the same formulas as workloads/gen.py:upwind_2d),
// b = A x* with an exact x*, and runs intgmres::solve unpreconditioned and
// with ILU(0), printing every output bit (hex floats) for
// tests/test_gpu_parity.py::test_cpp_dropin_solve to compare with the oracle.
//
//   g++ -std=c++20 -Iinclude tests/cpp/dropin_solve.cpp \
//       -Lpaper_2009_07495_b200 -ligm_b200 -Wl,-rpath,... -o dropin_solve
#include <intgmres/csr.hpp>
#include <intgmres/ilu.hpp>
#include <intgmres/refine.hpp>
#include <intgmres/split.hpp>

#include <cstdio>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

using namespace intgmres;

static void print_result(const char* tag, const SolveResult& r) {
  std::printf("%s refinements %d iters %ld overflows %llu converged %d\n", tag, r.report.refinements,
              r.report.total_inner_iterations, static_cast<unsigned long long>(r.report.overflow_total),
              r.report.converged ? 1 : 0);
  std::printf("%s relres", tag);
  for (double v : r.report.relres_history) std::printf(" %a", v);
  std::printf("\n%s x", tag);
  for (double v : r.x) std::printf(" %a", v);
  std::printf("\n");
}

// 5-point upwind operator with convection (b0, b1) on a g x g grid
static CsrMatrixF upwind(int g, double b0, double b1) {
  const double h = 1.0 / (g + 1);
  const double d = 4.0 / (h * h) + (b0 + b1) / h;
  std::vector<std::tuple<int, int, double>> t;
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      const int r = j * g + i;
      if (j > 0) t.emplace_back(r, r - g, -1.0 / (h * h) - b1 / h);
      if (i > 0) t.emplace_back(r, r - 1, -1.0 / (h * h) - b0 / h);
      t.emplace_back(r, r, d);
      if (i < g - 1) t.emplace_back(r, r + 1, -1.0 / (h * h));
      if (j < g - 1) t.emplace_back(r, r + g, -1.0 / (h * h));
    }
  return from_triplets(g * g, std::move(t));
}

static bool same(const SolveResult& a, const SolveResult& b) {
  return a.x == b.x && a.report.relres_history == b.report.relres_history &&
         a.report.inner_dims == b.report.inner_dims && a.report.gamma_history == b.report.gamma_history;
}

// The drop-in's verified operator cache: a repeated solve() on unchanged
// containers reuses the device upload (its content fingerprint is checked
// while the GPU solves); containers MUTATED IN PLACE -- same addresses and
// sizes, other values -- must be detected and solved afresh.
static int cache_check(int g) {
  struct Problem {
    RowScaled rs;
    SplitMatrix sp;
    IluFactors il;
    std::vector<double> b;
  };
  auto make = [&](double b0, double b1) {
    const CsrMatrixF a = upwind(g, b0, b1);
    std::vector<double> xs(a.n);
    for (int i = 0; i < a.n; ++i) xs[i] = (i % 7) * 0.25 - 0.75;
    Problem p;
    p.rs = row_scale(a, 32);
    p.b = scale_rhs(spmv_fp(a, xs), p.rs.scale);
    p.sp = build_split(p.rs.a, 32, 1);
    p.il = split_cast(factorize_ilu0(p.rs.a));
    return p;
  };
  RefineConfig cfg;
  cfg.tol = 1e-10;
  cfg.max_refinements = 60;
  cfg.m = 30;
  cfg.shifts = ShiftPlan::default_preconditioned(QFormat{30});
  Problem p = make(10.0, 10.0);
  const Problem q = make(3.0, 17.0);
  const SolveResult r1 = solve(p.sp, p.rs.a, p.b, cfg, &p.il);   // uploads
  const SolveResult r2 = solve(p.sp, p.rs.a, p.b, cfg, &p.il);   // cache hit, verified concurrently
  const SolveResult want = solve(q.sp, q.rs.a, q.b, cfg, &q.il);  // other containers: fresh upload
  (void)solve(p.sp, p.rs.a, p.b, cfg, &p.il);                      // p's upload is the cached one again
  const void* addr[3] = {p.sp.components[0].vals.data(), p.rs.a.vals.data(), p.il.lower.vals.data()};
  // q's values into p's containers, element by element: addresses and sizes stay
  std::copy(q.sp.components[0].vals.begin(), q.sp.components[0].vals.end(), p.sp.components[0].vals.begin());
  std::copy(q.rs.a.vals.begin(), q.rs.a.vals.end(), p.rs.a.vals.begin());
  std::copy(q.il.lower.vals.begin(), q.il.lower.vals.end(), p.il.lower.vals.begin());
  std::copy(q.il.upper.vals.begin(), q.il.upper.vals.end(), p.il.upper.vals.begin());
  const bool inplace = addr[0] == p.sp.components[0].vals.data() && addr[1] == p.rs.a.vals.data() &&
                       addr[2] == p.il.lower.vals.data();
  const SolveResult r3 = solve(p.sp, p.rs.a, q.b, cfg, &p.il);     // mutated in place
  std::printf("cache repeat_same %d inplace %d mutated_detected %d differs_from_first %d\n", same(r1, r2) ? 1 : 0,
              inplace ? 1 : 0, same(r3, want) ? 1 : 0, same(r3, r1) ? 0 : 1);
  return 0;
}

int main(int argc, char** argv) {
  const int g = argc > 1 ? std::atoi(argv[1]) : 32;
  if (argc > 2 && std::string(argv[2]) == "cache") {
    try {
      return cache_check(g);
    } catch (const std::exception& e) {
      std::printf("error %s\n", e.what());
      return 2;
    }
  }
  const double h = 1.0 / (g + 1), b0 = 10.0, b1 = 10.0;
  const double d = 4.0 / (h * h) + (b0 + b1) / h;
  const double south = -1.0 / (h * h) - b1 / h, west = -1.0 / (h * h) - b0 / h, east = -1.0 / (h * h),
               north = -1.0 / (h * h);
  const int n = g * g;
  std::vector<std::tuple<int, int, double>> t;
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      const int r = j * g + i;
      if (j > 0) t.emplace_back(r, r - g, south);
      if (i > 0) t.emplace_back(r, r - 1, west);
      t.emplace_back(r, r, d);
      if (i < g - 1) t.emplace_back(r, r + 1, east);
      if (j < g - 1) t.emplace_back(r, r + g, north);
    }
  const CsrMatrixF a = from_triplets(n, std::move(t));
  std::vector<double> xs(n);
  for (int i = 0; i < n; ++i) xs[i] = (i % 7) * 0.25 - 0.75;  // exact in binary
  const std::vector<double> bh = spmv_fp(a, xs);
  try {
    // unpreconditioned (config 1 settings)
    {
      const RowScaled rs = row_scale(a, 16);
      const std::vector<double> b = scale_rhs(bh, rs.scale);
      const SplitMatrix sp = build_split(rs.a, 16, 1);
      RefineConfig cfg;
      cfg.tol = 1e-10;
      cfg.max_refinements = 60;
      cfg.m = 30;
      cfg.shifts = ShiftPlan::default_unpreconditioned(QFormat{30});
      print_result("plain", solve(sp, rs.a, b, cfg));
    }
    // ILU(0)-preconditioned (config 2 settings on the same operator)
    {
      const RowScaled rs = row_scale(a, 32);
      const std::vector<double> b = scale_rhs(bh, rs.scale);
      const SplitMatrix sp = build_split(rs.a, 32, 1);
      const IluFactors il = split_cast(factorize_ilu0(rs.a));
      RefineConfig cfg;
      cfg.tol = 1e-10;
      cfg.max_refinements = 60;
      cfg.m = 30;
      cfg.shifts = ShiftPlan::default_preconditioned(QFormat{30});
      print_result("ilu", solve(sp, rs.a, b, cfg, &il));
    }
  } catch (const std::exception& e) {
    std::printf("error %s\n", e.what());
    return 2;
  }
  return 0;
}
