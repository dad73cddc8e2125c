// The reference's FP64 comparator API (intgmres::fp_cycle / solve_fp,
// include/intgmres/refsolve.hpp) linked against libigm_b200.so: config 1's
// matrix, exact b; prints results (hex floats) for
// tests/test_gpu_parity.py::test_cpp_refsolve to compare with the reference.
#include <intgmres/csr.hpp>
#include <intgmres/ilu.hpp>
#include <intgmres/refsolve.hpp>

#include <cstdio>
#include <cstdlib>
#include <tuple>
#include <vector>

using namespace intgmres;

int main(int argc, char** argv) {
  const int g = argc > 1 ? std::atoi(argv[1]) : 24;
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
  std::vector<double> xs(n), x0(n);
  for (int i = 0; i < n; ++i) {
    xs[i] = (i % 7) * 0.25 - 0.75;
    x0[i] = (i % 5) * 0.125;
  }
  const std::vector<double> b = spmv_fp(a, xs);
  const FpIluFactors f = factorize_ilu0(a);
  for (int pre = 0; pre < 2; ++pre) {
    PrecondFn pf;
    if (pre) pf = [&f](const std::vector<double>& y) { return apply_fp(f, y); };
    const FpCycleResult c = fp_cycle(a, 20, b, x0, pf);
    std::printf("cycle%d dim %d r0 %a x", pre, c.dim, c.r0_norm);
    for (double v : c.x) std::printf(" %a", v);
    std::printf("\n");
    FpGmresConfig cfg;
    cfg.m = 20;
    cfg.tol = 1e-10;
    const FpSolveResult s = solve_fp(a, b, cfg, pre ? &f : nullptr);
    std::printf("solve%d restarts %d iters %ld conv %d x", pre, s.restarts, s.iterations, s.converged ? 1 : 0);
    for (double v : s.x) std::printf(" %a", v);
    std::printf("\n");
  }
  return 0;
}
