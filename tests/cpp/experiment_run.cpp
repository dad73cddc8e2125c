// run_experiment of the drop-in API (include/intgmres/experiment.hpp) on a
// Matrix Market file written here (config 1's matrix): prints each run's CSV
// and summary for tests/test_gpu_parity.py::test_cpp_experiment, which runs
// the reference library's run_experiment on the same file.
#include <intgmres/csr.hpp>
#include <intgmres/experiment.hpp>
#include <intgmres/mm_io.hpp>

#include <cstdio>
#include <cstdlib>
#include <tuple>
#include <vector>

using namespace intgmres;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const int g = argc > 2 ? std::atoi(argv[2]) : 24;
  const double h = 1.0 / (g + 1);
  const double d = 4.0 / (h * h) + 20.0 / h, lo = -1.0 / (h * h) - 10.0 / h, hi = -1.0 / (h * h);
  std::vector<std::tuple<int, int, double>> t;
  for (int j = 0; j < g; ++j)
    for (int i = 0; i < g; ++i) {
      const int r = j * g + i;
      if (j > 0) t.emplace_back(r, r - g, lo);
      if (i > 0) t.emplace_back(r, r - 1, lo);
      t.emplace_back(r, r, d);
      if (i < g - 1) t.emplace_back(r, r + 1, hi);
      if (j < g - 1) t.emplace_back(r, r + g, hi);
    }
  save_matrix_market(argv[1], from_triplets(g * g, std::move(t)));
  const int runs[3][2] = {{0, 0}, {0, 1}, {1, 1}};  // (solver, precond)
  for (const auto& rr : runs) {
    ExperimentSpec spec;
    spec.matrix_path = argv[1];
    spec.solver = rr[0] ? SolverKind::fp64 : SolverKind::integer;
    spec.precond = rr[1] ? PrecondKind::ilu0 : PrecondKind::none;
    spec.m = 20;
    spec.tol = 1e-10;
    spec.max_refinements = 60;
    const ExperimentResult r = run_experiment(spec);
    std::printf("### %d %d\n%s%s\n", rr[0], rr[1], r.csv.c_str(), r.summary.c_str());
  }
  return 0;
}
