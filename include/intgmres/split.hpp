// intgmres/split.hpp -- drop-in for the reference's split.hpp: row scaling,
// the integer splitting (host setup) and the integer SpMV (GPU).
#pragma once

#include "intgmres/csr.hpp"
#include "intgmres/fxp.hpp"

#include <vector>

namespace intgmres {

struct RowScaled {
  CsrMatrixF a;
  std::vector<double> scale;
};

RowScaled row_scale(const CsrMatrixF& a, int alpha_a);
std::vector<double> scale_rhs(const std::vector<double>& b, const std::vector<double>& scale);

struct SplitMatrix {
  int n = 0;
  std::vector<CsrMatrixI> components;  // shared pattern
  std::vector<int> alphas;             // alphas[0] == 0
  int alpha_a = 0;
  std::vector<double> scale_diag;
  bool exact = false;
  int depth() const { return static_cast<int>(components.size()) - 1; }
};

SplitMatrix build_split(const CsrMatrixF& a, int alpha_a, int max_components,
                        std::vector<double> scale_diag = {});
FxVector spmv(const SplitMatrix& m, int s, const FxVector& v, FxTrace* t = nullptr);
std::vector<double> spmv_fp(const SplitMatrix& m, int s, const std::vector<double>& x);
CsrMatrixF reconstruct_fp(const SplitMatrix& m, int s);

}  // namespace intgmres
