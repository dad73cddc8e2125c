// intgmres/ilu.hpp -- drop-in for the reference's ilu.hpp: ILU(0) setup on
// the host, integer and FP64 substitutions on the GPU (wavefront kernels).
#pragma once

#include "intgmres/csr.hpp"
#include "intgmres/fxp.hpp"

#include <vector>

namespace intgmres {

struct FpIluFactors {
  CsrMatrixF lower;          // unit lower, diagonal 1.0 stored
  std::vector<double> diag;  // D
  CsrMatrixF upper;          // unit upper, diagonal 1.0 stored
};

FpIluFactors factorize_ilu0(const CsrMatrixF& a);

struct IluFactors {
  CsrMatrixI lower;  // L * D_l
  CsrMatrixI upper;  // D_u * U
  std::vector<int> diag_pos_lower;
  std::vector<int> diag_pos_upper;
};

IluFactors split_cast(const FpIluFactors& f);
FxVector apply_inverse(const IluFactors& f, const FxVector& y, FxTrace* t = nullptr);
std::vector<double> apply_inverse_fp(const IluFactors& f, const std::vector<double>& y);
std::vector<double> apply_fp(const FpIluFactors& f, const std::vector<double>& y);

}  // namespace intgmres
