// setup.cu -- device-side setup: the reference's
// row_scale (split.cpp:61-79), build_split (split.cpp:90-135) and
// factorize_ilu0 + split_cast (ilu.cpp:25-120) on the GPU, bit-identical to
// the host code.
//
// Every floating-point result is a per-row (or per-entry) sequence of
// correctly rounded IEEE operations in the reference's order -- explicit
// __ddiv_rn / __dmul_rn / __dsub_rn / __dsqrt_rn, the library is compiled
// -fmad=false -- so the only parallelism is ACROSS rows / entries:
//   * row_scale, build_split, split_cast: independent per row / entry;
//   * factorize_ilu0: row i reads the finished rows j < i of its lower
//     pattern, i.e. the same DAG as the forward substitution.  Rows are
//     processed one DAG level per launch, one thread per row (the host orders
//     the rows by level: index work only).  Inside a row the updates run in
//     the reference's order: for each lower entry k (ascending j) the
//     multiplier lu[k] /= lu[diag j], then for each upper entry kk of row j
//     (ascending column) lu[pos] -= lu[k] * lu[kk] where pos is row i's entry
//     of that column (the reference's iw[] lookup, here a merge walk over the
//     two ascending column lists; the last duplicate wins as with iw[]).
// Errors are reported as the smallest offending row (the first one the
// sequential reference would meet): atomicMin on an int.
#include "igm_internal.cuh"

#include <climits>

namespace igm {
namespace {

__device__ __forceinline__ u64 abs_bits(double v) {
  return static_cast<u64>(__double_as_longlong(fabs(v)));
}

// max over non-NaN |v| (std::max(acc, |v|) from 0.0 never takes a NaN);
// non-negative doubles order as their bit patterns
__device__ __forceinline__ void max_bits_reduce(u64 mx, u64* out) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 t = __shfl_down_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(reinterpret_cast<unsigned long long*>(out), mx);
}

__device__ __forceinline__ u64 nan_free(u64 bits) {
  return bits > 0x7ff0000000000000ull ? 0 : bits;
}

// row_scale (split.cpp:61-79): d_i = ldexp(max_k |a_ik|, -alpha); a_ik / d_i
__global__ void __launch_bounds__(256) k_row_scale(int n, const int* __restrict__ rp,
                                                   const double* __restrict__ v, int alpha,
                                                   double* __restrict__ out, double* __restrict__ scale,
                                                   int* err_row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = rp[i], b = rp[i + 1];
  double mx = 0.0;
  for (int k = a; k < b; ++k) {
    const double t = fabs(v[k]);
    mx = mx < t ? t : mx;
  }
  if (mx == 0.0) {
    atomicMin(err_row, i);
    return;
  }
  const double d = ldexp(mx, -alpha);
  scale[i] = d;
  for (int k = a; k < b; ++k) out[k] = __ddiv_rn(v[k], d);
}

// build_split layer 0 (split.cpp:105-112): trunc, exact remainder, max|rem|
__global__ void k_split_first(long long nnz, const double* __restrict__ v, i64* __restrict__ comp,
                              double* __restrict__ rem, u64* mx_out) {
  u64 mx = 0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const i64 c = __double2ll_rz(v[k]);
    comp[k] = c;
    const double r = __dsub_rn(v[k], __ll2double_rn(c));
    rem[k] = r;
    const u64 bb = nan_free(abs_bits(r));
    mx = bb > mx ? bb : mx;
  }
  max_bits_reduce(mx, mx_out);
}

// a later layer (split.cpp:121-130): c = trunc(ldexp(rem, alpha)),
// rem -= ldexp(c, -alpha), max|rem|
__global__ void k_split_next(long long nnz, double* __restrict__ rem, int alpha, i64* __restrict__ comp,
                             u64* mx_out) {
  u64 mx = 0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double r0 = rem[k];
    const i64 c = __double2ll_rz(ldexp(r0, alpha));
    comp[k] = c;
    const double r = __dsub_rn(r0, ldexp(__ll2double_rn(c), -alpha));
    rem[k] = r;
    const u64 bb = nan_free(abs_bits(r));
    mx = bb > mx ? bb : mx;
  }
  max_bits_reduce(mx, mx_out);
}

// diag_positions (ilu.cpp:11-22) + the row sizes of the split factors
// (ilu.cpp:57-77: j <= i -> lower, j >= i -> upper)
__global__ void __launch_bounds__(256) k_ilu_pattern(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                     int* __restrict__ diag, int* __restrict__ lcnt,
                                                     int* __restrict__ ucnt, int* err_row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = -1, nl = 0, nu = 0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int c = ci[k];
    if (c == i) p = k;
    nl += c <= i;
    nu += c >= i;
  }
  diag[i] = p;
  lcnt[i] = nl;
  ucnt[i] = nu;
  if (p < 0) atomicMin(err_row, i);
}

// factorize_ilu0 (ilu.cpp:25-52) for the rows of one DAG level
__global__ void __launch_bounds__(128) k_ilu_rows(int cnt, const int* __restrict__ rows, const int* __restrict__ rp,
                                                  const int* __restrict__ ci, const int* __restrict__ diag,
                                                  double* lu, int* err_row) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int i = rows[t];
  const int e = rp[i + 1];
  for (int k = rp[i]; k < e; ++k) {
    const int j = ci[k];
    if (j >= i) break;  // columns ascend: lower part done
    const double l = __ddiv_rn(lu[k], lu[diag[j]]);
    lu[k] = l;
    int p = k + 1;
    const int je = rp[j + 1];
    for (int kk = diag[j] + 1; kk < je; ++kk) {
      const int c = ci[kk];
      while (p < e && ci[p] < c) ++p;
      if (p >= e) break;
      if (ci[p] == c) {
        int q = p;
        while (q + 1 < e && ci[q + 1] == c) ++q;  // iw[] holds the last duplicate
        lu[q] = __dsub_rn(lu[q], __dmul_rn(l, lu[kk]));
      }
    }
  }
  if (lu[diag[i]] == 0.0) atomicMin(err_row, i);
}

// split the merged factors and cast (ilu.cpp:54-120): lower = L * D_l
// (columns scaled by dl_j = sqrt|d_j|), upper = D_u * U (rows scaled by
// du_i = sign(d_i) sqrt|d_i|, U = lu / d_i), each product truncated
__global__ void __launch_bounds__(256) k_split_cast(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const int* __restrict__ diag, const double* __restrict__ lu,
                                                    const int* __restrict__ lrp, const int* __restrict__ urp,
                                                    int* __restrict__ lci, i64* __restrict__ lv,
                                                    int* __restrict__ ldp, int* __restrict__ uci,
                                                    i64* __restrict__ uv, int* __restrict__ udp, int* err_row) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = lu[diag[i]];
  const double r = __dsqrt_rn(fabs(d));
  const double du = d < 0 ? -r : r;
  int lo = lrp[i], up = urp[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    if (j < i) {
      lci[lo] = j;
      lv[lo++] = __double2ll_rz(__dmul_rn(lu[k], __dsqrt_rn(fabs(lu[diag[j]]))));
    } else if (j == i) {
      lci[lo] = i;
      ldp[i] = lo;
      lv[lo++] = __double2ll_rz(__dmul_rn(1.0, r));
      uci[up] = i;
      udp[i] = up;
      uv[up++] = __double2ll_rz(__dmul_rn(1.0, du));
    } else {
      uci[up] = j;
      uv[up++] = __double2ll_rz(__dmul_rn(__ddiv_rn(lu[k], d), du));
    }
  }
  if (lv[ldp[i]] == 0 || uv[udp[i]] == 0) atomicMin(err_row, i);
}

}  // namespace

void launch_row_scale(cudaStream_t st, int n, const int* rp, const double* v, int alpha, double* out,
                      double* scale, int* err_row) {
  k_row_scale<<<(n + 255) / 256 > 0 ? (n + 255) / 256 : 1, 256, 0, st>>>(n, rp, v, alpha, out, scale, err_row);
  ++g_launches;
}

void launch_split_layer(cudaStream_t st, long long nnz, const double* v, double* rem, int alpha, i64* comp,
                        u64* mx_out, bool first) {
  const int g = static_cast<int>(std::max<long long>(1, std::min<long long>((nnz + 255) / 256, 148LL * 16)));
  if (first)
    k_split_first<<<g, 256, 0, st>>>(nnz, v, comp, rem, mx_out);
  else
    k_split_next<<<g, 256, 0, st>>>(nnz, rem, alpha, comp, mx_out);
  ++g_launches;
}

void launch_ilu_pattern(cudaStream_t st, int n, const int* rp, const int* ci, int* diag, int* lcnt, int* ucnt,
                        int* err_row) {
  k_ilu_pattern<<<(n + 255) / 256 > 0 ? (n + 255) / 256 : 1, 256, 0, st>>>(n, rp, ci, diag, lcnt, ucnt, err_row);
  ++g_launches;
}

void launch_ilu_level(cudaStream_t st, int cnt, const int* rows, const int* rp, const int* ci, const int* diag,
                      double* lu, int* err_row) {
  if (cnt <= 0) return;
  k_ilu_rows<<<(cnt + 127) / 128, 128, 0, st>>>(cnt, rows, rp, ci, diag, lu, err_row);
  ++g_launches;
}

void launch_split_cast(cudaStream_t st, int n, const int* rp, const int* ci, const int* diag, const double* lu,
                       const int* lrp, const int* urp, int* lci, i64* lv, int* ldp, int* uci, i64* uv, int* udp,
                       int* err_row) {
  k_split_cast<<<(n + 255) / 256 > 0 ? (n + 255) / 256 : 1, 256, 0, st>>>(n, rp, ci, diag, lu, lrp, urp, lci, lv,
                                                                          ldp, uci, uv, udp, err_row);
  ++g_launches;
}

}  // namespace igm
