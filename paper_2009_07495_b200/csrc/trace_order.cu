// trace_order.cu -- FxTrace::events in the reference's sequential order.
//
// The reference appends one OverflowEvent{kernel, op, restart, step} per
// wrapped primitive, in program order, and keeps the first 1024
// (fxp.hpp:51-103); solve() returns that list as SolveReport::overflow_events
// (refine.cpp:100).  The cycle kernels count events per (step, kernel, op)
// in parallel -- exact totals, but no order.  When a cycle had events and
// the caller's list still has room, this file rebuilds the ordered list:
//
//  * vector calls (spmv, precond forward/backward, dot_i, axpy_i, norm,
//    vec_div) are replayed on the device from the cycle's own basis and
//    accumulators (all calls are bit-deterministic), and for each call a
//    LOCATE pass lists its events: one thread per element recomputes the
//    element's op sequence (the running-sum adds of dot/norm from an
//    exclusive wrapping scan of the terms), an exclusive scan of the
//    per-element counts gives every event's position, and the elements
//    whose events fall inside the remaining room write their op codes;
//  * the scalar work of each step (fx_dot / fx_sqrt finalisations, the
//    stored rotations, t_mp, (c, s), the g update) is replayed on the host
//    from the same accumulators, in gmres_int.cpp's order.
//
// Element order = the reference's loop order: spmv component-major
// (split.cpp:141-153), forward substitution rows ascending and backward rows
// descending (ilu.cpp:126-153), the vector kernels l ascending
// (fxp.cpp:49-104), vec_div per element (gmres_int.cpp:118-124).
#include "igm_internal.cuh"

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

namespace igm {

namespace {

constexpr int kMaxOps = 160;  // per element: 2 * (row length) + 1 (rows up to 79 entries)

// ---- per-element op sequences ------------------------------------------------
// ops(e, codes): the number of events of element e; codes (if non-null) gets
// their op tags in program order

struct SpmvEl {  // e = l * n + i: component l of row i (split.cpp:141-153)
  long long n;
  const int* rp;
  const int* ci;
  const i64* vals;
  long long nnz;
  const int* alphas;
  const i64* v;
  __device__ int ops(long long e, unsigned char* c) const {
    const int l = static_cast<int>(e / n);
    const long long i = e % n;
    i64 out = 0;
    int k = 0;
    for (int ll = 0; ll <= l; ++ll) {
      const i64* cv = vals + static_cast<long long>(ll) * nnz;
      i64 acc = 0;
      for (int q = rp[i]; q < rp[i + 1]; ++q) {
        const i64 a = cv[q], b = v[ci[q]];
        const i64 p = wmul(a, b);
        if (ll == l) {
          if (mul_ovf(a, b) && k < kMaxOps) {
            if (c) c[k] = OP_MUL;
            ++k;
          }
          if (add_ovf(acc, p) && k < kMaxOps) {
            if (c) c[k] = OP_ADD;
            ++k;
          }
        }
        acc = wadd(acc, p);
      }
      const i64 t = asr(acc, alphas[ll]);
      if (ll == l && add_ovf(out, t) && k < kMaxOps) {
        if (c) c[k] = OP_ADD;
        ++k;
      }
      out = wadd(out, t);
    }
    return k;
  }
};

struct TriEl {  // one substitution row: acc = y_i; per entry mul, sub; then div (ilu.cpp:126-153)
  long long n;
  bool backward;
  const int* rp;
  const int* ci;
  const i64* val;
  const i64* diag;
  const i64* y;
  const i64* z;
  __device__ int ops(long long e, unsigned char* c) const {
    const long long i = backward ? n - 1 - e : e;
    i64 acc = y[i];
    int k = 0;
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const i64 l = val[q], zj = z[ci[q]];
      const i64 p = wmul(l, zj);
      if (mul_ovf(l, zj) && k < kMaxOps) {
        if (c) c[k] = OP_MUL;
        ++k;
      }
      if (sub_ovf(acc, p) && k < kMaxOps) {
        if (c) c[k] = OP_SUB;
        ++k;
      }
      acc = wsub(acc, p);
    }
    if (acc == INT64_MIN && diag[i] == -1 && k < kMaxOps) {
      if (c) c[k] = OP_DIV;
      ++k;
    }
    return k;
  }
};

// terms of the running sums: dot (a >> b1)(b >> b2) / norm (a >> b1)^2
__global__ void k_terms(long long n, const i64* __restrict__ w, const i64* __restrict__ v, int b1, int b2,
                        u64* __restrict__ t) {
  for (long long l = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; l < n;
       l += static_cast<long long>(gridDim.x) * blockDim.x) {
    const i64 a = asr(w[l], b1), b = v ? asr(v[l], b2) : a;
    t[l] = static_cast<u64>(wmul(a, b));
  }
}

struct RedEl {  // fx_dot / fx_norm element: mul, then add onto the running sum (fxp.cpp:57-61, 77-81)
  const i64* w;
  const i64* v;  // null: the norm's squares
  int b1, b2;
  const u64* pre;  // exclusive wrapping prefix of the terms
  __device__ int ops(long long l, unsigned char* c) const {
    const i64 a = asr(w[l], b1), b = v ? asr(v[l], b2) : a;
    int k = 0;
    if (mul_ovf(a, b)) {
      if (c) c[k] = OP_MUL;
      ++k;
    }
    if (add_ovf(static_cast<i64>(pre[l]), wmul(a, b))) {
      if (c) c[k] = OP_ADD;
      ++k;
    }
    return k;
  }
};

struct AxpyEl {  // fx_axpy_sub element: mul(hs, v), sub(w, p >> post) (fxp.cpp:98-103); w = the input
  const i64* w;
  const i64* v;
  i64 hs;
  int post;
  __device__ int ops(long long l, unsigned char* c) const {
    const i64 vl = v[l];
    const i64 d = asr(wmul(hs, vl), post);
    int k = 0;
    if (mul_ovf(hs, vl)) {
      if (c) c[k] = OP_MUL;
      ++k;
    }
    if (sub_ovf(w[l], d)) {
      if (c) c[k] = OP_SUB;
      ++k;
    }
    return k;
  }
};

struct DivEl {  // fx_div(w_l, hnext): shl(num), div, shl(q) (fxp.hpp:220-235)
  const i64* w;
  i64 den;
  int b1, e;
  __device__ int ops(long long l, unsigned char* c) const {
    const i64 a = w[l];
    int k = 0;
    if (shl_ovf(a, b1)) {
      if (c) c[k] = OP_SHL;
      ++k;
    }
    const i64 num = wrap_shl(a, b1);
    i64 q;
    if (num == INT64_MIN && den == -1) {
      if (c) c[k] = OP_DIV;
      ++k;
      q = num;
    } else {
      q = sdiv_trunc(num, den);
    }
    if (e >= 0 && shl_ovf(q, e)) {
      if (c) c[k] = OP_SHL;
      ++k;
    }
    return k;
  }
};

template <class El>
__global__ void k_ev_count(long long ne, El el, long long* cnt) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    cnt[e] = el.ops(e, nullptr);
}

template <class El>
__global__ void k_ev_emit(long long ne, El el, const long long* pos, const long long* cnt, long long room,
                          unsigned char* out) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < ne;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = pos[e];
    if (cnt[e] == 0 || p >= room) continue;
    unsigned char c[kMaxOps];
    const int k = el.ops(e, c);
    for (int t = 0; t < k && p + t < room; ++t) out[p + t] = c[t];
  }
}

int grid_of(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

void ck_(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw LaunchFail(std::string("trace locate (") + what + "): " + cudaGetErrorString(e));
}

}  // namespace

// Device scratch of one locate (grown on demand, freed by the caller)
struct LocateScratch {
  long long* cnt = nullptr;
  long long* pos = nullptr;
  u64* terms = nullptr;
  u64* pre = nullptr;
  unsigned char* codes = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  long long cap = 0, tcap = 0;
  ~LocateScratch() {
    cudaFree(cnt);
    cudaFree(pos);
    cudaFree(terms);
    cudaFree(pre);
    cudaFree(codes);
    cudaFree(tmp);
  }
  void ensure(long long ne) {
    if (ne <= cap) return;
    cudaFree(cnt);
    cudaFree(pos);
    ck_(cudaMalloc(&cnt, sizeof(long long) * std::max(ne, 1LL)), "locate scratch");
    ck_(cudaMalloc(&pos, sizeof(long long) * std::max(ne, 1LL)), "locate scratch");
    cap = ne;
  }
  void ensure_terms(long long n) {
    if (n <= tcap) return;
    cudaFree(terms);
    cudaFree(pre);
    ck_(cudaMalloc(&terms, sizeof(u64) * std::max(n, 1LL)), "locate scratch");
    ck_(cudaMalloc(&pre, sizeof(u64) * std::max(n, 1LL)), "locate scratch");
    tcap = n;
  }
  void ensure_tmp(size_t b) {
    if (b <= tmp_bytes) return;
    cudaFree(tmp);
    ck_(cudaMalloc(&tmp, std::max<size_t>(b, 16)), "locate scratch");
    tmp_bytes = b;
  }
};

namespace {

// events of one call, appended in order (at most `room` of them); returns
// the call's total event count
template <class El>
long long locate_call(cudaStream_t st, LocateScratch& S, long long ne, const El& el, long long room,
                      std::vector<unsigned char>& out) {
  if (ne <= 0) return 0;
  S.ensure(ne);
  k_ev_count<El><<<grid_of(ne), 256, 0, st>>>(ne, el, S.cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, S.cnt, S.pos, ne, st);
  S.ensure_tmp(tb);
  cub::DeviceScan::ExclusiveSum(S.tmp, tb, S.cnt, S.pos, ne, st);
  long long last[2] = {0, 0};
  ck_(cudaMemcpyAsync(&last[0], S.pos + (ne - 1), sizeof(long long), cudaMemcpyDeviceToHost, st), "locate");
  ck_(cudaMemcpyAsync(&last[1], S.cnt + (ne - 1), sizeof(long long), cudaMemcpyDeviceToHost, st), "locate");
  ck_(cudaStreamSynchronize(st), "locate");
  const long long total = last[0] + last[1];
  const long long take = std::min(total, room);
  if (take > 0) {
    unsigned char* d_out = nullptr;
    ck_(cudaMalloc(&d_out, static_cast<size_t>(take)), "locate out");
    k_ev_emit<El><<<grid_of(ne), 256, 0, st>>>(ne, el, S.pos, S.cnt, take, d_out);
    const size_t o = out.size();
    out.resize(o + static_cast<size_t>(take));
    ck_(cudaMemcpyAsync(out.data() + o, d_out, static_cast<size_t>(take), cudaMemcpyDeviceToHost, st), "locate");
    ck_(cudaStreamSynchronize(st), "locate");
    cudaFree(d_out);
  }
  ck_(cudaGetLastError(), "locate kernels");
  return total;
}

// exclusive wrapping prefix of the running-sum terms into S.pre
void prefix_terms(cudaStream_t st, LocateScratch& S, long long n, const i64* w, const i64* v, int b1, int b2) {
  S.ensure_terms(n);
  k_terms<<<grid_of(n), 256, 0, st>>>(n, w, v, b1, b2, S.terms);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, S.terms, S.pre, n, st);
  S.ensure_tmp(tb);
  cub::DeviceScan::ExclusiveSum(S.tmp, tb, S.terms, S.pre, n, st);
}

}  // namespace

long long locate_spmv(cudaStream_t st, LocateScratch& S, const DevSplit& m, int s, const i64* v, long long room,
                      std::vector<unsigned char>& out) {
  SpmvEl el{m.n, m.row_ptr, m.col_idx, m.vals, m.nnz, m.alphas, v};
  return locate_call(st, S, static_cast<long long>(m.n) * (s + 1), el, room, out);
}

long long locate_tri(cudaStream_t st, LocateScratch& S, const DevTri& t, bool backward, const i64* y, const i64* z,
                     long long room, std::vector<unsigned char>& out) {
  TriEl el{t.n, backward, t.c_rp, t.c_ci, t.c_val, t.c_diag, y, z};
  return locate_call(st, S, t.n, el, room, out);
}

long long locate_red(cudaStream_t st, LocateScratch& S, long long n, const i64* w, const i64* v, int b1, int b2,
                     long long room, std::vector<unsigned char>& out) {
  prefix_terms(st, S, n, w, v, b1, b2);
  RedEl el{w, v, b1, b2, S.pre};
  return locate_call(st, S, n, el, room, out);
}

long long locate_axpy(cudaStream_t st, LocateScratch& S, long long n, const i64* w, const i64* v, i64 hs, int post,
                      long long room, std::vector<unsigned char>& out) {
  AxpyEl el{w, v, hs, post};
  return locate_call(st, S, n, el, room, out);
}

long long locate_vec_div(cudaStream_t st, LocateScratch& S, long long n, const i64* w, i64 den, int b1, int e,
                         long long room, std::vector<unsigned char>& out) {
  DivEl el{w, den, b1, e};
  return locate_call(st, S, n, el, room, out);
}

LocateScratch* locate_scratch_new() { return new LocateScratch(); }
void locate_scratch_free(LocateScratch* s) { delete s; }

}  // namespace igm
