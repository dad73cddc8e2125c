// capi.cu -- the extern "C" boundary (include/igm.h) and the host drivers
// that enqueue the device cycle / refinement loop.
//
// Control flow: a whole int-GMRES(m) cycle is enqueued on the context's
// stream without any host round trip (kernels early-exit through the Ctl
// block after a break or an error).  The host synchronises once per cycle
// (run_cycle) or once per refinement (solve), exactly where the reference's
// outer loop needs a scalar decision (refine.cpp:52-55, 85).
#include "igm_internal.cuh"
#include "schedule.hpp"
#include "pencil.hpp"
#include "pencil27.cuh"

#include <algorithm>
#include <climits>
#include <cub/cub.cuh>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

using namespace igm;

namespace {

thread_local std::string t_err;

igm_status set_err(igm_status s, const std::string& msg) {
  t_err = msg;
  return s;
}

struct CudaFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ApiFail {
  igm_status st;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFail(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
igm_status guarded(F&& fn) {
  try {
    fn();
    return IGM_OK;
  } catch (const ApiFail& f) {
    return set_err(f.st, f.msg);
  } catch (const CudaFail& e) {
    return set_err(IGM_CUDA_ERROR, e.what());
  } catch (const LaunchFail& e) {
    return set_err(IGM_CUDA_ERROR, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(IGM_CUDA_ERROR, "host allocation failed");
  }
}

[[noreturn]] void fail(igm_status s, const std::string& m) { throw ApiFail{s, m}; }

const char* em_text(int id) {
  switch (id) {
    case EM_NORM_NEG: return "fx_norm: accumulator wrapped negative";
    case EM_DIV_ZERO: return "fx_div: shifted divisor is zero";
    case EM_ENCODE: return "encode: value outside representable range";
    case EM_HESS_ZERO: return "solve_hessenberg: zero diagonal";
    case EM_GAMMA_ZERO: return "gamma_scale: zero residual";
    default: return "device error";
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  // +64 bytes: bulk L2 prefetches round ranges up to 16-byte granules
  ck(cudaMalloc(&p, count * sizeof(T) + 64), "cudaMalloc");
  return static_cast<T*>(p);
}

template <class T>
T* dupload(const T* src, size_t count, cudaStream_t st) {
  T* d = dalloc<T>(count);
  if (count) ck(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyDefault, st), "upload");
  return d;
}

template <class T>
std::vector<T> to_host(const T* src, size_t count) {
  std::vector<T> h(count);
  if (count) ck(cudaMemcpy(h.data(), src, count * sizeof(T), cudaMemcpyDefault), "to_host");
  return h;
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

}  // namespace

void igm_internal_set_error(const std::string& msg) { t_err = msg; }

// ---------------------------------------------------------------------------
// context

struct Work {
  long long n = 0;
  int m = 0;
  i64* basis = nullptr;  // (m+1) * n
  i64* w = nullptr;
  i64* z = nullptr;
  i64* vin = nullptr;
  double* r = nullptr;
  double* r0 = nullptr;
  double* t1 = nullptr;
  double* x = nullptr;
  double* b = nullptr;
  double* x0 = nullptr;
  // per-cycle small arrays, one allocation
  unsigned char* small = nullptr;
  size_t small_bytes = 0;
  u64 *acc = nullptr, *absacc = nullptr, *nacc = nullptr, *nabs = nullptr, *cnt = nullptr;
  u64* snap = nullptr;  // k_arnoldi2's pass snapshot slots {accumulator, arrivals} per (step, pass)
  u64* vmx = nullptr;  // per CTA and basis vector: max |v_i| over the CTA's rows (k_arnoldi certificates)
  i64 *hess = nullptr, *g = nullptr, *cs = nullptr, *sn = nullptr, *gabs = nullptr;
  int* steprec = nullptr;
  double *y = nullptr, *wts = nullptr, *bnorms = nullptr;
  unsigned char* h_small = nullptr;  // pinned mirror
};

struct igm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  Ctl* ctl = nullptr;
  Ctl* h_ctl = nullptr;  // pinned
  Work ws;
  // primitive scratch
  u64* red = nullptr;  // acc, abs hi, abs lo, cnt[OP_COUNT]
  u64* h_red = nullptr;
  void* n2s = nullptr;  // norm2 per-block scratch (norm2_scratch_bytes)
  size_t n2s_bytes = 0;
  // FP64 engine: reconstructed operator values (reconstruct_fp) + scalars
  double* fp_vals = nullptr;
  size_t fp_vals_n = 0;
  double* fp_sc = nullptr;  // [r0n, wnorm_pre, h_0..h_m, hnext] + fdot partials + weights
  size_t fp_sc_n = 0;
  // exact running-sum overflow counting (igm_set_exact_overflow_counts)
  bool exact_adds = false;
  void* adds_s = nullptr;
  size_t adds_bytes = 0;
};

// scratch of the exact add-event count (grown on demand; stream-ordered use)
void* adds_scratch(igm_ctx* c, long long n) {
  const size_t need = exact_adds_scratch_bytes(n);
  if (need > c->adds_bytes) {
    ck(cudaStreamSynchronize(c->stream), "adds scratch");
    dfree(c->adds_s);
    c->adds_s = dalloc<unsigned char>(need);
    c->adds_bytes = need;
  }
  return c->adds_s;
}

// norm2 scratch for vectors of length n (grown on demand; stream-ordered use)
void* n2_scratch(igm_ctx* c, long long n) {
  const size_t need = norm2_scratch_bytes(n);
  if (need > c->n2s_bytes) {
    ck(cudaStreamSynchronize(c->stream), "norm2 scratch");
    dfree(c->n2s);
    c->n2s = dalloc<unsigned char>(need);
    c->n2s_bytes = need;
  }
  return c->n2s;
}

namespace {

void ws_free(Work& w) {
  dfree(w.basis); dfree(w.w); dfree(w.z); dfree(w.vin); dfree(w.r); dfree(w.r0); dfree(w.t1);
  dfree(w.x); dfree(w.b); dfree(w.x0); dfree(w.small); dfree(w.vmx);
  if (w.h_small) cudaFreeHost(w.h_small);
  w = Work{};
}

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

void ws_ensure(igm_ctx* c, long long n, int m) {
  Work& w = c->ws;
  if (n <= w.n && m <= w.m && w.basis) return;
  const long long nn = std::max<long long>(n, w.n);
  const int mm = std::max(m, w.m);
  ws_free(w);
  w.n = nn;
  w.m = mm;
  w.basis = dalloc<i64>(static_cast<size_t>(mm + 1) * nn);
  w.w = dalloc<i64>(nn);
  w.z = dalloc<i64>(nn);
  w.vin = dalloc<i64>(nn);
  w.r = dalloc<double>(nn);
  w.r0 = dalloc<double>(nn);
  w.t1 = dalloc<double>(nn);
  w.x = dalloc<double>(nn);
  w.b = dalloc<double>(nn);
  w.x0 = dalloc<double>(nn);
  w.vmx = dalloc<u64>(static_cast<size_t>(kVmxRows) * (mm + 2));
  // small arrays
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
  const size_t o_acc = take(sizeof(u64) * mm * (mm + 1));
  const size_t o_abs = take(sizeof(u64) * mm * (mm + 1) * 2);
  const size_t o_snap = take(sizeof(u64) * mm * (mm + 1) * 2);
  const size_t o_nacc = take(sizeof(u64) * mm);
  const size_t o_nabs = take(sizeof(u64) * mm * 2);
  const size_t o_cnt = take(sizeof(u64) * mm * K_COUNT * OP_COUNT);
  const size_t o_hess = take(sizeof(i64) * (mm + 1) * mm);
  const size_t o_g = take(sizeof(i64) * (mm + 1));
  const size_t o_cs = take(sizeof(i64) * mm);
  const size_t o_sn = take(sizeof(i64) * mm);
  const size_t o_gabs = take(sizeof(i64) * mm);
  const size_t o_rec = take(sizeof(int) * mm);
  const size_t o_y = take(sizeof(double) * mm);
  const size_t o_wts = take(sizeof(double) * mm);
  const size_t o_bn = take(sizeof(double) * (mm + 1));
  w.small_bytes = off;
  w.small = dalloc<unsigned char>(off);
  ck(cudaMallocHost(reinterpret_cast<void**>(&w.h_small), off), "cudaMallocHost");
  w.acc = reinterpret_cast<u64*>(w.small + o_acc);
  w.absacc = reinterpret_cast<u64*>(w.small + o_abs);
  w.snap = reinterpret_cast<u64*>(w.small + o_snap);
  w.nacc = reinterpret_cast<u64*>(w.small + o_nacc);
  w.nabs = reinterpret_cast<u64*>(w.small + o_nabs);
  w.cnt = reinterpret_cast<u64*>(w.small + o_cnt);
  w.hess = reinterpret_cast<i64*>(w.small + o_hess);
  w.g = reinterpret_cast<i64*>(w.small + o_g);
  w.cs = reinterpret_cast<i64*>(w.small + o_cs);
  w.sn = reinterpret_cast<i64*>(w.small + o_sn);
  w.gabs = reinterpret_cast<i64*>(w.small + o_gabs);
  w.steprec = reinterpret_cast<int*>(w.small + o_rec);
  w.y = reinterpret_cast<double*>(w.small + o_y);
  w.wts = reinterpret_cast<double*>(w.small + o_wts);
  w.bnorms = reinterpret_cast<double*>(w.small + o_bn);
}

// host view of the small arrays after a cycle
template <class T>
const T* hview(const Work& w, const void* dptr) {
  return reinterpret_cast<const T*>(w.h_small + (static_cast<const unsigned char*>(dptr) - w.small));
}

ShiftsD to_sd(const igm_shifts& s) {
  return ShiftsD{s.dot_b1, s.dot_b2, s.axpy_b1, s.norm_b1, s.div_b1, s.div_b2, s.givens_b2, s.rot_b};
}

// ShiftPlan::validate (fxp.cpp:106-127)
void validate_shifts(const igm_shifts& p, int f) {
  auto right = [f](int b, const char* name) {
    if (b < 0 || (b > 0 && b >= f))
      fail(IGM_INVALID_ARGUMENT, std::string("ShiftPlan: ") + name + " must lie in [0, frac_bits)");
  };
  right(p.dot_b1, "dot_b1");
  right(p.dot_b2, "dot_b2");
  right(p.axpy_b1, "axpy_b1");
  right(p.norm_b1, "norm_b1");
  right(p.div_b2, "div_b2");
  right(p.givens_b2, "givens_b2");
  if (p.div_b1 < 0 || p.div_b1 > f) fail(IGM_INVALID_ARGUMENT, "ShiftPlan: div_b1 must lie in [0, frac_bits]");
  if (p.rot_b != 0) fail(IGM_INVALID_ARGUMENT, "ShiftPlan: rot_b must be 0");
  if (2 * (f - p.norm_b1) > 62)
    fail(IGM_INVALID_ARGUMENT, "ShiftPlan: norm accumulator needs 2*(frac_bits - norm_b1) <= 62");
}

void check_qformat(int f) {
  if (f < 0 || f > 62) fail(IGM_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 62]");
}

void check_shift(int b, const char* who) {
  if (b < 0 || b > 63) fail(IGM_INVALID_ARGUMENT, std::string(who) + ": shift out of [0, 63]");
}

// Staging: a device view of a caller buffer (copy-in for host memory).
template <class T>
struct In {
  const T* d = nullptr;
  T* owned = nullptr;
  In(const T* p, size_t count, cudaStream_t st, T* scratch = nullptr) {
    if (!p) return;
    if (is_device_ptr(p)) {
      d = p;
    } else {
      T* dst = scratch ? scratch : (owned = dalloc<T>(count));
      if (count) ck(cudaMemcpyAsync(dst, p, count * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
      d = dst;
    }
  }
  ~In() { dfree(owned); }
  In(const In&) = delete;
  In& operator=(const In&) = delete;
};

// An output: device pointer used directly, host pointer gets a D2H copy.
template <class T>
struct Out {
  T* user;
  T* d = nullptr;
  T* owned = nullptr;
  size_t count;
  bool host;
  Out(T* p, size_t cnt, T* scratch = nullptr) : user(p), count(cnt) {
    host = !is_device_ptr(p);
    if (!host) d = p;
    else d = scratch ? scratch : (owned = dalloc<T>(cnt));
  }
  void fetch(cudaStream_t st) {
    if (host && count) ck(cudaMemcpyAsync(user, d, count * sizeof(T), cudaMemcpyDeviceToHost, st), "D2H");
  }
  ~Out() { dfree(owned); }
  Out(const Out&) = delete;
  Out& operator=(const Out&) = delete;
};

// ----- trace bookkeeping ----------------------------------------------------

const int kKernelOrder[] = {K_SPMV, K_PRECOND, K_DOT, K_AXPY, K_NORM, K_VEC_DIV,
                            K_GIVENS, K_GIVENS_NORM, K_GIVENS_DIV, K_ROT};

void trace_add(igm_trace* t, int kernel, int op, u64 count, int restart, int step) {
  if (!t || count == 0) return;
  t->total += count;
  for (u64 i = 0; i < count && t->n_events < t->cap_events && t->events; ++i) {
    int32_t* e = t->events + 4 * t->n_events;
    e[0] = kernel; e[1] = op; e[2] = restart; e[3] = step;
    t->n_events++;
  }
}

// ordered event lists of the primitives (trace_order.cu): the counters give
// the totals, a locate pass gives the list in the reference's element order
bool list_room(const igm_trace* t) { return t && t->checked && t->events && t->n_events < t->cap_events; }
long long list_left(const igm_trace* t) { return static_cast<long long>(t->cap_events) - t->n_events; }
void list_push(igm_trace* t, int kernel, std::vector<unsigned char>& codes) {
  for (unsigned char op : codes) {
    if (t->n_events >= t->cap_events) break;
    int32_t* e = t->events + 4 * t->n_events;
    e[0] = kernel; e[1] = op; e[2] = t->restart; e[3] = t->step;
    t->n_events++;
  }
  codes.clear();
}
struct Locator {
  std::unique_ptr<LocateScratch, void (*)(LocateScratch*)> s{locate_scratch_new(), locate_scratch_free};
  std::vector<unsigned char> codes;
};

void trace_shift(igm_trace* t, int kernel, int b1, int b2, long long times = 1) {
  if (!t || !t->record_shifts || times <= 0) return;
  for (long long i = 0; i < times; ++i) {
    if (t->n_shifts < t->cap_shifts && t->shifts) {
      int32_t* s = t->shifts + 3 * t->n_shifts;
      s[0] = kernel; s[1] = b1; s[2] = b2;
    } else if (t->n_shifts >= t->cap_shifts) {
      t->n_shifts += times - i;
      return;
    }
    t->n_shifts++;
  }
}

// ----- host-side ILU schedule ------------------------------------------------

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

void build_tri(igm_ctx* c, DevTri& t, int n, const int* rp, const int* ci, const i64* vals,
               const int* dpos, bool upper) {
  TriSchedule S;
  try {
    S = build_tri_schedule(n, rp, ci, vals, dpos, upper, num_sms(c->device), env_int("IGM_TRI_TILE", 0));
  } catch (const std::invalid_argument& e) {
    fail(IGM_INVALID_ARGUMENT, e.what());
  } catch (const std::logic_error& e) {
    fail(IGM_LOGIC_ERROR, e.what());
  }
  cudaStream_t st = c->stream;
  t.n = n;
  t.maxd = S.maxd;
  t.stride = S.stride;
  t.ntiles = S.ntiles;
  t.acyclic = S.acyclic;
  t.nseg = static_cast<int>(S.seg_level.size());
  t.nlevels = S.nlevels;
  t.tile_cap = std::max(1, S.max_tile_rows);  // shared-memory slots the kernel reserves
  for (int q = 0; q < S.ntiles; ++q)
    t.max_tile_segs = std::max(t.max_tile_segs, S.tile_seg[q + 1] - S.tile_seg[q]);
  for (int d = 0; d < 3; ++d) {
    t.grid[d] = S.grid[d];
    t.brick[d] = S.brick[d];
  }
  t.tile_pbase = dupload(S.tile_pbase.data(), S.tile_pbase.size(), st);
  t.tile_seg = dupload(S.tile_seg.data(), S.tile_seg.size(), st);
  t.seg_level = dupload(S.seg_level.data(), S.seg_level.size(), st);
  t.seg_rows = dupload(S.seg_rows.data(), S.seg_rows.size(), st);
  t.seg_wptr = dupload(S.seg_wptr.data(), S.seg_wptr.size(), st);
  t.seg_wt = dupload(S.seg_wt.data(), S.seg_wt.size(), st);
  t.p_row = dupload(S.p_row.data(), S.p_row.size(), st);
  t.p_nd = dupload(S.p_nd.data(), S.p_nd.size(), st);
  t.p_dep = dupload(S.p_dep.data(), S.p_dep.size(), st);
  t.p_val = dupload(S.p_val.data(), S.p_val.size(), st);
  t.p_xrp = dupload(S.p_xrp.data(), S.p_xrp.size(), st);
  t.p_xdep = dupload(S.p_xdep.data(), S.p_xdep.size(), st);
  t.p_xval = dupload(S.p_xval.data(), S.p_xval.size(), st);
  t.p_mag = dupload(S.p_mag.data(), S.p_mag.size(), st);
  t.p_info = dupload(S.p_info.data(), S.p_info.size(), st);
  t.p_diag = dupload(S.p_diag.data(), S.p_diag.size(), st);
  t.p_rec = dupload(S.p_rec.data(), S.p_rec.size(), st);
  t.rec_bytes = S.rec_bytes;
  t.compact = S.compact;
  t.seg_xptr = dupload(S.seg_xptr.data(), S.seg_xptr.size(), st);
  t.seg_xrow = dupload(S.seg_xrow.data(), S.seg_xrow.size(), st);
  t.max_seg_ext = S.max_seg_ext;
  t.c_rp = dupload(S.c_rp.data(), S.c_rp.size(), st);
  t.c_ci = dupload(S.c_ci.data(), S.c_ci.size(), st);
  t.c_val = dupload(S.c_val.data(), S.c_val.size(), st);
  t.c_diag = dupload(S.c_diag.data(), std::max<size_t>(S.c_diag.size(), 1), st);
  t.xz = dalloc<ulonglong2>(static_cast<size_t>(std::max(n, 1)));
  ck(cudaMemsetAsync(t.xz, 0, sizeof(ulonglong2) * std::max(n, 1), st), "xz");
  t.yperm = dalloc<i64>(static_cast<size_t>(n) + 2);
  t.stats = dalloc<u64>(4);  // [max|y|, max|z|, recount CTAs done, pad]
  ck(cudaMemset(t.stats, 0, 4 * sizeof(u64)), "stats");
  t.maxabs_l = 0;
  for (const i64 v : S.c_val) {
    const u64 a = v < 0 ? 0ull - static_cast<u64>(v) : static_cast<u64>(v);
    t.maxabs_l = std::max(t.maxabs_l, a);
  }
  t.prog = dalloc<int>(S.ntiles);
  t.ticket = dalloc<int>(2);  // [tickets taken, CTAs finished]
  ck(cudaMemsetAsync(t.ticket, 0, 2 * sizeof(int), st), "ticket");
  if (S.grid[0] > 0 && env_int("IGM_PENCIL", 1) != 0) {  // structured 7-point: the pencil wavefront
    // bricks are coupled through DSMEM in clusters along y (tri_pencil2.cuh):
    // the largest power of two <= 8 that the brick rows fill
    const int nby = (S.grid[1] + kPenY - 1) / kPenY;
    int cy = nby >= 8 ? 8 : nby >= 4 ? 4 : nby >= 2 ? 2 : 1;
    cy = env_int("IGM_PEN_CY", cy);
    if (cy != 1 && cy != 2 && cy != 4 && cy != 8) cy = 1;
    const PencilStream P = build_pencil_stream(n, rp, ci, vals, dpos, upper, S.grid[0], S.grid[1], S.grid[2], 16,
                                               false, cy);
    if (P.ok) {
      t.pen_cy = P.cy;
      t.pen = true;
      t.pen_gx = P.gx;
      t.pen_gy = P.gy;
      t.pen_gz = P.gz;
      t.pen_nbx = P.nbx;
      t.pen_nby = P.nby;
      t.pen_nbricks = P.nbricks;
      t.pen_S = P.S;
      t.pen_pad = P.pad;
      t.pen_blk = dupload(P.blk.data(), P.blk.size(), st);
      const PencilStream Q =
          build_pencil_stream(n, rp, ci, vals, dpos, upper, S.grid[0], S.grid[1], S.grid[2], 16, true, cy);
      if (Q.ok) t.pen_blk_fp = dupload(Q.blk.data(), Q.blk.size(), st);
      t.pen_bot = dupload(P.brick_of_ticket.data(), P.brick_of_ticket.size(), st);
    }
  }
  if (!t.pen && S.grid[0] > 0 && env_int("IGM_PENCIL", 1) != 0) {  // structured 27-point: the 27-point pencil
    Pencil27Stream Q = build_pencil27_stream(n, rp, ci, vals, dpos, upper, S.grid[0], S.grid[1], S.grid[2]);
    if (Q.ok && Q.nbricks <= pencil27_max_resident(c->device)) {  // every brick resident at once
      t.pen27 = true;
      t.p27_gx = Q.gx;
      t.p27_gy = Q.gy;
      t.p27_gz = Q.gz;
      t.p27_nbx = Q.nbx;
      t.p27_nbricks = Q.nbricks;
      t.p27_rec = dupload(Q.rec.data(), Q.rec.size(), st);
      Q = Pencil27Stream{};
      const Pencil27Stream Qf =
          build_pencil27_stream(n, rp, ci, vals, dpos, upper, S.grid[0], S.grid[1], S.grid[2], true);
      if (Qf.ok) t.p27_rec_fp = dupload(Qf.rec.data(), Qf.rec.size(), st);
    }
  }
  ck(cudaStreamSynchronize(st), "upload_ilu sync");
}

void free_tri(DevTri& t) {
  for (void* p : {static_cast<void*>(t.tile_pbase), static_cast<void*>(t.tile_seg),
                  static_cast<void*>(t.seg_level), static_cast<void*>(t.seg_rows),
                  static_cast<void*>(t.seg_wptr), static_cast<void*>(t.seg_wt),
                  static_cast<void*>(t.p_row), static_cast<void*>(t.p_nd), static_cast<void*>(t.p_dep),
                  static_cast<void*>(t.p_val), static_cast<void*>(t.p_xrp), static_cast<void*>(t.p_xdep),
                  static_cast<void*>(t.p_xval), static_cast<void*>(t.p_mag), static_cast<void*>(t.p_info),
                  static_cast<void*>(t.p_diag), static_cast<void*>(t.p_rec), static_cast<void*>(t.xz),
                  static_cast<void*>(t.seg_xptr), static_cast<void*>(t.seg_xrow), static_cast<void*>(t.c_rp),
                  static_cast<void*>(t.c_ci), static_cast<void*>(t.c_val), static_cast<void*>(t.c_diag),
                  static_cast<void*>(t.prog), static_cast<void*>(t.yperm), static_cast<void*>(t.stats),
                  static_cast<void*>(t.ticket), t.pen_blk, t.pen_blk_fp, static_cast<void*>(t.pen_bot), t.p27_rec, t.p27_rec_fp})
    dfree(p);
  t = DevTri{};
}

// ----- the cycle -------------------------------------------------------------

enum CycleMode { CM_RUN_CYCLE = 0, CM_SOLVE = 1 };

struct CycleParams {
  const DevSplit* m;
  int M, f, s;
  igm_shifts sh;
  const DevIlu* pre;
  bool checked;
  bool collect_norms;
};

// Enqueue one cycle.  CM_SOLVE: r0 = (ws.r / gamma), x updated in ws.x.
// CM_RUN_CYCLE: r0 = b - A x0 (x0 may be null), x_out = x0 + correction.
void enqueue_cycle(igm_ctx* c, const CycleParams& p, CycleMode mode, const double* d_b,
                   const double* d_x0, double* d_xout) {
  Work& w = c->ws;
  cudaStream_t st = c->stream;
  const long long n = p.m->n;
  const int M = p.M, f = p.f, ld = M + 1;
  const ShiftsD sh = to_sd(p.sh);
  Ctl* ctl = c->ctl;
  ck(cudaMemsetAsync(w.small, 0, w.small_bytes, st), "memset small");
  launch_cycle_init(st, ctl, w.g, f);
  // ---- r0 in floating point (gmres_int.cpp:61-70)
  const double* r0 = nullptr;
  if (mode == CM_SOLVE) {
    if (p.pre) {
      const double* gbits = reinterpret_cast<const double*>(&ctl->rmax_bits);
      launch_tri_fp(st, p.pre->lower, false, w.r, w.t1, ctl, gbits);
      launch_tri_fp(st, p.pre->upper, true, w.t1, w.r0, ctl, nullptr);
    } else {
      launch_scale_div(st, n, w.r, w.r0, ctl);
    }
    r0 = w.r0;
  } else {
    const double* src = d_b;
    if (d_x0) {
      launch_spmv_fp_split(st, *p.m, p.s, d_x0, d_b, w.t1, ctl);
      src = w.t1;
    }
    if (p.pre) {
      launch_tri_fp(st, p.pre->lower, false, src, w.r, ctl, nullptr);
      launch_tri_fp(st, p.pre->upper, true, w.r, w.r0, ctl, nullptr);
      r0 = w.r0;
    } else {
      r0 = src;
    }
  }
  launch_norm2_serial(st, n, r0, nullptr, ctl, 3, n2_scratch(c, n));
  launch_encode(st, n, r0, w.basis, f, ctl);
  // ---- Arnoldi steps (gmres_int.cpp:90-160)
  const size_t cstride = static_cast<size_t>(K_COUNT) * OP_COUNT;
  // exact add-event counting (8(f) row 4) runs the separate pass kernels
  // with a counting pass after each reduction
  const bool exact = p.checked && c->exact_adds;
  void* adds = exact ? adds_scratch(c, n) : nullptr;
  const long long arn_S = exact ? 0 : arnoldi_slice(n, c->device);
  if (p.checked)  // the maxima over all rows of this cycle's basis vectors (atomicMax targets)
    ck(cudaMemsetAsync(w.vmx + static_cast<size_t>(kVmxRows - 1) * (ld + 1), 0, sizeof(u64) * (ld + 1), st), "vmx");
  unsigned gbase = 0;  // grid-barrier arrivals so far in this cycle (Ctl::gbar reset by cycle_init)
  for (int j = 0; j < M; ++j) {
    u64* cstep = w.cnt + static_cast<size_t>(j) * cstride;
    i64* vj = w.basis + static_cast<long long>(j) * n;
    // v_j's magnitude bound for the SpMV's certificate: the per-CTA maxima the
    // persistent Arnoldi kernel of step j-1 recorded when it wrote v_j
    const bool vb_ok = p.checked && j > 0;  // (k_arnoldi* and k_vec_div both record it)
    const u64* vb = vb_ok ? w.vmx + static_cast<size_t>(kVmxRows - 1) * (ld + 1) + j : nullptr;
    if (p.pre) {
      launch_spmv_int(st, *p.m, p.s, vj, w.z, cstep + K_SPMV * OP_COUNT, ctl, p.checked, vb);
      // checked mode: one recount launch for the pair (w.z, w.vin and w.w all
      // outlive it), no stats memsets
      const bool pair = p.checked && p.pre->lower.n == p.pre->upper.n;
      launch_tri_int(st, p.pre->lower, false, w.z, w.vin, cstep + K_PRECOND * OP_COUNT, ctl, p.checked, pair);
      launch_tri_int(st, p.pre->upper, true, w.vin, w.w, cstep + K_PRECOND * OP_COUNT, ctl, p.checked, pair);
      if (pair)
        launch_tri_count_pair(st, p.pre->lower, p.pre->upper, w.z, w.vin, w.w, cstep + K_PRECOND * OP_COUNT, ctl);
    } else {
      launch_spmv_int(st, *p.m, p.s, vj, w.w, cstep + K_SPMV * OP_COUNT, ctl, p.checked, vb);
    }
    u64* accj = w.acc + static_cast<size_t>(j) * (M + 1);
    u64* absj = w.absacc + static_cast<size_t>(j) * (M + 1) * 2;
    if (arn_S > 0) {  // one persistent launch: passes, scalar work and vec_div
      launch_arnoldi(st, n, j, arn_S, w.w, w.basis, accj, absj, w.nacc + j, w.nabs + 2 * j, f, sh, cstep, w.hess, ld,
                     w.g, w.cs, w.sn, w.gabs, ctl, gbase, p.checked, w.vmx,
                     w.snap + static_cast<size_t>(j) * (M + 1) * 2);
      gbase += static_cast<unsigned>(arnoldi_barriers(j, arn_S));
      continue;
    }
    for (int i = 0; i <= j; ++i) {
      const i64* vi = w.basis + static_cast<long long>(i) * n;
      const i64* vp = i > 0 ? w.basis + static_cast<long long>(i - 1) * n : nullptr;
      launch_mgs_pass(st, n, i == 0 ? 0 : 1, w.w, vp, vi, i > 0 ? accj + (i - 1) : nullptr,
                      accj + i, absj + 2 * i, f, sh, cstep + K_AXPY * OP_COUNT,
                      cstep + K_DOT * OP_COUNT, ctl, p.checked);
      if (exact)
        launch_exact_adds(st, n, 0, w.w, vi, sh.dot_b1, sh.dot_b2, absj + 2 * i, ctl,
                          cstep + K_DOT * OP_COUNT + OP_ADD, adds);
    }
    launch_mgs_pass(st, n, 2, w.w, vj, nullptr, accj + j, w.nacc + j, w.nabs + 2 * j, f, sh,
                    cstep + K_AXPY * OP_COUNT, cstep + K_NORM * OP_COUNT, ctl, p.checked);
    if (exact)
      launch_exact_adds(st, n, 1, w.w, nullptr, sh.norm_b1, sh.norm_b1, w.nabs + 2 * j, ctl,
                        cstep + K_NORM * OP_COUNT + OP_ADD, adds);
    launch_step_scalar(st, j, f, sh, accj, absj, w.nacc + j, w.nabs + 2 * j, w.hess, ld, w.g, w.cs,
                       w.sn, w.gabs, w.w, cstep, ctl, exact ? 2 : (p.checked ? 1 : 0));
    launch_vec_div(st, n, w.w, w.basis + static_cast<long long>(j + 1) * n, f, sh,
                   cstep + K_VEC_DIV * OP_COUNT, ctl, p.checked,
                   p.checked ? w.vmx + static_cast<size_t>(kVmxRows - 1) * (ld + 1) + j + 1 : nullptr);
  }
  // ---- least squares and update (gmres_int.cpp:163-180)
  launch_cycle_finish(st, M, f, w.hess, w.g, w.y, w.wts, ctl);
  if (mode == CM_SOLVE)
    launch_xupdate(st, n, M, f, w.basis, w.wts, nullptr, w.x, ctl, 1);
  else
    launch_xupdate(st, n, M, f, w.basis, w.wts, d_x0, d_xout, ctl, 0);
  if (p.collect_norms) launch_basis_norms(st, n, M + 1, f, w.basis, n2_scratch(c, n), w.bnorms, ctl);
}

// copy Ctl + small arrays back (async on the stream; caller syncs)
void fetch_cycle_state(igm_ctx* c) {
  ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream), "ctl D2H");
  ck(cudaMemcpyAsync(c->ws.h_small, c->ws.small, c->ws.small_bytes, cudaMemcpyDeviceToHost, c->stream),
     "small D2H");
}

// The cycle's overflow events in the reference's sequential order
// (trace_order.cu): the vector calls of every step with events are replayed
// on the device from the cycle's basis and accumulators and located element
// by element; the scalar work (fx_dot / fx_sqrt finalisations, the stored
// rotations, t_mp, (c, s), g) is replayed here in gmres_int.cpp:90-160's
// order.  Appends to t->events until it is full; t->total is the caller's.
void ordered_events(igm_ctx* c, const CycleParams& p, igm_trace* t, int restart, long long n, int steps_run) {
  Work& w = c->ws;
  cudaStream_t st = c->stream;
  const u64* cnt = hview<u64>(w, w.cnt);
  const u64* acc = hview<u64>(w, w.acc);
  const u64* nacc = hview<u64>(w, w.nacc);
  const int M = p.M, f = p.f;
  const igm_shifts& s = p.sh;
  const size_t cstride = static_cast<size_t>(K_COUNT) * OP_COUNT;
  auto room = [&]() -> long long { return static_cast<long long>(t->cap_events) - t->n_events; };
  auto push = [&](int k, int op, int step) {
    if (t->n_events >= t->cap_events) return;
    int32_t* e = t->events + 4 * t->n_events;
    e[0] = k; e[1] = op; e[2] = restart; e[3] = step;
    t->n_events++;
  };
  std::unique_ptr<LocateScratch, void (*)(LocateScratch*)> S(locate_scratch_new(), locate_scratch_free);
  std::vector<unsigned char> codes;
  auto flush = [&](int k, int step) {
    for (unsigned char op : codes) push(k, op, step);
    codes.clear();
  };
  std::vector<i64> g(static_cast<size_t>(M) + 1, 0), hc(static_cast<size_t>(M), 0), hsn(static_cast<size_t>(M), 0);
  g[0] = static_cast<i64>(1) << f;
  std::vector<i64> col(static_cast<size_t>(M) + 2);
  const int gb2 = s.givens_b2;
  auto fxm_g = [&](i64 a, i64 b, int step) {  // fx_mul(a, b, 0, givens_b2, f) (gmres_int.cpp:18-21)
    const i64 y = asr(b, gb2);
    if (mul_ovf(a, y)) push(K_GIVENS, OP_MUL, step);
    return asr(wmul(a, y), f - gb2);
  };
  // fx_div(a, b, div_b1, div_b2) (fxp.hpp:220-235); false when it throws
  auto fxdiv = [&](i64 a, i64 b, int k, int step, i64* out) {
    if (shl_ovf(a, s.div_b1)) push(k, OP_SHL, step);
    const i64 num = wrap_shl(a, s.div_b1);
    const i64 den = asr(b, s.div_b2);
    if (den == 0) return false;
    i64 q;
    if (num == INT64_MIN && den == -1) {
      push(k, OP_DIV, step);
      q = num;
    } else {
      q = num / den;
    }
    const int e = f - s.div_b1 - s.div_b2;
    if (e >= 0) {
      if (shl_ovf(q, e)) push(k, OP_SHL, step);
      *out = wrap_shl(q, e);
    } else {
      *out = asr(q, -e);
    }
    return true;
  };
  // counts that may miss running-sum adds (add_inexact): locate every call
  const bool all = c->h_ctl->add_inexact != 0;
  for (int j = 0; j < steps_run && room() > 0; ++j) {
    const u64* cj = cnt + static_cast<size_t>(j) * cstride;
    auto ktot = [&](int k) {
      u64 v = all ? 1 : 0;
      for (int op = 1; op < OP_COUNT; ++op) v += cj[k * OP_COUNT + op];
      return v;
    };
    const bool vec = ktot(K_SPMV) + ktot(K_PRECOND) + ktot(K_DOT) + ktot(K_AXPY) + ktot(K_NORM) + ktot(K_VEC_DIV) > 0;
    const u64* aj = acc + static_cast<size_t>(j) * (M + 1);
    // ---- w = M^{-1} A v_j (gmres_int.cpp:94-99)
    if (vec) {
      const i64* vj = w.basis + static_cast<long long>(j) * n;
      i64* y = p.pre ? w.z : w.w;
      launch_spmv_int(st, *p.m, p.s, vj, y, nullptr, nullptr, false);
      if (ktot(K_SPMV)) {
        locate_spmv(st, *S, *p.m, p.s, vj, room(), codes);
        flush(K_SPMV, j);
      }
      if (p.pre) {
        launch_tri_int(st, p.pre->lower, false, w.z, w.vin, nullptr, nullptr, false);
        launch_tri_int(st, p.pre->upper, true, w.vin, w.w, nullptr, nullptr, false);
        if (ktot(K_PRECOND)) {
          locate_tri(st, *S, p.pre->lower, false, w.z, w.vin, room(), codes);
          flush(K_PRECOND, j);
          locate_tri(st, *S, p.pre->upper, true, w.vin, w.w, room(), codes);
          flush(K_PRECOND, j);
        }
      }
    }
    // ---- modified Gram-Schmidt (gmres_int.cpp:101-110)
    const int e_dot = f - s.dot_b1 - s.dot_b2;
    for (int i = 0; i <= j; ++i) {
      const i64* vi = w.basis + static_cast<long long>(i) * n;
      if (vec && ktot(K_DOT)) {
        locate_red(st, *S, n, w.w, vi, s.dot_b1, s.dot_b2, room(), codes);
        flush(K_DOT, j);
      }
      const i64 a = static_cast<i64>(aj[i]);
      i64 hij;
      if (e_dot >= 0) {
        hij = asr(a, e_dot);
      } else {
        if (shl_ovf(a, -e_dot)) push(K_DOT, OP_SHL, j);
        hij = wrap_shl(a, -e_dot);
      }
      col[i] = hij;
      if (vec) {
        if (ktot(K_AXPY)) {
          locate_axpy(st, *S, n, w.w, vi, asr(hij, s.axpy_b1), f - s.axpy_b1, room(), codes);
          flush(K_AXPY, j);
        }
        launch_axpy_only(st, n, w.w, hij, vi, f, s.axpy_b1, nullptr, false);
      }
    }
    // ---- h_{j+1,j} = fx_norm(w) (gmres_int.cpp:112-114, fxp.cpp:69-86)
    if (vec && ktot(K_NORM)) {
      locate_red(st, *S, n, w.w, nullptr, s.norm_b1, s.norm_b1, room(), codes);
      flush(K_NORM, j);
    }
    const i64 nsum = static_cast<i64>(nacc[j]);
    if (nsum < 0) break;  // domain_error
    i64 hnext;
    {
      const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(nsum)));
      if (shl_ovf(r, s.norm_b1)) push(K_NORM, OP_SHL, j);
      hnext = wrap_shl(r, s.norm_b1);
    }
    col[j + 1] = hnext;
    const bool happy = hnext == 0;
    // ---- v_{j+1} = w / h_{j+1,j} (gmres_int.cpp:116-125)
    if (!happy) {
      const i64 den = asr(hnext, s.div_b2);
      if (den == 0) {  // fx_div of element 0 throws after its shl
        i64 w0 = 0;
        ck(cudaMemcpyAsync(&w0, w.w, sizeof(i64), cudaMemcpyDeviceToHost, st), "w0");
        ck(cudaStreamSynchronize(st), "w0");
        if (shl_ovf(w0, s.div_b1)) push(K_VEC_DIV, OP_SHL, j);
        break;
      }
      if (vec && ktot(K_VEC_DIV)) {
        locate_vec_div(st, *S, n, w.w, den, s.div_b1, f - s.div_b1 - s.div_b2, room(), codes);
        flush(K_VEC_DIV, j);
      }
    }
    // ---- stored rotations (gmres_int.cpp:8-25)
    for (int i = 0; i < j; ++i) {
      const i64 ci = hc[i], si = hsn[i], hi = col[i], hn = col[i + 1];
      const i64 a = fxm_g(ci, hi, j), b = fxm_g(si, hn, j), d = fxm_g(ci, hn, j), e = fxm_g(si, hi, j);
      if (add_ovf(a, b)) push(K_GIVENS, OP_ADD, j);
      if (sub_ovf(d, e)) push(K_GIVENS, OP_SUB, j);
      col[i] = wadd(a, b);
      col[i + 1] = wsub(d, e);
    }
    // ---- t_mp = fx_norm((h_jj, h_{j+1,j})) (gmres_int.cpp:132-137)
    i64 tmp;
    {
      const i64 s0 = asr(col[j], s.norm_b1), s1 = asr(col[j + 1], s.norm_b1);
      if (mul_ovf(s0, s0)) push(K_GIVENS_NORM, OP_MUL, j);
      i64 ac = wmul(s0, s0);
      if (mul_ovf(s1, s1)) push(K_GIVENS_NORM, OP_MUL, j);
      const i64 p1 = wmul(s1, s1);
      if (add_ovf(ac, p1)) push(K_GIVENS_NORM, OP_ADD, j);
      ac = wadd(ac, p1);
      if (ac < 0) break;  // domain_error
      const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(ac)));
      if (shl_ovf(r, s.norm_b1)) push(K_GIVENS_NORM, OP_SHL, j);
      tmp = wrap_shl(r, s.norm_b1);
    }
    if (tmp == 0) break;
    // ---- (c, s) (gmres_int.cpp:139-147)
    i64 cj_, sj_;
    if (!fxdiv(col[j], tmp, K_GIVENS_DIV, j, &cj_)) break;
    if (!fxdiv(col[j + 1], tmp, K_GIVENS_DIV, j, &sj_)) break;
    hc[j] = cj_;
    hsn[j] = sj_;
    // ---- g (gmres_int.cpp:149-153)
    {
      const i64 g_old = g[j];
      if (sub_ovf(0, sj_)) push(K_ROT, OP_SUB, j);
      const i64 neg_s = wsub(0, sj_);
      auto fxm_r = [&](i64 a, i64 b) {
        const i64 x = asr(a, s.rot_b), y = asr(b, s.rot_b);
        if (mul_ovf(x, y)) push(K_ROT, OP_MUL, j);
        return asr(wmul(x, y), 2 * f - 2 * s.rot_b - f);
      };
      g[j + 1] = fxm_r(neg_s, g_old);
      g[j] = fxm_r(cj_, g_old);
    }
    if (happy) break;
  }
}

// Fold one cycle's device counters into the trace; returns the cycle total.
u64 account_cycle(igm_ctx* c, const CycleParams& p, igm_trace* t, int restart, long long n) {
  const Work& w = c->ws;
  const Ctl& h = *c->h_ctl;
  const u64* cnt = hview<u64>(w, w.cnt);
  u64 total = 0;
  // how many Arnoldi steps ran (including a step that broke or failed)
  int steps_run;
  if (h.err && h.err_step >= -1) steps_run = h.err_step + 1;
  else if (h.r0n == 0.0) steps_run = 0;
  else if (!h.stop) steps_run = p.M;
  else if (h.nbasis == h.dim) steps_run = h.dim;   // happy breakdown
  else steps_run = std::min(p.M, h.dim + 1);       // t_mp == 0 break
  const size_t cstride = static_cast<size_t>(K_COUNT) * OP_COUNT;
  for (int j = 0; j < steps_run; ++j)
    for (int kk : kKernelOrder)
      for (int op = 1; op < OP_COUNT; ++op) total += cnt[j * cstride + kk * OP_COUNT + op];
  if (t && (total || h.add_inexact)) {
    t->total += total;
    // the event list in the reference's order (the totals above are exact
    // whatever the list's room)
    if (t->events && t->n_events < t->cap_events) ordered_events(c, p, t, restart, n, steps_run);
  }
  if (t) {
    if (h.add_inexact) t->exact = 0;
    // shift records, synthesised in the reference's call order
    if (t->record_shifts) {
      const auto& s = p.sh;
      const u64* nacc = hview<u64>(w, w.nacc);
      for (int j = 0; j < steps_run; ++j) {
        for (int i = 0; i <= j; ++i) {
          trace_shift(t, K_DOT, s.dot_b1, s.dot_b2);
          trace_shift(t, K_AXPY, s.axpy_b1, 0);
        }
        trace_shift(t, K_NORM, s.norm_b1, s.norm_b1);
        const bool last = (j == steps_run - 1);
        // a domain_error of the last step stops the log where the reference
        // throws: fx_norm of w (after its record), vec_div of element 0 (after
        // one record), t_mp's fx_norm, or the first Givens fx_div
        int err_at = 0;  // 1 norm, 2 vec_div, 3 givens_norm, 4 givens_div
        if (last && h.err) {
          const i64 nsum = static_cast<i64>(nacc[j]);
          if (nsum < 0) {
            err_at = 1;
          } else {
            const i64 hnext = wrap_shl(static_cast<i64>(isqrt_u64(static_cast<u64>(nsum))), s.norm_b1);
            if (hnext != 0 && asr(hnext, s.div_b2) == 0) err_at = 2;
            else err_at = h.err_msg == EM_NORM_NEG ? 3 : 4;
          }
        }
        if (err_at == 1) break;
        const bool broke_tmp = last && h.stop && !h.err && h.dim == j;  // t_mp == 0
        const bool vecdiv = err_at == 2 || (err_at == 0 && (!last || h.nbasis == j + 2)) ||
                            (err_at >= 3 && h.nbasis == j + 2);
        if (vecdiv) trace_shift(t, K_VEC_DIV, s.div_b1, s.div_b2, err_at == 2 ? 1 : n);
        if (err_at == 2) break;
        trace_shift(t, K_GIVENS, 0, s.givens_b2, 4LL * j);
        trace_shift(t, K_GIVENS_NORM, s.norm_b1, s.norm_b1);
        if (broke_tmp || err_at == 3) break;
        trace_shift(t, K_GIVENS_DIV, s.div_b1, s.div_b2, err_at == 4 ? 1 : 2);
        if (err_at == 4) break;
        trace_shift(t, K_ROT, s.rot_b, s.rot_b, 2);
      }
    }
  }
  return total;
}

void raise_device_error(igm_ctx* c) {
  const Ctl& h = *c->h_ctl;
  if (h.err) fail(static_cast<igm_status>(h.err), em_text(h.err_msg));
}

igm_ctx* need_ctx(igm_ctx* c) {
  if (!c) fail(IGM_INVALID_ARGUMENT, "null igm_ctx");
  ck(cudaSetDevice(c->device), "cudaSetDevice");
  return c;
}

void reset_ctl(igm_ctx* c) { ck(cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->stream), "ctl reset"); }

}  // namespace

// ===========================================================================
extern "C" {

const char* igm_last_error(void) { return t_err.c_str(); }
const char* igm_version(void) { return "igm_b200 0.1 (sm_100a)"; }

igm_status igm_ctx_create(int device, igm_ctx** out) {
  return guarded([&] {
    if (!out) fail(IGM_INVALID_ARGUMENT, "igm_ctx_create: null out");
    int nd = 0;
    ck(cudaGetDeviceCount(&nd), "cudaGetDeviceCount");
    if (device < 0 || device >= nd) fail(IGM_INVALID_ARGUMENT, "igm_ctx_create: bad device index");
    ck(cudaSetDevice(device), "cudaSetDevice");
    auto c = std::make_unique<igm_ctx>();
    c->device = device;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    c->ctl = dalloc<Ctl>(1);
    ck(cudaMallocHost(reinterpret_cast<void**>(&c->h_ctl), sizeof(Ctl)), "pinned ctl");
    c->red = dalloc<u64>(3 + OP_COUNT);
    ck(cudaMallocHost(reinterpret_cast<void**>(&c->h_red), sizeof(u64) * (3 + OP_COUNT)), "pinned red");
    ck(cudaMemset(c->ctl, 0, sizeof(Ctl)), "memset ctl");
    *out = c.release();
  });
}

void igm_ctx_destroy(igm_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  ws_free(c->ws);
  dfree(c->ctl);
  dfree(c->red);
  dfree(c->n2s);
  dfree(c->fp_vals);
  dfree(c->fp_sc);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  if (c->h_red) cudaFreeHost(c->h_red);
  cudaStreamDestroy(c->stream);
  dfree(c->adds_s);
  delete c;
}

igm_status igm_ctx_synchronize(igm_ctx* c) {
  return guarded([&] { ck(cudaStreamSynchronize(need_ctx(c)->stream), "sync"); });
}

void* igm_ctx_stream(igm_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

uint64_t igm_ctx_launch_count(igm_ctx*) { return g_launches; }

igm_status igm_set_exact_overflow_counts(igm_ctx* c, int on) {
  return guarded([&] {
    need_ctx(c);
    c->exact_adds = on != 0;
  });
}

void igm_profile_enable(int on) { prof_enable(on != 0); }

// debug hook: per-segment phase timestamps of one ILU tile (4 u64 per segment)
int igm_debug_arn_ts(int j, unsigned long long* out, int cap) { return debug_arn_ts(j, out, cap); }
int igm_debug_fx_selftest(int n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  return debug_fx_selftest(n, reinterpret_cast<const u64*>(a), reinterpret_cast<const u64*>(b),
                           reinterpret_cast<u64*>(out));
}

void igm_debug_tri_trace(int tile, unsigned long long* device_buf) {
  igm::tri_trace_setup(tile, device_buf);
}

int igm_profile_collect(double* ms, uint64_t* count) {
  static_assert(sizeof(uint64_t) == sizeof(unsigned long long), "u64");
  prof_collect(ms, reinterpret_cast<unsigned long long*>(count));
  return KC_COUNT;
}

// ---- uploads
igm_status igm_upload_split(igm_ctx* c, int n, int nnz, const int* row_ptr, const int* col_idx,
                            int ncomp, const int64_t* comp_vals, const int* alphas,
                            igm_split** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "upload_split: null out");
    if (n < 0 || nnz < 0 || ncomp < 1) fail(IGM_INVALID_ARGUMENT, "upload_split: bad sizes");
    auto m = std::make_unique<igm_split>();
    m->device = c->device;
    m->n = n;
    m->nnz = nnz;
    m->ncomp = ncomp;
    m->row_ptr = dupload(row_ptr, n + 1, c->stream);
    m->col_idx = dupload(col_idx, nnz, c->stream);
    m->vals = dupload(comp_vals, static_cast<size_t>(ncomp) * nnz, c->stream);
    m->alphas = dupload(alphas, ncomp, c->stream);
    m->h_alphas = is_device_ptr(alphas) ? to_host(alphas, ncomp) : std::vector<int>(alphas, alphas + ncomp);
    m->max_row = device_max_row(c->stream, n, m->row_ptr);
    m->max_abs0 = device_max_abs(c->stream, nnz, m->vals);
    // sliced-ELL copy of component 0 (kernels.cu k_spmv_int_sell) for rows of 9..32 entries.
    // Measured: config 3 (15 entries) 75 -> 58 us per call, config 4 (27) 1.96 -> 1.2 ms; 7-point
    // rows stay on the register-batched CSR kernel (config 2: 43.9 us against 46.2 us with SELL)
    // ... except on very long vectors (config 5, n = 64M: 1.10 -> 0.91 ms per call), where the
    // thread-contiguous CSR loads no longer merge in the L1 as well
    const bool sell_rows = m->max_row >= env_int("IGM_SPMV_SELL_MIN", 9) ||
                           (m->max_row > 0 && n >= env_int("IGM_SPMV_SELL_BIGN", 8 << 20));
    if (sell_rows && m->max_row <= 32 && n >= 4096 && env_int("IGM_SPMV_SELL", 1) != 0) {
      const size_t slots = (static_cast<size_t>(n) + 31) / 32 * 32 * static_cast<size_t>(m->max_row);
      void *sv = nullptr, *sc = nullptr;
      if (cudaMalloc(&sv, slots * sizeof(i64)) == cudaSuccess && cudaMalloc(&sc, slots * sizeof(int)) == cudaSuccess) {
        m->sell_vals = static_cast<i64*>(sv);
        m->sell_cols = static_cast<int*>(sc);
        m->sell_w = m->max_row;
        ck(cudaMemsetAsync(sv, 0, slots * sizeof(i64), c->stream), "sell");
        ck(cudaMemsetAsync(sc, 0, slots * sizeof(int), c->stream), "sell");
        launch_build_sell(c->stream, n, m->sell_w, m->row_ptr, m->col_idx, m->vals, m->sell_vals, m->sell_cols);
      } else {  // no room for the second copy: the CSR kernels serve
        cudaGetLastError();
        if (sv) cudaFree(sv);
      }
    }
    ck(cudaStreamSynchronize(c->stream), "upload sync");
    *out = m.release();
  });
}

void igm_split_free(igm_split* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  dfree(m->row_ptr); dfree(m->col_idx); dfree(m->vals); dfree(m->alphas);
  dfree(m->sell_vals); dfree(m->sell_cols);
  delete m;
}

igm_status igm_upload_csrf(igm_ctx* c, int n, const int* row_ptr, const int* col_idx,
                           const double* vals, igm_csrf** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "upload_csrf: null out");
    if (n < 0) fail(IGM_INVALID_ARGUMENT, "upload_csrf: bad size");
    int nnz = 0;
    ck(cudaMemcpy(&nnz, row_ptr + n, sizeof(int), cudaMemcpyDefault), "nnz");
    auto a = std::make_unique<igm_csrf>();
    a->device = c->device;
    a->n = n;
    a->nnz = nnz;
    a->row_ptr = dupload(row_ptr, n + 1, c->stream);
    a->col_idx = dupload(col_idx, nnz, c->stream);
    a->vals = dupload(vals, nnz, c->stream);
    ck(cudaStreamSynchronize(c->stream), "upload sync");
    *out = a.release();
  });
}

void igm_csrf_free(igm_csrf* a) {
  if (!a) return;
  cudaSetDevice(a->device);
  dfree(a->row_ptr); dfree(a->col_idx); dfree(a->vals);
  delete a;
}

igm_status igm_upload_ilu(igm_ctx* c, int n, const int* lrp, const int* lci, const int64_t* lv,
                          const int* ldp, const int* urp, const int* uci, const int64_t* uv,
                          const int* udp, igm_ilu** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "upload_ilu: null out");
    if (n < 0) fail(IGM_INVALID_ARGUMENT, "upload_ilu: bad size");
    auto hv = [](const auto* p, size_t cnt) {
      using T = std::remove_const_t<std::remove_pointer_t<decltype(p)>>;
      return is_device_ptr(p) ? to_host(p, cnt) : std::vector<T>(p, p + cnt);
    };
    const std::vector<int> Lrp = hv(lrp, n + 1), Urp = hv(urp, n + 1);
    const std::vector<int> Lci = hv(lci, Lrp[n]), Uci = hv(uci, Urp[n]);
    const std::vector<i64> Lv = hv(lv, Lrp[n]), Uv = hv(uv, Urp[n]);
    const std::vector<int> Ldp = hv(ldp, n), Udp = hv(udp, n);
    auto f = std::make_unique<igm_ilu>();
    f->device = c->device;
    f->n = n;
    build_tri(c, f->lower, n, Lrp.data(), Lci.data(), Lv.data(), Ldp.data(), false);
    build_tri(c, f->upper, n, Urp.data(), Uci.data(), Uv.data(), Udp.data(), true);
    *out = f.release();
  });
}

void igm_ilu_free(igm_ilu* f) {
  if (!f) return;
  cudaSetDevice(f->device);
  free_tri(f->lower);
  free_tri(f->upper);
  delete f;
}

int igm_ilu_pencil(const igm_ilu* f, int backward) {
  if (!f) return 0;
  const DevTri& t = backward ? f->upper : f->lower;
  return t.pen ? t.pen_nbricks : (t.pen27 ? t.p27_nbricks : 0);
}

int igm_debug_pencil_stream(int n, const int* rp, const int* ci, const int64_t* vals, const int* dpos, int upper,
                            int gx, int gy, int gz, int* out4) {
  const PencilStream P = build_pencil_stream(n, rp, ci, vals, dpos, upper != 0, gx, gy, gz);
  if (!P.ok) return 0;
  out4[0] = P.nbricks;
  out4[1] = P.S;
  out4[2] = P.nbx;
  out4[3] = P.nby;
  return 1;
}

int igm_debug_pencil27_stream(int n, const int* rp, const int* ci, const int64_t* vals, const int* dpos, int upper,
                              int gx, int gy, int gz, long long* out2) {
  const Pencil27Stream P = build_pencil27_stream(n, rp, ci, vals, dpos, upper != 0, gx, gy, gz);
  if (!P.ok) return 0;
  out2[0] = P.nbricks;
  out2[1] = static_cast<long long>(P.rec.size() / kP27Rec);
  return 1;
}

int igm_ilu_levels(const igm_ilu* f, int backward) {
  return f ? (backward ? f->upper.nlevels : f->lower.nlevels) : 0;
}

int igm_debug_tri_schedule(int n, const int* rp, const int* ci, const int64_t* vals, const int* dpos,
                           int upper, int num_sms_, int* out8) {
  try {
    const TriSchedule S = build_tri_schedule(n, rp, ci, vals, dpos, upper != 0, num_sms_, 0);
    const int v[8] = {S.ntiles, static_cast<int>(S.seg_level.size()), S.nlevels, S.maxd, S.grid[0], S.grid[1],
                      S.grid[2], S.brick[0] * 1000000 + S.brick[1] * 1000 + S.brick[2]};
    for (int i = 0; i < 8; ++i) out8[i] = v[i];
    return validate_tri_schedule(S, rp, ci, upper != 0);
  } catch (const std::exception& e) {
    t_err = e.what();
    return -1;
  }
}

void igm_ilu_schedule_info(const igm_ilu* f, int backward, int* out8) {
  const DevTri& t = backward ? f->upper : f->lower;
  const int v[8] = {t.ntiles, t.nseg, t.nlevels, t.maxd, t.grid[0], t.grid[1], t.grid[2],
                    t.brick[0] * 1000000 + t.brick[1] * 1000 + t.brick[2]};
  for (int i = 0; i < 8; ++i) out8[i] = v[i];
}

// ---- primitives
igm_status igm_spmv(igm_ctx* c, const igm_split* m, int s, const int64_t* v, int64_t* out,
                    igm_trace* t) {
  return guarded([&] {
    need_ctx(c);
    if (s < 0 || s > m->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "spmv: component index out of range");
    const bool chk = t && t->checked;
    In<i64> dv(v, m->n, c->stream);
    Out<i64> dout(out, m->n);
    ck(cudaMemsetAsync(c->red, 0, sizeof(u64) * (3 + OP_COUNT), c->stream), "memset");
    reset_ctl(c);
    launch_spmv_int(c->stream, *m, s, dv.d, dout.d, c->red + 3, c->ctl, chk);
    dout.fetch(c->stream);
    ck(cudaMemcpyAsync(c->h_red, c->red, sizeof(u64) * (3 + OP_COUNT), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (chk) {
      const u64 tot = c->h_red[3 + OP_MUL] + c->h_red[3 + OP_ADD];
      t->total += tot;
      if (tot && list_room(t)) {  // split.cpp:141-153 order
        Locator L;
        locate_spmv(c->stream, *L.s, *m, s, dv.d, list_left(t), L.codes);
        list_push(t, t->kernel, L.codes);
      }
    }
  });
}

igm_status igm_apply_inverse(igm_ctx* c, const igm_ilu* f, const int64_t* y, int64_t* out,
                             igm_trace* t) {
  return guarded([&] {
    need_ctx(c);
    const bool chk = t && t->checked;
    ws_ensure(c, f->n, 1);
    In<i64> dy(y, f->n, c->stream);
    Out<i64> dout(out, f->n);
    ck(cudaMemsetAsync(c->red, 0, sizeof(u64) * (3 + OP_COUNT), c->stream), "memset");
    reset_ctl(c);
    launch_tri_int(c->stream, f->lower, false, dy.d, c->ws.z, c->red + 3, c->ctl, chk);
    launch_tri_int(c->stream, f->upper, true, c->ws.z, dout.d, c->red + 3, c->ctl, chk);
    dout.fetch(c->stream);
    ck(cudaMemcpyAsync(c->h_red, c->red, sizeof(u64) * (3 + OP_COUNT), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (chk) {
      const u64 tot = c->h_red[3 + OP_MUL] + c->h_red[3 + OP_SUB] + c->h_red[3 + OP_DIV];
      t->total += tot;
      if (tot && list_room(t)) {  // ilu.cpp:126-153 order: forward rows, then backward rows descending
        Locator L;
        locate_tri(c->stream, *L.s, f->lower, false, dy.d, c->ws.z, list_left(t), L.codes);
        list_push(t, t->kernel, L.codes);
        locate_tri(c->stream, *L.s, f->upper, true, c->ws.z, dout.d, list_left(t), L.codes);
        list_push(t, t->kernel, L.codes);
      }
    }
  });
}

igm_status igm_apply_inverse_fp(igm_ctx* c, const igm_ilu* f, const double* y, double* out) {
  return guarded([&] {
    need_ctx(c);
    ws_ensure(c, f->n, 1);
    In<double> dy(y, f->n, c->stream);
    Out<double> dout(out, f->n);
    reset_ctl(c);
    launch_tri_fp(c->stream, f->lower, false, dy.d, c->ws.t1, c->ctl, nullptr);
    launch_tri_fp(c->stream, f->upper, true, c->ws.t1, dout.d, c->ctl, nullptr);
    dout.fetch(c->stream);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

// list: the caller's trace when its event list has room -- the elements'
// events in order (fxp.cpp:57-61 / 77-81) are appended after the reduction
static void fx_red_common(igm_ctx* c, long long n, int mode, const int64_t* v, const int64_t* w,
                          int b1, int b2, bool chk, igm_trace* list = nullptr) {
  In<i64> dv(v, n, c->stream);
  In<i64> dw(mode == 0 ? w : nullptr, n, c->stream);
  if (list && n > 0) {
    Locator L;
    locate_red(c->stream, *L.s, n, dv.d, mode == 0 ? dw.d : nullptr, b1, b2, list_left(list), L.codes);
    list_push(list, list->kernel, L.codes);
  }
  ck(cudaMemsetAsync(c->red, 0, sizeof(u64) * (3 + OP_COUNT), c->stream), "memset");
  if (n > 0) launch_fx_red(c->stream, n, mode, dv.d, dw.d, b1, b2, c->red, c->red + 1, c->red + 3, chk);
  if (n > 0 && chk && c->exact_adds)  // exact running-sum events (no-op under the certificate)
    launch_exact_adds(c->stream, n, mode, dv.d, dw.d, b1, b2, c->red + 1, nullptr, c->red + 3 + OP_ADD,
                      adds_scratch(c, n));
  ck(cudaMemcpyAsync(c->h_red, c->red, sizeof(u64) * (3 + OP_COUNT), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "sync");
}

static bool abs_small_h(const u64* ab) {
  const unsigned __int128 s = (static_cast<unsigned __int128>(ab[0]) << 32) + ab[1];
  return s < (static_cast<unsigned __int128>(1) << 63);
}

igm_status igm_fx_dot(igm_ctx* c, int64_t n, const int64_t* v, const int64_t* w, int f, int b1,
                      int b2, int64_t* out, igm_trace* t) {
  return guarded([&] {
    need_ctx(c);
    check_shift(b1, "fx_dot");
    check_shift(b2, "fx_dot");
    if (t) trace_shift(t, t->kernel, b1, b2);
    const bool chk = t && t->checked;
    fx_red_common(c, n, 0, v, w, b1, b2, chk, list_room(t) ? t : nullptr);
    const i64 acc = static_cast<i64>(c->h_red[0]);
    if (chk) {
      t->total += c->h_red[3 + OP_MUL];
      if (c->exact_adds) t->total += c->h_red[3 + OP_ADD];
      else if (!abs_small_h(c->h_red + 1)) t->exact = 0;
    }
    const int e = f - b1 - b2;
    if (e >= 0) {
      *out = asr(acc, e);
    } else {
      if (chk && shl_ovf(acc, -e)) trace_add(t, t->kernel, OP_SHL, 1, t->restart, t->step);
      *out = wrap_shl(acc, -e);
    }
  });
}

igm_status igm_fx_norm(igm_ctx* c, int64_t n, const int64_t* v, int f, int b1, int64_t* out,
                       igm_trace* t) {
  return guarded([&] {
    need_ctx(c);
    check_shift(b1, "fx_norm");
    const int acc_frac = 2 * (f - b1);
    if (acc_frac < 0 || acc_frac > 62)
      fail(IGM_INVALID_ARGUMENT,
           "fx_norm: accumulator format not representable (need 2*(f-b1) in [0, 62])");
    if (t) trace_shift(t, t->kernel, b1, b1);
    const bool chk = t && t->checked;
    fx_red_common(c, n, 1, v, nullptr, b1, b1, chk, list_room(t) ? t : nullptr);
    const i64 acc = static_cast<i64>(c->h_red[0]);
    if (chk) {
      const u64 nmul = c->h_red[3 + OP_MUL];
      t->total += nmul;
      if (c->exact_adds) {
        t->total += c->h_red[3 + OP_ADD];
      } else if (nmul == 0) {
        const unsigned __int128 s = (static_cast<unsigned __int128>(c->h_red[1]) << 32) + c->h_red[2];
        const u64 wraps = static_cast<u64>((s + (static_cast<unsigned __int128>(1) << 63)) >> 64);
        t->total += wraps;
      } else if (!abs_small_h(c->h_red + 1)) {
        t->exact = 0;
      }
    }
    if (acc < 0) fail(IGM_DOMAIN_ERROR, "fx_norm: accumulator wrapped negative");
    const i64 r = static_cast<i64>(isqrt_u64(static_cast<u64>(acc)));
    const int e = f - acc_frac / 2;
    if (e >= 0) {
      if (chk && shl_ovf(r, e)) trace_add(t, t->kernel, OP_SHL, 1, t->restart, t->step);
      *out = wrap_shl(r, e);
    } else {
      *out = asr(r, -e);
    }
  });
}

igm_status igm_fx_axpy_sub(igm_ctx* c, int64_t n, int64_t* w, int64_t h, const int64_t* v, int f,
                           int b1, igm_trace* t) {
  return guarded([&] {
    need_ctx(c);
    check_shift(b1, "fx_axpy_sub");
    if (f - b1 < 0) fail(IGM_INVALID_ARGUMENT, "fx_axpy_sub: b1 exceeds frac_bits");
    if (t) trace_shift(t, t->kernel, b1, 0);
    const bool chk = t && t->checked;
    In<i64> dv(v, n, c->stream);
    const bool wdev = is_device_ptr(w);
    i64* dw = w;
    i64* owned = nullptr;
    if (!wdev) {
      owned = dalloc<i64>(n);
      dw = owned;
      ck(cudaMemcpyAsync(dw, w, sizeof(i64) * n, cudaMemcpyHostToDevice, c->stream), "H2D");
    }
    ck(cudaMemsetAsync(c->red, 0, sizeof(u64) * (3 + OP_COUNT), c->stream), "memset");
    Locator L;
    if (chk && n > 0 && list_room(t))  // fxp.cpp:98-103 order, located on the input w
      locate_axpy(c->stream, *L.s, n, dw, dv.d, asr(h, b1), f - b1, list_left(t), L.codes);
    if (n > 0) launch_axpy_only(c->stream, n, dw, h, dv.d, f, b1, c->red + 3, chk);
    if (!wdev) ck(cudaMemcpyAsync(w, dw, sizeof(i64) * n, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaMemcpyAsync(c->h_red, c->red, sizeof(u64) * (3 + OP_COUNT), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    dfree(owned);
    if (chk) {
      t->total += c->h_red[3 + OP_MUL] + c->h_red[3 + OP_SUB];
      list_push(t, t->kernel, L.codes);
    }
  });
}

igm_status igm_spmv_fp(igm_ctx* c, const igm_csrf* a, const double* x, double* y) {
  return guarded([&] {
    need_ctx(c);
    In<double> dx(x, a->n, c->stream);
    Out<double> dy(y, a->n);
    launch_residual(c->stream, *a, dx.d, nullptr, dy.d, c->ctl, false);
    dy.fetch(c->stream);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

igm_status igm_residual_fp(igm_ctx* c, const igm_csrf* a, const double* x, const double* b,
                           double* r, double* relnorm) {
  return guarded([&] {
    need_ctx(c);
    In<double> dx(x, a->n, c->stream);
    In<double> db(b, a->n, c->stream);
    Out<double> dr(r, a->n);
    reset_ctl(c);
    launch_residual(c->stream, *a, dx.d, db.d, dr.d, c->ctl, false);
    launch_norm2_serial(c->stream, a->n, db.d, nullptr, c->ctl, 1, n2_scratch(c, a->n));
    launch_norm2_serial(c->stream, a->n, dr.d, nullptr, c->ctl, 2, n2_scratch(c, a->n));
    dr.fetch(c->stream);
    ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (relnorm) *relnorm = c->h_ctl->relnorm;
  });
}

igm_status igm_spmv_fp_split(igm_ctx* c, const igm_split* m, int s, const double* x, double* y) {
  return guarded([&] {
    need_ctx(c);
    if (s < 0 || s > m->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "spmv_fp: component index out of range");
    In<double> dx(x, m->n, c->stream);
    Out<double> dy(y, m->n);
    reset_ctl(c);
    launch_spmv_fp_split(c->stream, *m, s, dx.d, nullptr, dy.d, c->ctl);
    dy.fetch(c->stream);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

igm_status igm_norm2(igm_ctx* c, int64_t n, const double* v, double* out) {
  return guarded([&] {
    need_ctx(c);
    In<double> dv(v, n, c->stream);
    double* d = dalloc<double>(1);
    launch_norm2_serial(c->stream, n, dv.d, d, c->ctl, 0, n2_scratch(c, n));
    ck(cudaMemcpyAsync(c->h_red, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    std::memcpy(out, c->h_red, sizeof(double));
    dfree(d);
  });
}

igm_status igm_gamma_scale(igm_ctx* c, int64_t n, const double* r, double* gamma, double* b_k) {
  return guarded([&] {
    need_ctx(c);
    In<double> dr(r, n, c->stream);
    Out<double> db(b_k, n);
    reset_ctl(c);
    if (n > 0) launch_gamma(c->stream, n, dr.d, c->ctl);
    ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    u64 bits = c->h_ctl->rmax_bits;
    double g;
    std::memcpy(&g, &bits, sizeof g);
    if (g == 0.0) fail(IGM_INVALID_ARGUMENT, "gamma_scale: zero residual");
    if (n > 0) launch_scale_div(c->stream, n, dr.d, db.d, c->ctl);
    db.fetch(c->stream);
    ck(cudaStreamSynchronize(c->stream), "sync");
    *gamma = g;
  });
}

// ---- run_cycle
igm_status igm_run_cycle(igm_ctx* c, const igm_split* m, const igm_cycle_cfg* cfg,
                         const double* b, const double* x0, double* x_out, igm_cycle_out* out,
                         igm_trace* t) {
  igm_status st = guarded([&] {
    need_ctx(c);
    if (!cfg || !m) fail(IGM_INVALID_ARGUMENT, "run_cycle: null argument");
    if (cfg->m < 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
    if (cfg->s < 0 || cfg->s > m->ncomp - 1)
      fail(IGM_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
    check_qformat(cfg->frac_bits);
    validate_shifts(cfg->shifts, cfg->frac_bits);
    if (cfg->precond && cfg->precond->n != m->n) fail(IGM_INVALID_ARGUMENT, "run_cycle: dimension mismatch");
    const long long n = m->n;
    ws_ensure(c, n, cfg->m);
    Work& w = c->ws;
    In<double> db(b, n, c->stream, w.b);
    // x0 all-zero => skip spmv_fp exactly like gmres_int.cpp:63-68
    const double* dx0 = nullptr;
    std::unique_ptr<In<double>> dx0h;
    if (x0) {
      bool nonzero = true;
      if (!is_device_ptr(x0)) {
        nonzero = false;
        for (long long i = 0; i < n; ++i) nonzero = nonzero || x0[i] != 0.0;
      }
      if (nonzero) {
        dx0h = std::make_unique<In<double>>(x0, n, c->stream, w.x0);
        dx0 = dx0h->d;
      }
    }
    Out<double> dx(x_out, n, w.x);
    CycleParams p{m, cfg->m, cfg->frac_bits, cfg->s, cfg->shifts, cfg->precond, t && t->checked,
                  cfg->collect_basis_norms != 0};
    reset_ctl(c);
    if (t) t->exact = 1;
    enqueue_cycle(c, p, CM_RUN_CYCLE, db.d, dx0, dx.d);
    fetch_cycle_state(c);
    ck(cudaStreamSynchronize(c->stream), "cycle sync");
    const Ctl& h = *c->h_ctl;
    account_cycle(c, p, t, t ? t->restart : 0, n);
    raise_device_error(c);
    dx.fetch(c->stream);
    const int M = cfg->m;
    if (out) {
      out->dim = h.dim;
      out->r0_norm = h.r0n;
      const double sc = std::ldexp(1.0, -cfg->frac_bits);
      const i64* gabs = hview<i64>(w, w.gabs);
      const i64* cs = hview<i64>(w, w.cs);
      const i64* sn = hview<i64>(w, w.sn);
      for (int j = 0; j < h.dim; ++j) {
        if (out->g_abs) out->g_abs[j] = std::fabs(static_cast<double>(gabs[j]) * sc);
        if (out->cos_d) out->cos_d[j] = static_cast<double>(cs[j]) * sc;
        if (out->sin_d) out->sin_d[j] = static_cast<double>(sn[j]) * sc;
      }
      const int nb = h.r0n == 0.0 ? 0 : h.nbasis;
      out->n_basis = nb;
      out->n_basis_norms = (cfg->collect_basis_norms && h.r0n != 0.0) ? nb : 0;
      if (out->basis_norms && out->n_basis_norms) {
        const double* bn = hview<double>(w, w.bnorms);
        for (int k = 0; k < nb; ++k) out->basis_norms[k] = bn[k];
      }
      if (out->basis && nb)
        ck(cudaMemcpyAsync(out->basis, w.basis, sizeof(i64) * n * nb, cudaMemcpyDefault, c->stream), "basis D2H");
      if (out->hess) std::memcpy(out->hess, hview<i64>(w, w.hess), sizeof(i64) * (M + 1) * M);
      if (out->g) std::memcpy(out->g, hview<i64>(w, w.g), sizeof(i64) * (M + 1));
      if (out->cos_raw) std::memcpy(out->cos_raw, cs, sizeof(i64) * M);
      if (out->sin_raw) std::memcpy(out->sin_raw, sn, sizeof(i64) * M);
      if (h.r0n == 0.0) {  // early return: no state was built (gmres_int.cpp:72-73)
        if (out->g) std::memset(out->g, 0, sizeof(i64) * (M + 1));
      }
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
  return st;
}

// ---- solve
// FP64 GMRES(m) cycle (refsolve.cpp:9-105).  On entry ws.r0 holds
// b - A x0 (pre_r0: the preconditioner is still to be applied to it) or the
// preconditioned r0.  SpMV, preconditioner (integer factors in FP64, or a
// host callback), norms, scalings and the x update follow the reference's
// operation order bit for bit; the MGS dots are deterministic tree
// reductions.  Givens rotations and the back substitution run on the host
// exactly as in refsolve.cpp.  x: mode 1 adds gamma * correction (the
// refinement, refine.cpp:87), mode 0 accumulates onto x0 (fp_cycle).
// Returns the Krylov dimension.
struct FpPre {
  const igm_ilu* ilu = nullptr;
  igm_fp_precond_fn fn = nullptr;
  void* user = nullptr;
};

static void fp_apply_pre(igm_ctx* c, const FpPre& P, long long n, const double* in, double* scratch, double* out) {
  cudaStream_t st = c->stream;
  if (P.ilu) {
    launch_tri_fp(st, P.ilu->lower, false, in, scratch, c->ctl, nullptr);
    launch_tri_fp(st, P.ilu->upper, true, scratch, out, c->ctl, nullptr);
  } else if (P.fn) {
    std::vector<double> hin(static_cast<size_t>(n)), hout(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(hin.data(), in, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "precond D2H");
    ck(cudaStreamSynchronize(st), "sync");
    if (P.fn(P.user, n, hin.data(), hout.data()) != 0) fail(IGM_RUNTIME_ERROR, "fp_cycle: preconditioner failed");
    ck(cudaMemcpyAsync(out, hout.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "precond H2D");
    ck(cudaStreamSynchronize(st), "sync");  // hout is read by the copy
  } else if (out != in) {
    ck(cudaMemcpyAsync(out, in, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "copy");
  }
}

static int fp_cycle_core(igm_ctx* c, const DevCsrf& A, int M, const FpPre& P, bool pre_r0, double gamma,
                         double* x, int xmode, double* r0n_out, std::vector<double>* gabs) {
  Work& w = c->ws;
  cudaStream_t st = c->stream;
  const long long n = A.n;
  const size_t need = static_cast<size_t>(M) + 8 + fdot_blocks() + static_cast<size_t>(M) + 2;
  if (c->fp_sc_n < need) {
    ck(cudaStreamSynchronize(st), "fp scratch");
    dfree(c->fp_sc);
    c->fp_sc = dalloc<double>(need);
    c->fp_sc_n = need;
  }
  double* sc = c->fp_sc;                   // [0] r0n, [1] wnorm_pre, [2..] h_0..h_j, hnext
  double* part = sc + M + 6;               // fdot partials
  double* wts = part + fdot_blocks();      // x-update weights
  double* V = reinterpret_cast<double*>(w.basis);  // (m+1) x n doubles (same bytes as the int basis)
  Ctl* ctl = c->ctl;
  if (pre_r0) fp_apply_pre(c, P, n, w.r0, w.t1, w.r0);
  launch_norm2_serial(st, n, w.r0, sc, ctl, 0, n2_scratch(c, n));
  double r0n = 0.0;
  ck(cudaMemcpyAsync(&r0n, sc, sizeof(double), cudaMemcpyDeviceToHost, st), "r0n");
  ck(cudaStreamSynchronize(st), "sync");
  if (r0n_out) *r0n_out = r0n;
  if (r0n == 0.0) return 0;
  launch_fscale(st, n, w.r0, V, sc);
  const int ld = M + 1;
  std::vector<double> hess(static_cast<size_t>(ld) * M, 0.0), g(ld, 0.0), cs(M, 0.0), sn(M, 0.0);
  std::vector<double> hbuf(M + 4);
  g[0] = 1.0;
  int dim = 0;
  for (int j = 0; j < M; ++j) {
    double* col = &hess[static_cast<size_t>(j) * ld];
    const double* vj = V + static_cast<long long>(j) * n;
    launch_residual(st, A, vj, nullptr, w.t1, ctl, false);  // w = A v_j
    fp_apply_pre(c, P, n, w.t1, w.r, w.t1);
    launch_norm2_serial(st, n, w.t1, sc + 1, ctl, 0, n2_scratch(c, n));  // wnorm_pre
    for (int i = 0; i <= j; ++i)
      launch_fdot_axpy(st, n, w.t1, V + static_cast<long long>(i) * n, part, sc + 2 + i);
    launch_norm2_serial(st, n, w.t1, sc + 3 + j, ctl, 0, n2_scratch(c, n));  // hnext
    ck(cudaMemcpyAsync(hbuf.data(), sc + 1, sizeof(double) * (j + 3), cudaMemcpyDeviceToHost, st), "h");
    ck(cudaStreamSynchronize(st), "sync");
    const double wnorm_pre = hbuf[0];
    for (int i = 0; i <= j; ++i) col[i] = hbuf[1 + i];
    const double hnext = hbuf[2 + j];
    col[j + 1] = hnext;
    const bool happy = hnext <= wnorm_pre * (8.0 * DBL_EPSILON);
    if (!happy) launch_fscale(st, n, w.t1, V + static_cast<long long>(j + 1) * n, sc + 3 + j);
    for (int i = 0; i < j; ++i) {
      const double hi = col[i], hn = col[i + 1];
      col[i] = cs[i] * hi + sn[i] * hn;
      col[i + 1] = cs[i] * hn - sn[i] * hi;
    }
    const double t = std::hypot(col[j], col[j + 1]);
    if (t == 0.0) break;
    cs[j] = col[j] / t;
    sn[j] = col[j + 1] / t;
    col[j] = t;
    col[j + 1] = 0.0;
    const double g_old = g[j];
    g[j + 1] = -sn[j] * g_old;
    g[j] = cs[j] * g_old;
    dim = j + 1;
    if (gabs) gabs->push_back(std::fabs(g[j + 1]));
    if (happy) break;
  }
  if (dim > 0) {
    std::vector<double> y(dim), wt(dim);
    for (int i = dim - 1; i >= 0; --i) {
      double acc = g[i];
      for (int jj = i + 1; jj < dim; ++jj) acc -= hess[static_cast<size_t>(jj) * ld + i] * y[jj];
      y[i] = acc / hess[static_cast<size_t>(i) * ld + i];
    }
    for (int jj = 0; jj < dim; ++jj) wt[jj] = r0n * y[jj];
    ck(cudaMemcpyAsync(wts, wt.data(), sizeof(double) * dim, cudaMemcpyHostToDevice, st), "wts");
    launch_fxupdate(st, n, dim, V, wts, gamma, x, xmode);
    ck(cudaStreamSynchronize(st), "sync");  // wt (host) is read by the copy above
  }
  return dim;
}

// the refinement's FP engine cycle: b = r / gamma, x0 = 0, x += gamma * correction
static int fp_cycle_solve(igm_ctx* c, const DevCsrf& A, int M, double gamma, const igm_ilu* pre) {
  Work& w = c->ws;
  if (pre) {  // b / gamma fused into the preconditioner's gather
    const double* gbits = reinterpret_cast<const double*>(&c->ctl->rmax_bits);
    launch_tri_fp(c->stream, pre->lower, false, w.r, w.t1, c->ctl, gbits);
    launch_tri_fp(c->stream, pre->upper, true, w.t1, w.r0, c->ctl, nullptr);
  } else {
    launch_scale_div(c->stream, A.n, w.r, w.r0, c->ctl);
  }
  FpPre P;
  P.ilu = pre;
  return fp_cycle_core(c, A, M, P, false, gamma, w.x, 1, nullptr, nullptr);
}

igm_status igm_solve(igm_ctx* c, const igm_split* m, const igm_csrf* a_fp, const double* b,
                     const igm_refine_cfg* cfg, const igm_ilu* precond, double* x_out,
                     igm_report* rep, igm_trace* ext) {
  return guarded([&] {
    need_ctx(c);
    if (!cfg || !m || !a_fp || !rep) fail(IGM_INVALID_ARGUMENT, "solve: null argument");
    if (a_fp->n != m->n) fail(IGM_INVALID_ARGUMENT, "solve: dimension mismatch");
    if (cfg->max_refinements < 0) fail(IGM_INVALID_ARGUMENT, "solve: max_refinements must be >= 0");
    const auto t0 = std::chrono::steady_clock::now();
    const long long n = m->n;
    const int M = std::max(cfg->m, 1);
    ws_ensure(c, n, M);
    Work& w = c->ws;
    cudaStream_t st = c->stream;
    const bool checked = ext ? ext->checked != 0 : cfg->checked != 0;
    igm_trace own{};
    own.checked = checked;
    igm_trace* t = ext ? ext : &own;
    t->exact = 1;
    rep->converged = 0;
    rep->refinements = 0;
    rep->total_inner_iterations = 0;
    rep->n_relres = 0;
    rep->overflow_total = 0;
    rep->overflow_exact = 1;

    In<double> db(b, n, st, w.b);
    ck(cudaMemsetAsync(w.x, 0, sizeof(double) * n, st), "x=0");
    reset_ctl(c);
    launch_norm2_serial(st, n, db.d, nullptr, c->ctl, 1, n2_scratch(c, n));  // ||b||
    launch_residual(st, *a_fp, w.x, db.d, w.r, c->ctl, true);
    launch_norm2_serial(st, n, w.r, nullptr, c->ctl, 2, n2_scratch(c, n));
    ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
    ck(cudaStreamSynchronize(st), "sync");
    double relnorm = c->h_ctl->relnorm;
    rep->relres_history[rep->n_relres++] = relnorm;
    int fp_depth = -1;  // FP engine: depth the reconstructed operator was built for

    for (int k = 0; k < cfg->max_refinements && relnorm >= cfg->tol; ++k) {
      const u64 rbits = c->h_ctl->rmax_bits;
      double rmax;
      std::memcpy(&rmax, &rbits, sizeof rmax);
      if (rmax == 0.0) break;
      t->restart = k;
      const u64 before = t->total;
      const int depth = cfg->s_schedule_fn ? cfg->s_schedule_fn(cfg->s_schedule_user, k)
                        : cfg->s_schedule  ? cfg->s_schedule[k]
                                           : cfg->s;
      if (cfg->engine == 1) {  // Engine::floating_point (refine.cpp:74-82)
        if (depth < 0 || depth > m->ncomp - 1)
          fail(IGM_INVALID_ARGUMENT, "reconstruct_fp: component index out of range");
        if (cfg->m < 1) fail(IGM_INVALID_ARGUMENT, "fp_cycle: m must be >= 1");
        if (depth != fp_depth) {  // operator rebuilt lazily when the depth changes
          if (c->fp_vals_n < static_cast<size_t>(std::max(m->nnz, 1))) {
            ck(cudaStreamSynchronize(st), "fp vals");
            dfree(c->fp_vals);
            c->fp_vals = dalloc<double>(std::max(m->nnz, 1));
            c->fp_vals_n = static_cast<size_t>(std::max(m->nnz, 1));
          }
          launch_recon_vals(st, *m, depth, c->fp_vals);
          fp_depth = depth;
        }
        DevCsrf Ar;
        Ar.n = m->n;
        Ar.nnz = m->nnz;
        Ar.row_ptr = m->row_ptr;
        Ar.col_idx = m->col_idx;
        Ar.vals = c->fp_vals;
        Ar.device = m->device;
        const int dim = fp_cycle_solve(c, Ar, cfg->m, rmax, precond);
        raise_device_error(c);
        if (dim == 0) break;
        ck(cudaMemsetAsync(&c->ctl->rmax_bits, 0, sizeof(u64), st), "rmax reset");
        launch_residual(st, *a_fp, w.x, db.d, w.r, c->ctl, true);
        launch_norm2_serial(st, n, w.r, nullptr, c->ctl, 2, n2_scratch(c, n));
        ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
        ck(cudaStreamSynchronize(st), "sync");
        rep->refinements = k + 1;
        rep->total_inner_iterations += dim;
        rep->inner_dims[k] = dim;
        rep->gamma_history[k] = rmax;
        rep->overflow_per_restart[k] = t->total - before;
        relnorm = c->h_ctl->relnorm;
        rep->relres_history[rep->n_relres++] = relnorm;
        continue;
      }
      // run_cycle validation (gmres_int.cpp:47-52)
      if (cfg->m < 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
      if (depth < 0 || depth > m->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
      check_qformat(cfg->frac_bits);
      validate_shifts(cfg->shifts, cfg->frac_bits);
      CycleParams p{m, cfg->m, cfg->frac_bits, depth, cfg->shifts, precond, checked, false};
      enqueue_cycle(c, p, CM_SOLVE, nullptr, nullptr, nullptr);
      // next residual (the x update is skipped on device when dim == 0)
      fetch_cycle_state(c);  // ctl snapshot incl. gamma, before the reset below
      ck(cudaStreamSynchronize(st), "cycle sync");
      const Ctl hc = *c->h_ctl;
      account_cycle(c, p, t, k, n);
      if (hc.add_inexact) rep->overflow_exact = 0;
      raise_device_error(c);
      const int dim = hc.dim;
      if (dim == 0) break;
      ck(cudaMemsetAsync(&c->ctl->rmax_bits, 0, sizeof(u64), st), "rmax reset");
      launch_residual(st, *a_fp, w.x, db.d, w.r, c->ctl, true);
      launch_norm2_serial(st, n, w.r, nullptr, c->ctl, 2, n2_scratch(c, n));
      ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
      ck(cudaStreamSynchronize(st), "sync");
      rep->refinements = k + 1;
      rep->total_inner_iterations += dim;
      rep->inner_dims[k] = dim;
      rep->gamma_history[k] = rmax;
      rep->overflow_per_restart[k] = t->total - before;
      relnorm = c->h_ctl->relnorm;
      rep->relres_history[rep->n_relres++] = relnorm;
    }
    rep->converged = relnorm < cfg->tol;
    rep->overflow_total = t->total;
    if (!t->exact) rep->overflow_exact = 0;
    if (x_out) {
      if (is_device_ptr(x_out))
        ck(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "x");
      else
        ck(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "x");
    }
    ck(cudaStreamSynchronize(st), "sync");
    rep->wall_time_sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- config-5 microbench: SpMV + MGS against k basis vectors, unchecked
igm_status igm_spmv_mgs(igm_ctx* c, const igm_split* m, int s, const int64_t* v_in,
                        const int64_t* basis, int k, int f, int dot_b1, int dot_b2, int axpy_b1,
                        int64_t* w, int64_t* h_out) {
  return guarded([&] {
    need_ctx(c);
    if (k < 1) fail(IGM_INVALID_ARGUMENT, "spmv_mgs: k must be >= 1");
    if (!is_device_ptr(v_in) || !is_device_ptr(basis) || !is_device_ptr(w))
      fail(IGM_INVALID_ARGUMENT, "spmv_mgs: v_in, basis and w must be device memory");
    cudaStream_t st = c->stream;
    const long long n = m->n;
    ws_ensure(c, 1, k);
    ShiftsD sh{dot_b1, dot_b2, axpy_b1, 0, 0, 0, 0, 0};
    ck(cudaMemsetAsync(c->ws.acc, 0, sizeof(u64) * (k + 1), st), "memset");
    reset_ctl(c);
    launch_spmv_int(st, *m, s, v_in, w, nullptr, c->ctl, false);
    for (int i = 0; i < k; ++i) {
      const i64* vi = basis + static_cast<long long>(i) * n;
      const i64* vp = i > 0 ? basis + static_cast<long long>(i - 1) * n : nullptr;
      launch_mgs_pass(st, n, i == 0 ? 0 : 1, w, vp, vi, i > 0 ? c->ws.acc + i - 1 : nullptr,
                      c->ws.acc + i, nullptr, f, sh, nullptr, nullptr, c->ctl, false);
    }
    launch_mgs_pass(st, n, 3, w, basis + static_cast<long long>(k - 1) * n, nullptr,
                    c->ws.acc + k - 1, nullptr, nullptr, f, sh, nullptr, nullptr, c->ctl, false);
    if (h_out) {
      std::vector<u64> acc(k);
      ck(cudaMemcpyAsync(acc.data(), c->ws.acc, sizeof(u64) * k, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      const int e = f - dot_b1 - dot_b2;
      for (int i = 0; i < k; ++i) {
        const i64 a = static_cast<i64>(acc[i]);
        h_out[i] = e >= 0 ? asr(a, e) : wrap_shl(a, -e);
      }
    }
  });
}

igm_status igm_fp_cycle(igm_ctx* c, const igm_csrf* a, int m, const double* b, const double* x0,
                        igm_fp_precond_fn precond, void* user, double* x_out, int* dim, double* r0_norm,
                        double* g_abs) {
  return guarded([&] {
    need_ctx(c);
    if (m < 1) fail(IGM_INVALID_ARGUMENT, "fp_cycle: m must be >= 1");
    if (!a || !b || !x0 || !x_out) fail(IGM_INVALID_ARGUMENT, "fp_cycle: dimension mismatch");
    const long long n = a->n;
    ws_ensure(c, n, m);
    Work& w = c->ws;
    cudaStream_t st = c->stream;
    reset_ctl(c);
    In<double> db(b, n, st);
    In<double> dx0(x0, n, st);
    launch_residual(st, *a, dx0.d, db.d, w.r0, c->ctl, false);  // r0 = b - A x0
    ck(cudaMemcpyAsync(w.x, dx0.d, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "x0");
    FpPre P;
    P.fn = precond;
    P.user = user;
    std::vector<double> gabs;
    double r0n = 0.0;
    const int d = fp_cycle_core(c, *a, m, P, true, 1.0, w.x, 0, &r0n, &gabs);
    if (dim) *dim = d;
    if (r0_norm) *r0_norm = r0n;
    if (g_abs)
      for (size_t i = 0; i < gabs.size(); ++i) g_abs[i] = gabs[i];
    ck(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n,
                       is_device_ptr(x_out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st),
       "x");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"


// ---- device-side setup (setup.cu) --------------------
namespace {
struct ErrRow {  // smallest offending row, reported by atomicMin
  int* d = nullptr;
  explicit ErrRow(cudaStream_t st) {
    d = dalloc<int>(1);
    const int big = INT_MAX;
    ck(cudaMemcpyAsync(d, &big, sizeof(int), cudaMemcpyHostToDevice, st), "err init");
  }
  int get(cudaStream_t st) const {
    int h = INT_MAX;
    ck(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st), "err D2H");
    ck(cudaStreamSynchronize(st), "sync");
    return h;
  }
  ~ErrRow() { dfree(d); }
};

template <class T>
std::vector<T> host_copy(const T* p, size_t count) {
  return is_device_ptr(p) ? to_host(p, count) : std::vector<T>(p, p + count);
}

// exclusive sum of cnt[0..n) into out[0..n] (out[n] = total)
void exclusive_sum(cudaStream_t st, int* cnt, int* out, int n) {
  ck(cudaMemsetAsync(cnt + n, 0, sizeof(int), st), "memset");
  size_t bytes = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, out, n + 1, st), "scan size");
  void* tmp = dalloc<unsigned char>(std::max<size_t>(bytes, 1));
  ck(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, out, n + 1, st), "scan");
  ck(cudaStreamSynchronize(st), "sync");
  dfree(tmp);
}
}  // namespace

extern "C" {

igm_status igm_row_scale_dev(igm_ctx* c, int n, const int* row_ptr, const double* vals, int alpha_a,
                             double* vals_out, double* scale_out) {
  return guarded([&] {
    need_ctx(c);
    if (n < 0 || !row_ptr) fail(IGM_INVALID_ARGUMENT, "row_scale: bad arguments");
    cudaStream_t st = c->stream;
    int nnz = 0;
    ck(cudaMemcpy(&nnz, row_ptr + n, sizeof(int), cudaMemcpyDefault), "nnz");
    In<int> rp(row_ptr, n + 1, st);
    In<double> v(vals, nnz, st);
    Out<double> out(vals_out, nnz), sc(scale_out, n);
    ErrRow err(st);
    launch_row_scale(st, n, rp.d, v.d, alpha_a, out.d, sc.d, err.d);
    const int bad = err.get(st);
    if (bad != INT_MAX) fail(IGM_RUNTIME_ERROR, "row_scale: row " + std::to_string(bad) + " has no nonzero entry");
    out.fetch(st);
    sc.fetch(st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

igm_status igm_build_split_dev(igm_ctx* c, int nnz, const double* vals, int alpha_a, int max_components,
                               int64_t* comp_vals_out, int* alphas_out, int* ncomp_out, int* exact_out) {
  return guarded([&] {
    need_ctx(c);
    if (max_components < 1) fail(IGM_INVALID_ARGUMENT, "build_split: need at least one component");
    if (nnz < 0 || !alphas_out || !ncomp_out || !exact_out) fail(IGM_INVALID_ARGUMENT, "build_split: bad arguments");
    cudaStream_t st = c->stream;
    In<double> v(vals, nnz, st);
    Out<i64> comp(comp_vals_out, static_cast<size_t>(max_components) * nnz);
    double* rem = dalloc<double>(std::max(nnz, 1));
    u64* mx = dalloc<u64>(1);
    auto max_rem = [&](bool first, int alpha, i64* layer) {
      ck(cudaMemsetAsync(mx, 0, sizeof(u64), st), "memset");
      launch_split_layer(st, nnz, v.d, rem, alpha, layer, mx, first);
      u64 h = 0;
      ck(cudaMemcpyAsync(&h, mx, sizeof(u64), cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      double d;
      std::memcpy(&d, &h, sizeof d);
      return d;
    };
    std::vector<int> alphas{0};
    double m = max_rem(true, 0, comp.d);
    igm_status st_err = IGM_OK;
    while (static_cast<int>(alphas.size()) < max_components) {
      if (m == 0.0) break;
      const int alpha = alpha_a - std::ilogb(m);
      if (alpha <= alphas.back()) {
        st_err = IGM_LOGIC_ERROR;
        break;
      }
      m = max_rem(false, alpha, comp.d + alphas.size() * static_cast<size_t>(nnz));
      alphas.push_back(alpha);
    }
    dfree(rem);
    dfree(mx);
    if (st_err != IGM_OK) fail(st_err, "build_split: exponents must increase");
    comp.count = alphas.size() * static_cast<size_t>(nnz);
    comp.fetch(st);
    ck(cudaStreamSynchronize(st), "sync");
    for (size_t l = 0; l < alphas.size(); ++l) alphas_out[l] = alphas[l];
    *ncomp_out = static_cast<int>(alphas.size());
    *exact_out = m == 0.0 ? 1 : 0;
  });
}

igm_status igm_factorize_split_cast_dev(igm_ctx* c, int n, const int* rp_, const int* ci_, const double* vals,
                                        int* lrp_o, int* lci_o, int64_t* lv_o, int* ldp_o, int* urp_o, int* uci_o,
                                        int64_t* uv_o, int* udp_o) {
  return igm_factorize_split_cast_dev_lu(c, n, rp_, ci_, vals, lrp_o, lci_o, lv_o, ldp_o, urp_o, uci_o, uv_o, udp_o,
                                         nullptr);
}

igm_status igm_factorize_split_cast_dev_lu(igm_ctx* c, int n, const int* rp_, const int* ci_, const double* vals,
                                           int* lrp_o, int* lci_o, int64_t* lv_o, int* ldp_o, int* urp_o, int* uci_o,
                                           int64_t* uv_o, int* udp_o, double* lu_o) {
  return guarded([&] {
    need_ctx(c);
    if (n < 0 || !rp_) fail(IGM_INVALID_ARGUMENT, "factorize_ilu0: bad arguments");
    cudaStream_t st = c->stream;
    // DAG levels of the lower pattern (index work on the host, O(nnz)):
    // level(i) = 1 + max level(j) over j < i in row i
    const std::vector<int> hrp = host_copy(rp_, static_cast<size_t>(n) + 1);
    const int nnz = hrp[n];
    const std::vector<int> hci = host_copy(ci_, static_cast<size_t>(nnz));
    std::vector<int> lev(static_cast<size_t>(n), 0);
    int nlev = n > 0 ? 1 : 0;
    for (int i = 0; i < n; ++i) {
      int l = 0;
      for (int k = hrp[i]; k < hrp[i + 1]; ++k) {
        const int j = hci[k];
        if (j >= i) break;
        l = std::max(l, lev[j] + 1);
      }
      lev[i] = l;
      nlev = std::max(nlev, l + 1);
    }
    std::vector<int> off(static_cast<size_t>(nlev) + 1, 0), order(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) ++off[lev[i] + 1];
    for (int l = 0; l < nlev; ++l) off[l + 1] += off[l];
    {
      std::vector<int> cur(off.begin(), off.end() - 1);
      for (int i = 0; i < n; ++i) order[cur[lev[i]]++] = i;
    }
    In<int> rp(rp_, n + 1, st), ci(ci_, nnz, st);
    In<double> v(vals, nnz, st);
    int* rows = dupload(order.data(), order.size(), st);
    double* lu = dalloc<double>(std::max(nnz, 1));
    if (nnz) ck(cudaMemcpyAsync(lu, v.d, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st), "lu");
    int* diag = dalloc<int>(std::max(n, 1));
    int* lcnt = dalloc<int>(n + 1);
    int* ucnt = dalloc<int>(n + 1);
    Out<int> lrp(lrp_o, n + 1), urp(urp_o, n + 1), ldp(ldp_o, n), udp(udp_o, n);
    auto cleanup = [&] { dfree(rows); dfree(lu); dfree(diag); dfree(lcnt); dfree(ucnt); };
    {
      ErrRow e(st);
      launch_ilu_pattern(st, n, rp.d, ci.d, diag, lcnt, ucnt, e.d);
      const int bad = e.get(st);
      if (bad != INT_MAX) {
        cleanup();
        fail(IGM_RUNTIME_ERROR,
             "factorize_ilu0: row " + std::to_string(bad) + " has no diagonal entry in the pattern");
      }
    }
    {
      ErrRow e(st);
      for (int l = 0; l < nlev; ++l) launch_ilu_level(st, off[l + 1] - off[l], rows + off[l], rp.d, ci.d, diag, lu, e.d);
      const int bad = e.get(st);
      if (bad != INT_MAX) {
        cleanup();
        fail(IGM_RUNTIME_ERROR, "factorize_ilu0: zero pivot in row " + std::to_string(bad));
      }
    }
    exclusive_sum(st, lcnt, lrp.d, n);
    exclusive_sum(st, ucnt, urp.d, n);
    int nl = 0, nu = 0;
    ck(cudaMemcpy(&nl, lrp.d + n, sizeof(int), cudaMemcpyDeviceToHost), "nl");
    ck(cudaMemcpy(&nu, urp.d + n, sizeof(int), cudaMemcpyDeviceToHost), "nu");
    Out<int> lci(lci_o, nl), uci(uci_o, nu);
    Out<i64> lv(lv_o, nl), uv(uv_o, nu);
    ErrRow e(st);
    launch_split_cast(st, n, rp.d, ci.d, diag, lu, lrp.d, urp.d, lci.d, lv.d, ldp.d, uci.d, uv.d, udp.d, e.d);
    const int bad = e.get(st);
    if (lu_o && nnz)  // the merged factors (cudaMemcpyDefault: lu_o may be host or device)
      ck(cudaMemcpy(lu_o, lu, sizeof(double) * nnz, cudaMemcpyDefault), "lu out");
    cleanup();
    if (bad != INT_MAX)
      fail(IGM_RUNTIME_ERROR, "split_cast: diagonal entry of row " + std::to_string(bad) +
                                  " truncates to zero; scale the matrix up before factorizing");
    for (auto* o : {&lrp, &urp, &ldp, &udp, &lci, &uci}) o->fetch(st);
    lv.fetch(st);
    uv.fetch(st);
    ck(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"

// ---- row-block (z-slab) partition: rank-local building blocks -------------
// The distributed driver (paper_2009_07495_b200/dist.py) owns the vectors and
// the collectives; these entries enqueue the same kernels as enqueue_cycle on
// the context stream, over device pointers, without synchronising.
namespace {
constexpr size_t kCntStride = static_cast<size_t>(K_COUNT) * OP_COUNT;
}  // namespace

struct igm_dstate {
  int device = 0, m = 0;
  Ctl* ctl = nullptr;
  Ctl* h_ctl = nullptr;
  unsigned char* small = nullptr;
  size_t small_bytes = 0;
  unsigned char* h_small = nullptr;
  u64 *red = nullptr, *lcnt = nullptr, *vcnt = nullptr, *cnt = nullptr;
  i64 *hess = nullptr, *g = nullptr, *cs = nullptr, *sn = nullptr, *gabs = nullptr;
  double *y = nullptr, *wts = nullptr, *chain = nullptr;
  void* n2s = nullptr;
  size_t n2s_bytes = 0;
  u64* slot(int j, int i) const { return red + (static_cast<size_t>(j) * (m + 2) + i) * 3; }
};

namespace {
igm_dstate* need_ds(igm_ctx* c, igm_dstate* d) {
  need_ctx(c);
  if (!d) fail(IGM_INVALID_ARGUMENT, "null igm_dstate");
  if (d->device != c->device) fail(IGM_INVALID_ARGUMENT, "igm_dstate belongs to another device");
  return d;
}
void* ds_n2(igm_ctx* c, igm_dstate* d, long long n) {
  const size_t need = norm2_scratch_bytes(n);
  if (need > d->n2s_bytes) {
    ck(cudaStreamSynchronize(c->stream), "norm2 scratch");
    dfree(d->n2s);
    d->n2s = dalloc<unsigned char>(need);
    d->n2s_bytes = need;
  }
  return d->n2s;
}
void need_dev(const void* p, const char* who) {
  if (p && !is_device_ptr(p)) fail(IGM_INVALID_ARGUMENT, std::string(who) + ": vectors must be device memory");
}
}  // namespace

extern "C" {

igm_status igm_dstate_create(igm_ctx* c, int m, igm_dstate** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "dstate_create: null out");
    if (m < 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
    auto d = std::make_unique<igm_dstate>();
    d->device = c->device;
    d->m = m;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
    const size_t o_red = take(sizeof(u64) * 3 * m * (m + 2));
    const size_t o_l = take(sizeof(u64) * m * kCntStride);
    const size_t o_v = take(sizeof(u64) * m * kCntStride);
    const size_t o_c = take(sizeof(u64) * m * kCntStride);
    const size_t o_h = take(sizeof(i64) * (m + 1) * m);
    const size_t o_g = take(sizeof(i64) * (m + 1));
    const size_t o_cs = take(sizeof(i64) * m);
    const size_t o_sn = take(sizeof(i64) * m);
    const size_t o_ga = take(sizeof(i64) * m);
    const size_t o_y = take(sizeof(double) * m);
    const size_t o_w = take(sizeof(double) * m);
    const size_t o_ch = take(sizeof(double) * 4);
    d->small_bytes = off;
    d->small = dalloc<unsigned char>(off);
    ck(cudaMallocHost(reinterpret_cast<void**>(&d->h_small), off), "cudaMallocHost");
    d->ctl = dalloc<Ctl>(1);
    ck(cudaMallocHost(reinterpret_cast<void**>(&d->h_ctl), sizeof(Ctl)), "cudaMallocHost");
    d->red = reinterpret_cast<u64*>(d->small + o_red);
    d->lcnt = reinterpret_cast<u64*>(d->small + o_l);
    d->vcnt = reinterpret_cast<u64*>(d->small + o_v);
    d->cnt = reinterpret_cast<u64*>(d->small + o_c);
    d->hess = reinterpret_cast<i64*>(d->small + o_h);
    d->g = reinterpret_cast<i64*>(d->small + o_g);
    d->cs = reinterpret_cast<i64*>(d->small + o_cs);
    d->sn = reinterpret_cast<i64*>(d->small + o_sn);
    d->gabs = reinterpret_cast<i64*>(d->small + o_ga);
    d->y = reinterpret_cast<double*>(d->small + o_y);
    d->wts = reinterpret_cast<double*>(d->small + o_w);
    d->chain = reinterpret_cast<double*>(d->small + o_ch);
    ck(cudaMemsetAsync(d->small, 0, d->small_bytes, c->stream), "memset");
    ck(cudaMemsetAsync(d->ctl, 0, sizeof(Ctl), c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "sync");
    *out = d.release();
  });
}

void igm_dstate_free(igm_dstate* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  dfree(d->small); dfree(d->ctl); dfree(d->n2s);
  if (d->h_small) cudaFreeHost(d->h_small);
  if (d->h_ctl) cudaFreeHost(d->h_ctl);
  delete d;
}

igm_status igm_dstate_buffer(igm_dstate* d, int which, int j, void** ptr, int64_t* bytes) {
  return guarded([&] {
    if (!d || !ptr || !bytes) fail(IGM_INVALID_ARGUMENT, "dstate_buffer: null argument");
    if (which != IGM_DS_VCNT && which != IGM_DS_RMAX && which != IGM_DS_CHAIN && (j < 0 || j >= d->m))
      fail(IGM_INVALID_ARGUMENT, "dstate_buffer: step out of range");
    switch (which) {
      case IGM_DS_RED: *ptr = d->slot(j, 0); *bytes = sizeof(u64) * 3 * (d->m + 2); break;
      case IGM_DS_LCNT: *ptr = d->lcnt + j * kCntStride; *bytes = sizeof(u64) * kCntStride; break;
      case IGM_DS_VCNT: *ptr = d->vcnt; *bytes = sizeof(u64) * kCntStride * d->m; break;
      case IGM_DS_RMAX: *ptr = &d->ctl->rmax_bits; *bytes = sizeof(u64); break;
      case IGM_DS_CHAIN: *ptr = d->chain; *bytes = sizeof(double) * 4; break;
      default: fail(IGM_INVALID_ARGUMENT, "dstate_buffer: unknown buffer");
    }
  });
}

igm_status igm_dc_reset(igm_ctx* c, igm_dstate* d) {
  return guarded([&] {
    need_ds(c, d);
    ck(cudaMemsetAsync(d->ctl, 0, sizeof(Ctl), c->stream), "ctl reset");
  });
}

igm_status igm_dc_residual(igm_ctx* c, igm_dstate* d, const igm_csrf* a, const double* x_ext, const double* b,
                           double* r) {
  return guarded([&] {
    need_ds(c, d);
    if (!a) fail(IGM_INVALID_ARGUMENT, "dc_residual: null matrix");
    need_dev(x_ext, "dc_residual"); need_dev(b, "dc_residual"); need_dev(r, "dc_residual");
    ck(cudaMemsetAsync(&d->ctl->rmax_bits, 0, sizeof(u64), c->stream), "rmax reset");
    launch_residual(c->stream, *a, x_ext, b, r, d->ctl, true);
  });
}

igm_status igm_dc_norm2(igm_ctx* c, igm_dstate* d, int64_t n, const double* v, const double* start, double* out,
                        int mode) {
  return guarded([&] {
    need_ds(c, d);
    if (mode != 1 && mode != 2 && mode != 3 && mode != 5) fail(IGM_INVALID_ARGUMENT, "dc_norm2: bad mode");
    if (mode == 5 && !out) fail(IGM_INVALID_ARGUMENT, "dc_norm2: null out");
    need_dev(v, "dc_norm2"); need_dev(start, "dc_norm2"); need_dev(out, "dc_norm2");
    launch_norm2_serial(c->stream, n, v, out, d->ctl, mode, ds_n2(c, d, n), start);
  });
}

igm_status igm_dc_begin(igm_ctx* c, igm_dstate* d, int f) {
  return guarded([&] {
    need_ds(c, d);
    check_qformat(f);
    ck(cudaMemsetAsync(d->small, 0, d->small_bytes, c->stream), "memset small");
    launch_cycle_init(c->stream, d->ctl, d->g, f);
  });
}

igm_status igm_dc_scale(igm_ctx* c, igm_dstate* d, int64_t n, const double* r, double* out) {
  return guarded([&] {
    need_ds(c, d);
    need_dev(r, "dc_scale"); need_dev(out, "dc_scale");
    launch_scale_div(c->stream, n, r, out, d->ctl);
  });
}

igm_status igm_dc_tri_fp(igm_ctx* c, igm_dstate* d, const igm_ilu* f, int backward, const double* in,
                         double* out) {
  return guarded([&] {
    need_ds(c, d);
    if (!f) fail(IGM_INVALID_ARGUMENT, "dc_tri_fp: null factors");
    need_dev(in, "dc_tri_fp"); need_dev(out, "dc_tri_fp");
    launch_tri_fp(c->stream, backward ? f->upper : f->lower, backward != 0, in, out, d->ctl, nullptr);
  });
}

igm_status igm_dc_encode(igm_ctx* c, igm_dstate* d, int64_t n, const double* r0, int64_t* v0, int f) {
  return guarded([&] {
    need_ds(c, d);
    need_dev(r0, "dc_encode"); need_dev(v0, "dc_encode");
    launch_encode(c->stream, n, r0, v0, f, d->ctl);
  });
}

igm_status igm_dc_spmv(igm_ctx* c, igm_dstate* d, const igm_split* m, int s, const int64_t* v_ext, int64_t* out,
                       int j, int checked) {
  return guarded([&] {
    need_ds(c, d);
    if (!m) fail(IGM_INVALID_ARGUMENT, "dc_spmv: null matrix");
    if (s < 0 || s > m->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
    if (j < 0 || j >= d->m) fail(IGM_INVALID_ARGUMENT, "dc_spmv: step out of range");
    need_dev(v_ext, "dc_spmv"); need_dev(out, "dc_spmv");
    launch_spmv_int(c->stream, *m, s, v_ext, out, d->lcnt + j * kCntStride + K_SPMV * OP_COUNT, d->ctl,
                    checked != 0);
  });
}

igm_status igm_dc_tri(igm_ctx* c, igm_dstate* d, const igm_ilu* f, int backward, const int64_t* in,
                      int64_t* out, int j, int checked) {
  return guarded([&] {
    need_ds(c, d);
    if (!f) fail(IGM_INVALID_ARGUMENT, "dc_tri: null factors");
    if (j < 0 || j >= d->m) fail(IGM_INVALID_ARGUMENT, "dc_tri: step out of range");
    need_dev(in, "dc_tri"); need_dev(out, "dc_tri");
    launch_tri_int(c->stream, backward ? f->upper : f->lower, backward != 0, in, out,
                   d->lcnt + j * kCntStride + K_PRECOND * OP_COUNT, d->ctl, checked != 0);
  });
}

igm_status igm_dc_tri_piped(igm_ctx* c, igm_dstate* d, const igm_ilu* f, int backward, const int64_t* in,
                            int64_t* out, int j, int checked, const void* zimp, void* zexp, int kexp,
                            uint64_t epoch) {
  return guarded([&] {
    need_ds(c, d);
    if (!f) fail(IGM_INVALID_ARGUMENT, "dc_tri_piped: null factors");
    if (j < 0 || j >= d->m) fail(IGM_INVALID_ARGUMENT, "dc_tri_piped: step out of range");
    need_dev(in, "dc_tri_piped"); need_dev(out, "dc_tri_piped");
    PenZ z;
    z.imp = static_cast<const ulonglong2*>(zimp);
    z.exp = static_cast<ulonglong2*>(zexp);
    z.kexp = kexp;
    z.epoch = epoch;
    const DevTri& t = backward ? f->upper : f->lower;
    if (!launch_tri_int_piped(c->stream, t, backward != 0, in, out, d->lcnt + j * kCntStride + K_PRECOND * OP_COUNT,
                              d->ctl, checked != 0, z))
      fail(IGM_INVALID_ARGUMENT, "dc_tri_piped: the factor is not a 7-point / 27-point pencil factor");
  });
}

igm_status igm_dev_alloc(igm_ctx* c, uint64_t bytes, void** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "dev_alloc: null output");
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes ? bytes : 16), "dev_alloc");
    ck(cudaMemset(p, 0, bytes ? bytes : 16), "dev_alloc");
    *out = p;
  });
}

void igm_dev_free(void* p) {
  if (p) cudaFree(p);
}

igm_status igm_ipc_handle(const void* dptr, unsigned char handle[64]) {
  return guarded([&] {
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)), "ipc handle");
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
  });
}

igm_status igm_ipc_open(igm_ctx* c, const unsigned char handle[64], void** dptr) {
  return guarded([&] {
    need_ctx(c);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    ck(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
  });
}

void igm_ipc_close(void* dptr) {
  if (dptr) cudaIpcCloseMemHandle(dptr);
}

}  // extern "C"

// ---- one-shot P2P mailbox reductions (igm.h: igm_mbox_*) -------------------
struct igm_mbox {
  int device = 0, rank = 0, world = 1, max_words = 0;
  ulonglong2* local = nullptr;  // [2][world][max_words]
  ulonglong2* peer[IGM_MBOX_MAX_WORLD] = {};
  bool ipc[IGM_MBOX_MAX_WORLD] = {};
  bool connected = false;
  unsigned long long seq = 0;  // reductions issued (identical on every rank)
  int* d_err = nullptr;        // a collect gave up waiting
  unsigned long long timeout_ns = 20000ull * 1000000ull;
};

namespace {

struct MboxPeers {
  ulonglong2* p[IGM_MBOX_MAX_WORLD];
};

__device__ __forceinline__ u64 mbox_tag(u64 seq, int i) { return (seq << 16) + static_cast<u64>(i) + 1; }

// thread (p, i): word i into slot [parity][rank] of rank p's mailbox
__global__ void k_mbox_publish(MboxPeers peers, const u64* __restrict__ words, int n, int rank, int world,
                               int max_words, u64 seq) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * world) return;
  const int p = t / n, i = t - p * n;
  const u64 v = words[i];
  const u64 tag = mbox_tag(seq, i) ^ v;
  ulonglong2* dst = peers.p[p] + (static_cast<size_t>((seq & 1) * world + rank) * max_words + i);
  asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.sys.global.b128 [%0], t; }" ::"l"(dst), "l"(v),
               "l"(tag)
               : "memory");
}

// one warp per word: lane p polls sender p's slot, then a shuffle reduction
__global__ void k_mbox_collect(const ulonglong2* __restrict__ local, u64* __restrict__ words, int n, int world,
                               int max_words, u64 seq, int op, unsigned long long timeout_ns, int* err) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  u64 v = 0;
  bool ok = true;
  if (lane < world) {
    const ulonglong2* src = local + (static_cast<size_t>((seq & 1) * world + lane) * max_words + i);
    const u64 want = mbox_tag(seq, i);
    unsigned long long t0 = 0;
    unsigned spins = 0;
    for (;;) {
      u64 a, b;
      asm volatile("{ .reg .b128 t; ld.relaxed.sys.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                   : "=l"(a), "=l"(b)
                   : "l"(src)
                   : "memory");
      if ((b ^ a) == want) {
        v = a;
        break;
      }
      if ((++spins & 1023u) == 0) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > timeout_ns) {
          ok = false;
          break;
        }
      }
    }
  } else if (op == IGM_MBOX_MAX) {
    v = static_cast<u64>(INT64_MIN);
  }
  __syncwarp();
  if (!__all_sync(0xffffffffu, ok)) {
    if (lane == 0) atomicExch(err, 1);
    return;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const u64 o = __shfl_xor_sync(0xffffffffu, v, d);
    if (op == IGM_MBOX_MAX) v = static_cast<i64>(o) > static_cast<i64>(v) ? o : v;
    else v += o;
  }
  if (lane == 0) words[i] = v;
}

void mbox_need(igm_ctx* c, igm_mbox* m, const void* words, int n) {
  need_ctx(c);
  if (!m) fail(IGM_INVALID_ARGUMENT, "mbox: null mailbox");
  if (m->device != c->device) fail(IGM_INVALID_ARGUMENT, "mbox: mailbox and context are on different devices");
  if (!m->connected) fail(IGM_INVALID_ARGUMENT, "mbox: not connected");
  if (n < 0 || n > m->max_words) fail(IGM_INVALID_ARGUMENT, "mbox: word count out of range");
  if (n > 0 && (!words || !is_device_ptr(words))) fail(IGM_INVALID_ARGUMENT, "mbox: words must be a device pointer");
}

void mbox_publish(igm_ctx* c, igm_mbox* m, const u64* words, int n) {
  ++m->seq;
  if (n == 0) return;
  MboxPeers pp;
  for (int p = 0; p < IGM_MBOX_MAX_WORLD; ++p) pp.p[p] = m->peer[p];
  const int total = n * m->world;
  k_mbox_publish<<<(total + 255) / 256, 256, 0, c->stream>>>(pp, words, n, m->rank, m->world, m->max_words, m->seq);
  ck(cudaPeekAtLastError(), "mbox publish");
  ++g_launches;
}

void mbox_collect(igm_ctx* c, igm_mbox* m, u64* words, int n, int op) {
  if (n == 0) return;
  k_mbox_collect<<<(n + 7) / 8, 256, 0, c->stream>>>(m->local, words, n, m->world, m->max_words, m->seq, op,
                                                      m->timeout_ns, m->d_err);
  ck(cudaPeekAtLastError(), "mbox collect");
  ++g_launches;
}

}  // namespace

extern "C" {

igm_status igm_mbox_create(igm_ctx* c, int rank, int world, int max_words, igm_mbox** out) {
  return guarded([&] {
    need_ctx(c);
    if (!out) fail(IGM_INVALID_ARGUMENT, "mbox_create: null out");
    if (world < 1 || world > IGM_MBOX_MAX_WORLD || rank < 0 || rank >= world)
      fail(IGM_INVALID_ARGUMENT, "mbox_create: rank / world out of range");
    if (max_words < 1 || max_words > IGM_MBOX_MAX_WORDS) fail(IGM_INVALID_ARGUMENT, "mbox_create: max_words out of range");
    auto m = std::make_unique<igm_mbox>();
    m->device = c->device;
    m->rank = rank;
    m->world = world;
    m->max_words = max_words;
    const size_t bytes = sizeof(ulonglong2) * 2 * world * max_words;
    // cudaMalloc (not a pool allocation): the buffer is exported over CUDA IPC
    ck(cudaMalloc(reinterpret_cast<void**>(&m->local), bytes), "mbox_create");
    ck(cudaMemset(m->local, 0, bytes), "mbox_create");
    ck(cudaMalloc(reinterpret_cast<void**>(&m->d_err), sizeof(int)), "mbox_create");
    ck(cudaMemset(m->d_err, 0, sizeof(int)), "mbox_create");
    m->peer[rank] = m->local;
    m->connected = world == 1;
    if (const char* e = std::getenv("IGM_MBOX_TIMEOUT_MS")) {
      const long long ms = std::atoll(e);
      if (ms > 0) m->timeout_ns = static_cast<unsigned long long>(ms) * 1000000ull;
    }
    *out = m.release();
  });
}

void igm_mbox_free(igm_mbox* m) {
  if (!m) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  for (int p = 0; p < m->world; ++p)
    if (m->ipc[p] && m->peer[p]) cudaIpcCloseMemHandle(m->peer[p]);
  cudaFree(m->local);
  cudaFree(m->d_err);
  cudaSetDevice(prev);
  delete m;
}

igm_status igm_mbox_handle(igm_mbox* m, unsigned char handle[64]) {
  return guarded([&] {
    if (!m || !handle) fail(IGM_INVALID_ARGUMENT, "mbox_handle: null argument");
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, m->local), "mbox_handle");
    std::memcpy(handle, &h, 64);
  });
}

igm_status igm_mbox_connect_ipc(igm_mbox* m, const unsigned char* handles) {
  return guarded([&] {
    if (!m || !handles) fail(IGM_INVALID_ARGUMENT, "mbox_connect_ipc: null argument");
    ck(cudaSetDevice(m->device), "cudaSetDevice");
    for (int p = 0; p < m->world; ++p) {
      if (p == m->rank || m->peer[p]) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * static_cast<size_t>(p), 64);
      void* q = nullptr;
      ck(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess), "mbox_connect_ipc");
      m->peer[p] = static_cast<ulonglong2*>(q);
      m->ipc[p] = true;
    }
    m->connected = true;
  });
}

igm_status igm_mbox_connect_local(igm_mbox* m, igm_mbox* const* all) {
  return guarded([&] {
    if (!m || !all) fail(IGM_INVALID_ARGUMENT, "mbox_connect_local: null argument");
    ck(cudaSetDevice(m->device), "cudaSetDevice");
    for (int p = 0; p < m->world; ++p) {
      const igm_mbox* o = all[p];
      if (!o || o->world != m->world || o->rank != p || o->max_words != m->max_words)
        fail(IGM_INVALID_ARGUMENT, "mbox_connect_local: mailbox list does not match the world");
      if (o->device != m->device) {
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, m->device, o->device), "peer access");
        if (!can) fail(IGM_CUDA_ERROR, "mbox_connect_local: no peer access between the devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ck(e, "peer access");
      }
      m->peer[p] = o->local;
    }
    m->connected = true;
  });
}

igm_status igm_mbox_publish(igm_ctx* c, igm_mbox* m, const uint64_t* words, int n) {
  return guarded([&] {
    mbox_need(c, m, words, n);
    mbox_publish(c, m, words, n);
  });
}

igm_status igm_mbox_collect(igm_ctx* c, igm_mbox* m, uint64_t* words, int n, int op) {
  return guarded([&] {
    mbox_need(c, m, words, n);
    if (op != IGM_MBOX_SUM && op != IGM_MBOX_MAX) fail(IGM_INVALID_ARGUMENT, "mbox: unknown reduction");
    mbox_collect(c, m, words, n, op);
  });
}

igm_status igm_mbox_allreduce(igm_ctx* c, igm_mbox* m, uint64_t* words, int n, int op) {
  return guarded([&] {
    mbox_need(c, m, words, std::min(n, m ? m->max_words : 0));
    if (n < 0) fail(IGM_INVALID_ARGUMENT, "mbox: word count out of range");
    if (op != IGM_MBOX_SUM && op != IGM_MBOX_MAX) fail(IGM_INVALID_ARGUMENT, "mbox: unknown reduction");
    if (m->world == 1) return;
    for (int o = 0; o < n; o += m->max_words) {
      const int k = std::min(m->max_words, n - o);
      mbox_publish(c, m, words + o, k);
      mbox_collect(c, m, words + o, k, op);
    }
  });
}

igm_status igm_mbox_status(igm_ctx* c, igm_mbox* m) {
  return guarded([&] {
    need_ctx(c);
    if (!m) fail(IGM_INVALID_ARGUMENT, "mbox: null mailbox");
    ck(cudaStreamSynchronize(c->stream), "mbox_status");
    int e = 0;
    ck(cudaMemcpy(&e, m->d_err, sizeof(int), cudaMemcpyDeviceToHost), "mbox_status");
    if (e) fail(IGM_CUDA_ERROR, "mbox: a reduction timed out waiting for a peer rank");
  });
}

igm_status igm_dc_mgs_pass(igm_ctx* c, igm_dstate* d, int64_t n, int j, int i, int64_t* w, const int64_t* vprev,
                           const int64_t* vcur, int f, const igm_shifts* sh, int checked) {
  return guarded([&] {
    need_ds(c, d);
    if (!sh) fail(IGM_INVALID_ARGUMENT, "dc_mgs_pass: null shifts");
    if (j < 0 || j >= d->m || i < 0 || i > j + 1) fail(IGM_INVALID_ARGUMENT, "dc_mgs_pass: step out of range");
    const int mode = i == 0 ? 0 : (i <= j ? 1 : 2);
    need_dev(w, "dc_mgs_pass"); need_dev(vprev, "dc_mgs_pass"); need_dev(vcur, "dc_mgs_pass");
    if ((mode != 2 && !vcur) || (mode != 0 && !vprev)) fail(IGM_INVALID_ARGUMENT, "dc_mgs_pass: missing vector");
    u64* lc = d->lcnt + j * kCntStride;
    u64* sl = d->slot(j, i);
    launch_mgs_pass(c->stream, n, mode, w, vprev, mode == 2 ? nullptr : vcur, i > 0 ? d->slot(j, i - 1) : nullptr,
                    sl, sl + 1, f, to_sd(*sh), lc + K_AXPY * OP_COUNT, lc + (mode == 2 ? K_NORM : K_DOT) * OP_COUNT,
                    d->ctl, checked != 0);
  });
}

igm_status igm_dc_step(igm_ctx* c, igm_dstate* d, int j, int f, const igm_shifts* sh, const int64_t* w,
                       int checked) {
  return guarded([&] {
    need_ds(c, d);
    if (!sh) fail(IGM_INVALID_ARGUMENT, "dc_step: null shifts");
    if (j < 0 || j >= d->m) fail(IGM_INVALID_ARGUMENT, "dc_step: step out of range");
    need_dev(w, "dc_step");
    u64* s0 = d->slot(j, 0);
    u64* sn = d->slot(j, j + 1);
    launch_step_scalar(c->stream, j, f, to_sd(*sh), s0, s0 + 1, sn, sn + 1, d->hess, d->m + 1, d->g, d->cs, d->sn,
                       d->gabs, w, d->cnt + j * kCntStride, d->ctl, checked != 0, 3, 3,
                       d->lcnt + j * kCntStride + K_NORM * OP_COUNT + OP_MUL);
  });
}

igm_status igm_dc_vec_div(igm_ctx* c, igm_dstate* d, int64_t n, int j, const int64_t* w, int64_t* vout, int f,
                          const igm_shifts* sh, int checked) {
  return guarded([&] {
    need_ds(c, d);
    if (!sh) fail(IGM_INVALID_ARGUMENT, "dc_vec_div: null shifts");
    if (j < 0 || j >= d->m) fail(IGM_INVALID_ARGUMENT, "dc_vec_div: step out of range");
    need_dev(w, "dc_vec_div"); need_dev(vout, "dc_vec_div");
    launch_vec_div(c->stream, n, w, vout, f, to_sd(*sh), d->vcnt + j * kCntStride + K_VEC_DIV * OP_COUNT, d->ctl,
                   checked != 0);
  });
}

igm_status igm_dc_finish(igm_ctx* c, igm_dstate* d, int f, int64_t n, const int64_t* basis, double* x) {
  return guarded([&] {
    need_ds(c, d);
    need_dev(basis, "dc_finish"); need_dev(x, "dc_finish");
    launch_cycle_finish(c->stream, d->m, f, d->hess, d->g, d->y, d->wts, d->ctl);
    launch_xupdate(c->stream, n, d->m, f, basis, d->wts, nullptr, x, d->ctl, 1);
  });
}

igm_status igm_dc_fetch(igm_ctx* c, igm_dstate* d, igm_dc_info* info) {
  return guarded([&] {
    need_ds(c, d);
    if (!info) fail(IGM_INVALID_ARGUMENT, "dc_fetch: null info");
    ck(cudaMemcpyAsync(d->h_ctl, d->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream), "ctl D2H");
    ck(cudaMemcpyAsync(d->h_small, d->small, d->small_bytes, cudaMemcpyDeviceToHost, c->stream), "small D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    const Ctl& h = *d->h_ctl;
    info->dim = h.dim;
    info->stop = h.stop;
    info->nbasis = h.nbasis;
    info->add_inexact = h.add_inexact;
    info->r0_norm = h.r0n;
    info->relnorm = h.relnorm;
    info->nb = h.nb;
    info->nr = h.nr;
    std::memcpy(&info->gamma, &h.rmax_bits, sizeof(double));
    u64 tot = 0;
    auto sum = [&](const u64* dev) {
      const u64* hp = reinterpret_cast<const u64*>(d->h_small + (reinterpret_cast<const unsigned char*>(dev) - d->small));
      for (size_t k = 0; k < kCntStride * d->m; ++k) tot += hp[k];
    };
    sum(d->lcnt); sum(d->vcnt); sum(d->cnt);
    info->overflows = tot;
    if (h.err) fail(static_cast<igm_status>(h.err), em_text(h.err_msg));
  });
}

igm_status igm_mgs_pass(igm_ctx* c, int64_t n, int mode, int64_t* w, const int64_t* vprev,
                        const int64_t* vcur, const uint64_t* hacc, uint64_t* acc_out, int f, int dot_b1,
                        int dot_b2, int axpy_b1) {
  return guarded([&] {
    need_ctx(c);
    if (mode != 0 && mode != 1 && mode != 3) fail(IGM_INVALID_ARGUMENT, "mgs_pass: mode must be 0, 1 or 3");
    if (n < 0) fail(IGM_INVALID_ARGUMENT, "mgs_pass: negative length");
    if (n == 0) return;
    if (!is_device_ptr(w) || (mode != 3 && (!is_device_ptr(vcur) || !is_device_ptr(acc_out))) ||
        (mode != 0 && (!is_device_ptr(vprev) || !is_device_ptr(hacc))))
      fail(IGM_INVALID_ARGUMENT, "mgs_pass: vectors and accumulators must be device memory");
    ShiftsD sh{dot_b1, dot_b2, axpy_b1, 0, 0, 0, 0, 0};
    launch_mgs_pass(c->stream, n, mode, w, vprev, vcur, hacc, acc_out, nullptr, f, sh, nullptr, nullptr, nullptr,
                    false);  // no Ctl: a free-standing pass never ends early
  });
}

}  // extern "C"

// ===========================================================================
// Config 3's WL = 32 variant (wl32.cu).  No reference function: the
// reference's unpreconditioned cycle / solve with int32 words (see igm.h).
struct igm_split32 : igm::Dev32Split {
  Wl32Work ws;  // per-handle cycle buffers (sized on first use)
};

namespace {

void ws32_ensure(igm_split32* m, int M) {
  Wl32Work& w = m->ws;
  const long long n = m->n;
  if (w.n == n && w.M >= M) return;
  dfree(w.basis);
  dfree(w.w);
  dfree(w.small);
  dfree(w.y);
  dfree(w.wts);
  w = Wl32Work{};
  w.n = n;
  w.M = M;
  w.basis = dalloc<int32_t>(static_cast<size_t>(M + 1) * n + 1);
  w.w = dalloc<int32_t>(static_cast<size_t>(n) + 1);
  const size_t na = static_cast<size_t>(M) * (M + 1);
  const size_t cnt = static_cast<size_t>(M) * K_COUNT * OP_COUNT;
  // u64 arrays first (alignment), then the 32-bit ones
  const size_t bytes = 8 * (na + M + cnt) + 4 * (na + M + static_cast<size_t>(M + 1) * M + (M + 1) + 2 * M) + 64;
  w.small = dalloc<unsigned char>(bytes);
  w.small_bytes = bytes;
  unsigned char* p = static_cast<unsigned char*>(w.small);
  w.abs = reinterpret_cast<u64*>(p);
  w.nabs = w.abs + na;
  w.cnt = w.nabs + M;
  uint32_t* q = reinterpret_cast<uint32_t*>(w.cnt + cnt);
  w.acc = q;
  w.nacc = w.acc + na;
  w.hess = reinterpret_cast<int32_t*>(w.nacc + M);
  w.g = w.hess + static_cast<size_t>(M + 1) * M;
  w.cs = w.g + (M + 1);
  w.sn = w.cs + M;
  w.y = dalloc<double>(M);
  w.wts = dalloc<double>(M);
}

void validate_shifts32(const igm_shifts& p, int f) {  // fxp.cpp:106-127 at WL = 32 (rot_b relaxed)
  if (f < 0 || f > 30) fail(IGM_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 30]");
  auto right = [&](int b, const char* name) {
    if (b < 0 || (b > 0 && b >= f)) fail(IGM_INVALID_ARGUMENT, std::string("ShiftPlan: ") + name + " must lie in [0, frac_bits)");
  };
  right(p.dot_b1, "dot_b1");
  right(p.dot_b2, "dot_b2");
  right(p.axpy_b1, "axpy_b1");
  right(p.norm_b1, "norm_b1");
  right(p.div_b2, "div_b2");
  right(p.givens_b2, "givens_b2");
  if (p.div_b1 < 0 || p.div_b1 > f) fail(IGM_INVALID_ARGUMENT, "ShiftPlan: div_b1 must lie in [0, frac_bits]");
  if (p.rot_b < 0 || (p.rot_b > 0 && p.rot_b >= f)) fail(IGM_INVALID_ARGUMENT, "ShiftPlan: rot_b must lie in [0, frac_bits)");
  if (2 * (f - p.norm_b1) > 30)
    fail(IGM_INVALID_ARGUMENT, "ShiftPlan: norm accumulator needs 2*(frac_bits - norm_b1) <= 30");
}

// one cycle at WL = 32 from the FP64 right-hand side r0 (device); returns dim
int cycle32(igm_ctx* c, igm_split32* m, const igm_cycle32_cfg& cfg, const double* r0, int xmode, double* x) {
  cudaStream_t st = c->stream;
  const long long n = m->n;
  ws32_ensure(m, cfg.m);
  ck(cudaMemsetAsync(m->ws.small, 0, m->ws.small_bytes, st), "wl32 zero");
  launch_norm2_serial(st, n, r0, nullptr, c->ctl, 3, n2_scratch(c, n));  // r0n (gmres_int.cpp:71-75)
  enqueue_cycle32(st, m->ws, *m, cfg.m, cfg.frac_bits, cfg.s, to_sd(cfg.shifts), r0, c->ctl, cfg.checked != 0, xmode,
                  x);
  ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
  ck(cudaStreamSynchronize(st), "wl32 cycle");
  raise_device_error(c);
  return c->h_ctl->dim;
}

u64 cycle32_overflows(igm_ctx* c, igm_split32* m, int M, bool* inexact) {
  std::vector<u64> cnt(static_cast<size_t>(M) * K_COUNT * OP_COUNT);
  ck(cudaMemcpy(cnt.data(), m->ws.cnt, cnt.size() * 8, cudaMemcpyDeviceToHost), "wl32 counters");
  u64 t = 0;
  for (u64 v : cnt) t += v;
  *inexact = c->h_ctl->add_inexact != 0;
  return t;
}

}  // namespace

igm_status igm_split32_from_split(igm_ctx* c, const igm_split* m, igm_split32** out) {
  return guarded([&] {
    need_ctx(c);
    if (!m || !out) fail(IGM_INVALID_ARGUMENT, "split32: null argument");
    auto* s = new igm_split32();
    s->n = m->n;
    s->nnz = m->nnz;
    s->ncomp = m->ncomp;
    s->row_ptr = m->row_ptr;  // the pattern is shared with the WL = 64 split
    s->col_idx = m->col_idx;
    s->own_pattern = false;
    s->max_row = m->max_row;
    s->h_alphas = m->h_alphas;
    s->device = c->device;
    const long long cnt = static_cast<long long>(m->ncomp) * m->nnz;
    s->vals = dalloc<int32_t>(static_cast<size_t>(std::max(cnt, 1LL)));
    s->alphas = dupload(m->h_alphas.data(), m->h_alphas.size(), c->stream);
    int* bad = dalloc<int>(1);
    ck(cudaMemsetAsync(bad, 0, sizeof(int), c->stream), "split32");
    launch_vals_to32(c->stream, cnt, m->vals, s->vals, bad);
    int hb = 0;
    ck(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "split32");
    ck(cudaStreamSynchronize(c->stream), "split32");
    dfree(bad);
    if (hb) {
      dfree(s->vals);
      dfree(s->alphas);
      delete s;
      fail(IGM_OVERFLOW_ERROR, "split32: a component value does not fit in int32");
    }
    *out = s;
  });
}

void igm_split32_free(igm_split32* m) {
  if (!m) return;
  cudaDeviceSynchronize();
  dfree(m->vals);
  dfree(m->alphas);
  if (m->own_pattern) {
    dfree(m->row_ptr);
    dfree(m->col_idx);
  }
  dfree(m->ws.basis);
  dfree(m->ws.w);
  dfree(m->ws.small);
  dfree(m->ws.y);
  dfree(m->ws.wts);
  delete m;
}

// The builder's plan.  Magnitudes in bits,
// worst case: a basis word may be O(1) (later Krylov vectors of config 3
// concentrate on few rows), v < 2^f; w = A v ~ 2^(alpha + 2) v; h ~ |w| 2^f ~
// 2^(f + alpha + 1); a sum of n terms needs L = log2(n)/2 bits of headroom.
igm_status igm_shifts32_plan(long long n, int alpha_a, int f, igm_shifts* out) {
  return guarded([&] {
    if (!out || n < 1) fail(IGM_INVALID_ARGUMENT, "shifts32_plan: bad argument");
    const double L = std::log2(static_cast<double>(n)) / 2;
    const double bv = f, bw = bv + alpha_a + 2, bh = f + alpha_a + 1;
    auto clampf = [&](double v, int hi) { return static_cast<int>(std::max(0.0, std::min(static_cast<double>(hi), v))); };
    const double need = bw + bv + L + 2 - 30;  // a sum of n dot terms in 30 bits
    const int b2 = clampf(std::floor(std::ceil(need - (bw - bv)) / 2), f - 1);
    const int b1 = clampf(std::ceil(need - b2), f - 1);
    igm_shifts p{};
    p.dot_b1 = b1;
    p.dot_b2 = b2;
    p.axpy_b1 = clampf(std::ceil(bh + bv - 30), f - 1);                    // (h >> b1) v in 30 bits
    p.norm_b1 = clampf(std::max(static_cast<double>(f - 15), std::ceil(f - (29 - 2.0 * (alpha_a + 1)) / 2)), f - 1);
    p.div_b1 = clampf(30 - bh, f);                                          // Givens: h << b1 in 30 bits
    p.div_b2 = clampf(std::min(static_cast<double>(f - p.div_b1), bh - 16), f - 1);  // 16 bits of divisor
    p.givens_b2 = clampf(std::ceil(bh + f + 1 - 30), f - 1);               // c (h >> b2) in 31 bits
    p.rot_b = std::max(0, f - 15);                                         // c g, s g in 30 bits
    *out = p;
  });
}

igm_status igm_run_cycle32(igm_ctx* c, const igm_split32* mc, const igm_cycle32_cfg* cfg, const double* b,
                           double* x_out, int* dim, double* r0_norm, int32_t* basis, int* n_basis, int32_t* hess,
                           int32_t* g, int32_t* cos_raw, int32_t* sin_raw, uint64_t* overflows) {
  return guarded([&] {
    need_ctx(c);
    if (!mc || !cfg || !b) fail(IGM_INVALID_ARGUMENT, "run_cycle32: null argument");
    if (cfg->m < 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
    if (cfg->s < 0 || cfg->s > mc->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
    validate_shifts32(cfg->shifts, cfg->frac_bits);
    auto* m = const_cast<igm_split32*>(mc);
    const long long n = m->n;
    const int M = cfg->m;
    ws_ensure(c, n, 1);
    cudaStream_t st = c->stream;
    In<double> db(b, n, st, c->ws.b);
    reset_ctl(c);
    const int d = cycle32(c, m, *cfg, db.d, 0, c->ws.x);
    if (dim) *dim = d;
    if (r0_norm) *r0_norm = c->h_ctl->r0n;
    if (n_basis) *n_basis = c->h_ctl->r0n == 0.0 ? 0 : c->h_ctl->nbasis;
    if (x_out) {
      if (d > 0) ck(cudaMemcpyAsync(x_out, c->ws.x, sizeof(double) * n, cudaMemcpyDefault, st), "x");
      else ck(cudaMemsetAsync(x_out, 0, 0, st), "x");  // x0 = 0: nothing to add
    }
    const int nb = c->h_ctl->r0n == 0.0 ? 0 : c->h_ctl->nbasis;
    if (basis && nb) ck(cudaMemcpyAsync(basis, m->ws.basis, sizeof(int32_t) * nb * n, cudaMemcpyDefault, st), "basis");
    if (hess) ck(cudaMemcpyAsync(hess, m->ws.hess, sizeof(int32_t) * (M + 1) * M, cudaMemcpyDefault, st), "hess");
    if (g) ck(cudaMemcpyAsync(g, m->ws.g, sizeof(int32_t) * (M + 1), cudaMemcpyDefault, st), "g");
    if (cos_raw) ck(cudaMemcpyAsync(cos_raw, m->ws.cs, sizeof(int32_t) * M, cudaMemcpyDefault, st), "cos");
    if (sin_raw) ck(cudaMemcpyAsync(sin_raw, m->ws.sn, sizeof(int32_t) * M, cudaMemcpyDefault, st), "sin");
    ck(cudaStreamSynchronize(st), "sync");
    if (x_out && d == 0 && !is_device_ptr(x_out)) std::fill(x_out, x_out + n, 0.0);
    bool inexact = false;
    const u64 ov = cycle32_overflows(c, m, M, &inexact);
    if (overflows) *overflows = ov;
  });
}

igm_status igm_solve32(igm_ctx* c, const igm_split32* mc, const igm_csrf* a_fp, const double* b, double tol,
                       int max_refinements, const igm_cycle32_cfg* cfg, double* x_out, igm_report* rep) {
  return guarded([&] {
    need_ctx(c);
    if (!mc || !a_fp || !b || !cfg || !rep) fail(IGM_INVALID_ARGUMENT, "solve32: null argument");
    if (a_fp->n != mc->n) fail(IGM_INVALID_ARGUMENT, "solve: dimension mismatch");
    if (max_refinements < 0) fail(IGM_INVALID_ARGUMENT, "solve: max_refinements must be >= 0");
    if (cfg->m < 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
    if (cfg->s < 0 || cfg->s > mc->ncomp - 1) fail(IGM_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
    validate_shifts32(cfg->shifts, cfg->frac_bits);
    auto* m = const_cast<igm_split32*>(mc);
    const auto t0 = std::chrono::steady_clock::now();
    const long long n = m->n;
    ws_ensure(c, n, 1);
    Work& w = c->ws;
    cudaStream_t st = c->stream;
    rep->converged = 0;
    rep->refinements = 0;
    rep->total_inner_iterations = 0;
    rep->n_relres = 0;
    rep->overflow_total = 0;
    rep->overflow_exact = 1;
    In<double> db(b, n, st, w.b);
    ck(cudaMemsetAsync(w.x, 0, sizeof(double) * n, st), "x=0");
    reset_ctl(c);
    launch_norm2_serial(st, n, db.d, nullptr, c->ctl, 1, n2_scratch(c, n));  // ||b||
    launch_residual(st, *a_fp, w.x, db.d, w.r, c->ctl, true);
    launch_norm2_serial(st, n, w.r, nullptr, c->ctl, 2, n2_scratch(c, n));
    ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
    ck(cudaStreamSynchronize(st), "sync");
    double relnorm = c->h_ctl->relnorm;
    rep->relres_history[rep->n_relres++] = relnorm;
    for (int k = 0; k < max_refinements && relnorm >= tol; ++k) {
      const u64 rbits = c->h_ctl->rmax_bits;
      double rmax;
      std::memcpy(&rmax, &rbits, sizeof rmax);
      if (rmax == 0.0) break;
      launch_scale_div(st, n, w.r, w.r0, c->ctl);  // b_k = r / gamma (refine.cpp:53-56)
      const int dim = cycle32(c, m, *cfg, w.r0, 1, w.x);
      bool inexact = false;
      const u64 ov = cycle32_overflows(c, m, cfg->m, &inexact);
      if (inexact) rep->overflow_exact = 0;
      if (dim == 0) break;
      ck(cudaMemsetAsync(&c->ctl->rmax_bits, 0, sizeof(u64), st), "rmax reset");
      launch_residual(st, *a_fp, w.x, db.d, w.r, c->ctl, true);
      launch_norm2_serial(st, n, w.r, nullptr, c->ctl, 2, n2_scratch(c, n));
      ck(cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st), "ctl");
      ck(cudaStreamSynchronize(st), "sync");
      rep->refinements = k + 1;
      rep->total_inner_iterations += dim;
      rep->inner_dims[k] = dim;
      rep->gamma_history[k] = rmax;
      rep->overflow_per_restart[k] = ov;
      rep->overflow_total += ov;
      relnorm = c->h_ctl->relnorm;
      rep->relres_history[rep->n_relres++] = relnorm;
    }
    rep->converged = relnorm < tol;
    if (x_out) ck(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n, cudaMemcpyDefault, st), "x");
    ck(cudaStreamSynchronize(st), "sync");
    rep->wall_time_sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}
