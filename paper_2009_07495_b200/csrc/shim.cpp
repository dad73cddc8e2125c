// shim.cpp -- the reference's C++ API (namespace intgmres, include/intgmres/)
// implemented over the C ABI of include/igm.h.
//
// Hot-path calls (spmv, apply_inverse[_fp], fx_dot/norm/axpy_sub, spmv_fp,
// norm2, residual_fp, gamma_scale, run_cycle, solve) marshal the
// std::vector-based reference types into device uploads and run on the B200.
// There is no CPU fallback: if no GPU is usable they throw.  Scalar Q-format
// helpers, Givens application on one column, the Hessenberg back substitution
// and the one-time setup (row scaling, splitting, ILU(0) + cast) are host C++
// exactly as in the reference (they are O(m) scalars or setup).
#include "intgmres/fxp.hpp"
#include "intgmres/csr.hpp"
#include "intgmres/split.hpp"
#include "intgmres/ilu.hpp"
#include "intgmres/gmres_int.hpp"
#include "intgmres/refine.hpp"
#include "igm.h"

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <future>
#include <memory>
#include <string>
#include <thread>

void igm_internal_set_error(const std::string& msg);

namespace intgmres {
namespace {

[[noreturn]] void rethrow(igm_status s) {
  const std::string m = igm_last_error();
  switch (s) {
    case IGM_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case IGM_DOMAIN_ERROR: throw std::domain_error(m);
    case IGM_OVERFLOW_ERROR: throw std::overflow_error(m);
    case IGM_LOGIC_ERROR: throw std::logic_error(m);
    case IGM_RUNTIME_ERROR: throw std::runtime_error(m);
    default: throw std::runtime_error("B200 device error: " + m);
  }
}

void ok(igm_status s) {
  if (s != IGM_OK) rethrow(s);
}

// one context per host thread (the reference API is single-threaded)
igm_ctx* ctx() {
  struct Holder {
    igm_ctx* c = nullptr;
    ~Holder() {
      if (c) igm_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) {
    const char* dev = std::getenv("IGM_DEVICE");
    ok(igm_ctx_create(dev ? std::atoi(dev) : 0, &h.c));
    // exact running-sum overflow events: opt-in, the
    // reference API has no switch for it
    const char* ex = std::getenv("IGM_EXACT_OVERFLOW");
    if (ex && std::atoi(ex) != 0) ok(igm_set_exact_overflow_counts(h.c, 1));
  }
  return h.c;
}

const char* kKernelNames[] = {"",       "spmv",   "precond", "dot",        "axpy",      "norm",
                              "vec_div", "givens", "givens_norm", "givens_div", "rot"};
const char* kOpNames[] = {"", "add", "sub", "mul", "shl", "div"};

// FxTrace <-> igm_trace bridge for one call.
struct TraceBridge {
  FxTrace* t;
  igm_trace d{};
  std::vector<int32_t> ev, sh;
  explicit TraceBridge(FxTrace* tr, std::size_t shift_cap = 0) : t(tr) {
    if (!t) return;
    d.checked = t->checked();
    d.record_shifts = t->records_shifts();
    d.kernel = -1;  // "the trace's current kernel"
    d.restart = t->restart();
    d.step = t->step();
    const std::size_t room = FxTrace::max_events - std::min(FxTrace::max_events, t->events.size());
    ev.resize(4 * room + 4);
    d.events = ev.data();
    d.cap_events = static_cast<int>(room);
    if (d.record_shifts) {
      sh.resize(3 * shift_cap + 3);
      d.shifts = sh.data();
      d.cap_shifts = static_cast<int>(shift_cap);
    }
    d.exact = 1;
  }
  igm_trace* ptr() { return t ? &d : nullptr; }
  std::string kname(int id) const {
    return (id >= 0 && id < 11) ? std::string(kKernelNames[id]) : std::string(t->kernel());
  }
  void flush() {
    if (!t) return;
    for (int i = 0; i < d.n_events; ++i) {
      const int32_t* e = ev.data() + 4 * i;
      t->add_overflows(kname(e[0]), kOpNames[e[1] >= 0 && e[1] < 6 ? e[1] : 0], e[2], e[3], 1);
    }
    if (d.total > static_cast<uint64_t>(d.n_events)) bump_rest(d.total - d.n_events);
    const long long ns = std::min<long long>(d.n_shifts, d.cap_shifts);
    for (long long i = 0; i < ns; ++i) {
      const int32_t* s = sh.data() + 3 * i;
      t->add_shift(kname(s[0]), s[1], s[2]);
    }
    t->set_exact(d.exact != 0);
  }
  // events beyond the device buffer: counted, never listed (the reference
  // caps its list at max_events anyway)
  void bump_rest(uint64_t n) {
    const std::size_t keep = t->events.size();
    t->add_overflows("", "", 0, 0, n);
    t->events.resize(keep);
  }
};

igm_shifts to_c(const ShiftPlan& p) {
  return igm_shifts{p.dot_b1, p.dot_b2, p.axpy_b1, p.norm_b1, p.div_b1, p.div_b2, p.givens_b2, p.rot_b};
}

// RAII device uploads of the reference containers
struct SplitUp {
  igm_split* h = nullptr;
  explicit SplitUp(const SplitMatrix& m) {
    if (m.components.empty()) throw std::invalid_argument("SplitMatrix has no components");
    const CsrMatrixI& c0 = m.components[0];
    const std::size_t nnz = c0.col_idx.size();
    std::vector<int64_t> vals(nnz * m.components.size());
    for (std::size_t l = 0; l < m.components.size(); ++l) {
      if (m.components[l].vals.size() != nnz) throw std::invalid_argument("SplitMatrix: components differ in size");
      std::memcpy(vals.data() + l * nnz, m.components[l].vals.data(), nnz * sizeof(int64_t));
    }
    std::vector<int> alphas(m.alphas);
    alphas.resize(m.components.size(), 0);
    ok(igm_upload_split(ctx(), m.n, static_cast<int>(nnz), c0.row_ptr.data(), c0.col_idx.data(),
                        static_cast<int>(m.components.size()), vals.data(), alphas.data(), &h));
  }
  ~SplitUp() { igm_split_free(h); }
};

struct CsrfUp {
  igm_csrf* h = nullptr;
  explicit CsrfUp(const CsrMatrixF& a) {
    ok(igm_upload_csrf(ctx(), a.n, a.row_ptr.data(), a.col_idx.data(), a.vals.data(), &h));
  }
  ~CsrfUp() { igm_csrf_free(h); }
};

struct IluUp {
  igm_ilu* h = nullptr;
  explicit IluUp(const IluFactors& f) {
    ok(igm_upload_ilu(ctx(), f.lower.n, f.lower.row_ptr.data(), f.lower.col_idx.data(),
                      f.lower.vals.data(), f.diag_pos_lower.data(), f.upper.row_ptr.data(),
                      f.upper.col_idx.data(), f.upper.vals.data(), f.diag_pos_upper.data(), &h));
  }
  ~IluUp() { igm_ilu_free(h); }
};

// ---- verified operator cache --------------------------------------------
// Repeated intgmres::solve / run_cycle calls on unchanged operators would
// re-upload (and rebuild the wavefront schedules and pencil streams of)
// several hundred MB per call.  An upload is reused when every array has the
// same address and size AND the same content fingerprint: a 64-bit
// multiply-xorshift hash of every byte, computed on host threads (the
// reference containers are plain std::vectors, so nothing else tells a
// mutated operator apart).  IGM_OPCACHE=0 disables it.
struct Span {
  const void* p;
  std::size_t n;
  bool operator==(const Span& o) const { return p == o.p && n == o.n; }
};

std::uint64_t hash_chunk(const unsigned char* p, std::size_t n, std::uint64_t seed) {
  constexpr std::uint64_t K = 0x9E3779B97F4A7C15ull;
  std::uint64_t h[4] = {seed, seed ^ 0x243F6A8885A308D3ull, seed ^ 0x13198A2E03707344ull, seed ^ 0xA4093822299F31D0ull};
  std::size_t i = 0;
  for (; i + 32 <= n; i += 32) {
    std::uint64_t w[4];
    std::memcpy(w, p + i, 32);
    for (int k = 0; k < 4; ++k) {
      h[k] = (h[k] ^ w[k]) * K;
      h[k] ^= h[k] >> 29;
    }
  }
  if (i < n) {  // the < 32 tail bytes, zero padded
    std::uint64_t w[4] = {0, 0, 0, 0};
    std::memcpy(w, p + i, n - i);
    for (int k = 0; k < 4; ++k) {
      h[k] = (h[k] ^ w[k]) * K;
      h[k] ^= h[k] >> 29;
    }
  }
  std::uint64_t r = (h[0] ^ (h[1] << 1) ^ (h[2] << 2) ^ (h[3] << 3) ^ n) * K;
  return r ^ (r >> 31);
}

std::uint64_t fingerprint(const std::vector<Span>& spans) {
  constexpr std::size_t kChunk = std::size_t{8} << 20;
  struct Job {
    const unsigned char* p;
    std::size_t n;
  };
  std::vector<Job> jobs;
  for (const Span& s : spans)
    for (std::size_t o = 0; o < s.n; o += kChunk)
      jobs.push_back({static_cast<const unsigned char*>(s.p) + o, std::min(kChunk, s.n - o)});
  std::vector<std::uint64_t> out(jobs.size());
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned nt = static_cast<unsigned>(std::min<std::size_t>(hw, jobs.size()));
  auto work = [&](unsigned t) {
    for (std::size_t j = t; j < jobs.size(); j += nt) out[j] = hash_chunk(jobs[j].p, jobs[j].n, 0x5851F42D4C957F2Dull + j);
  };
  if (nt <= 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  std::uint64_t h = 0xCBF29CE484222325ull ^ spans.size();
  for (std::uint64_t v : out) h = (h ^ v) * 0x100000001B3ull;
  return h;
}

template <class T>
Span span_of(const std::vector<T>& v) {
  return Span{v.data(), v.size() * sizeof(T)};
}

std::vector<Span> spans_of(const SplitMatrix& m) {
  std::vector<Span> s{Span{nullptr, static_cast<std::size_t>(m.n)}, span_of(m.alphas)};
  for (const CsrMatrixI& c : m.components) {
    s.push_back(span_of(c.row_ptr));
    s.push_back(span_of(c.col_idx));
    s.push_back(span_of(c.vals));
  }
  return s;
}
std::vector<Span> spans_of(const CsrMatrixF& a) {
  return {Span{nullptr, static_cast<std::size_t>(a.n)}, span_of(a.row_ptr), span_of(a.col_idx), span_of(a.vals)};
}
std::vector<Span> spans_of(const IluFactors& f) {
  return {Span{nullptr, static_cast<std::size_t>(f.lower.n)}, span_of(f.lower.row_ptr), span_of(f.lower.col_idx),
          span_of(f.lower.vals), span_of(f.diag_pos_lower), span_of(f.upper.row_ptr), span_of(f.upper.col_idx),
          span_of(f.upper.vals), span_of(f.diag_pos_upper)};
}

bool opcache_on() {
  static const bool on = [] {
    const char* e = std::getenv("IGM_OPCACHE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

// the cached upload of `obj` (one entry per operator type and host thread).
// When the addresses and sizes match the cached entry, the upload is handed
// out at once and `pending` receives the fingerprint job: the caller runs its
// GPU work on the cached copy while host threads verify the content, and
// repeats the work on a fresh upload if the verification fails (solve()).
struct PendingCheck {
  std::vector<Span> data;
  std::uint64_t want = 0;
  bool active = false;
};
template <class Up>
struct CacheEntry {
  std::vector<Span> key;
  std::uint64_t fp = 0;
  std::unique_ptr<Up> up;
};
template <class Up>
CacheEntry<Up>& cache_entry() {
  thread_local CacheEntry<Up> e;
  return e;
}
template <class Up, class Obj>
Up& cached_upload(const Obj& obj, std::unique_ptr<Up>& fresh, PendingCheck* pending = nullptr) {
  CacheEntry<Up>& e = cache_entry<Up>();
  if (!opcache_on()) {
    fresh = std::make_unique<Up>(obj);
    return *fresh;
  }
  std::vector<Span> key = spans_of(obj);
  std::vector<Span> data(key.begin() + 1, key.end());  // the n pseudo-span carries no bytes
  if (pending != nullptr && e.up && e.key == key) {  // same arrays: verify the content concurrently
    pending->data = std::move(data);
    pending->want = e.fp;
    pending->active = true;
    return *e.up;
  }
  const std::uint64_t fp = fingerprint(data);
  if (!e.up || !(e.key == key) || e.fp != fp) {
    e.up.reset();  // free the old upload first
    e.up = std::make_unique<Up>(obj);
    e.key = std::move(key);
    e.fp = fp;
  }
  return *e.up;
}
// a failed verification: the entry no longer describes the host arrays
template <class Up>
void cache_drop() {
  CacheEntry<Up>& e = cache_entry<Up>();
  e.up.reset();
  e.key.clear();
}

inline double absmax_update(double acc, double v) {
  const double a = std::fabs(v);
  return acc < a ? a : acc;  // std::max(acc, a)
}

}  // namespace

// ===========================================================================
// fxp (fxp.hpp / fxp.cpp)

FxScalar encode(double x, QFormat fmt) {
  if (!(std::fabs(x) < std::ldexp(1.0, fmt.int_bits())))
    throw std::overflow_error("encode: value outside representable range");
  return FxScalar{static_cast<std::int64_t>(std::ldexp(x, fmt.frac_bits())), fmt};
}

double decode(const FxScalar& a) { return std::ldexp(static_cast<double>(a.raw), -a.fmt.frac_bits()); }

FxVector encode_vector(const std::vector<double>& x, QFormat fmt) {
  FxVector v(x.size(), fmt);
  for (std::size_t i = 0; i < x.size(); ++i) v.raw[i] = encode(x[i], fmt).raw;
  return v;
}

std::vector<double> decode_vector(const FxVector& v) {
  std::vector<double> x(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) x[i] = decode(FxScalar{v.raw[i], v.fmt});
  return x;
}

FxScalar fx_add(const FxScalar& a, const FxScalar& b, FxTrace* t) {
  detail::require_same_format(a.fmt, b.fmt, "fx_add");
  return FxScalar{detail::add_checked(a.raw, b.raw, t), a.fmt};
}

FxScalar fx_sub(const FxScalar& a, const FxScalar& b, FxTrace* t) {
  detail::require_same_format(a.fmt, b.fmt, "fx_sub");
  return FxScalar{detail::sub_checked(a.raw, b.raw, t), a.fmt};
}

FxScalar fx_mul(const FxScalar& a, const FxScalar& b, int b1, int b2, int out_frac, FxTrace* t) {
  detail::require_same_format(a.fmt, b.fmt, "fx_mul");
  detail::require_shift_range(b1, "fx_mul");
  detail::require_shift_range(b2, "fx_mul");
  const QFormat out(out_frac);
  const int post = 2 * a.fmt.frac_bits() - b1 - b2 - out_frac;
  if (post < 0) throw std::invalid_argument("fx_mul: shifts exceed available precision");
  if (t) t->record_shift(b1, b2);
  const std::int64_t p = detail::mul_checked(detail::asr(a.raw, b1), detail::asr(b.raw, b2), t);
  return FxScalar{detail::asr(p, post), out};
}

FxScalar fx_div(const FxScalar& a, const FxScalar& b, int b1, int b2, FxTrace* t) {
  detail::require_same_format(a.fmt, b.fmt, "fx_div");
  detail::require_shift_range(b1, "fx_div");
  detail::require_shift_range(b2, "fx_div");
  if (t) t->record_shift(b1, b2);
  const std::int64_t num = detail::shl_checked(a.raw, b1, t);
  const std::int64_t den = detail::asr(b.raw, b2);
  if (den == 0) throw std::domain_error("fx_div: shifted divisor is zero");
  const std::int64_t q = detail::div_trunc_checked(num, den, t);
  const int e = a.fmt.frac_bits() - b1 - b2;
  return FxScalar{e >= 0 ? detail::shl_checked(q, e, t) : detail::asr(q, -e), a.fmt};
}

std::uint64_t isqrt(std::uint64_t v) {
  // floor(sqrt(v)): FP estimate then exact integer correction
  if (v == 0) return 0;
  std::uint64_t r = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(v)));
  while (r > 0 && static_cast<unsigned __int128>(r) * r > v) --r;
  while (static_cast<unsigned __int128>(r + 1) * (r + 1) <= v) ++r;
  return r;
}

FxScalar fx_sqrt(const FxScalar& a, int out_frac, FxTrace* t) {
  if (a.raw < 0) throw std::domain_error("fx_sqrt: negative input");
  const int fin = a.fmt.frac_bits();
  if (fin % 2 != 0) throw std::invalid_argument("fx_sqrt: input frac_bits must be even");
  const QFormat out(out_frac);
  const auto r = static_cast<std::int64_t>(isqrt(static_cast<std::uint64_t>(a.raw)));
  const int e = out_frac - fin / 2;
  return FxScalar{e >= 0 ? detail::shl_checked(r, e, t) : detail::asr(r, -e), out};
}

FxScalar fx_dot(const FxVector& v, const FxVector& w, int b1, int b2, FxTrace* t) {
  detail::require_same_format(v.fmt, w.fmt, "fx_dot");
  detail::require_shift_range(b1, "fx_dot");
  detail::require_shift_range(b2, "fx_dot");
  if (v.size() != w.size()) throw std::invalid_argument("fx_dot: length mismatch");
  TraceBridge tb(t, 1);
  std::int64_t out = 0;
  const igm_status s = igm_fx_dot(ctx(), static_cast<int64_t>(v.size()), v.raw.data(), w.raw.data(),
                                  v.fmt.frac_bits(), b1, b2, &out, tb.ptr());
  tb.flush();
  ok(s);
  return FxScalar{out, v.fmt};
}

FxScalar fx_norm(const FxVector& v, int b1, FxTrace* t) {
  TraceBridge tb(t, 1);
  std::int64_t out = 0;
  const igm_status s = igm_fx_norm(ctx(), static_cast<int64_t>(v.size()), v.raw.data(),
                                   v.fmt.frac_bits(), b1, &out, tb.ptr());
  tb.flush();
  ok(s);
  return FxScalar{out, v.fmt};
}

void fx_axpy_sub(FxVector& w, const FxScalar& h, const FxVector& v, int b1, FxTrace* t) {
  detail::require_same_format(w.fmt, v.fmt, "fx_axpy_sub");
  detail::require_same_format(w.fmt, h.fmt, "fx_axpy_sub");
  detail::require_shift_range(b1, "fx_axpy_sub");
  if (v.size() != w.size()) throw std::invalid_argument("fx_axpy_sub: length mismatch");
  TraceBridge tb(t, 1);
  const igm_status s = igm_fx_axpy_sub(ctx(), static_cast<int64_t>(w.size()), w.raw.data(), h.raw,
                                       v.raw.data(), w.fmt.frac_bits(), b1, tb.ptr());
  tb.flush();
  ok(s);
}

void ShiftPlan::validate(QFormat fmt) const {
  const int f = fmt.frac_bits();
  auto right = [f](int b, const char* name) {
    if (b < 0 || (b > 0 && b >= f))
      throw std::invalid_argument(std::string("ShiftPlan: ") + name + " must lie in [0, frac_bits)");
  };
  right(dot_b1, "dot_b1");
  right(dot_b2, "dot_b2");
  right(axpy_b1, "axpy_b1");
  right(norm_b1, "norm_b1");
  right(div_b2, "div_b2");
  right(givens_b2, "givens_b2");
  if (div_b1 < 0 || div_b1 > f) throw std::invalid_argument("ShiftPlan: div_b1 must lie in [0, frac_bits]");
  if (rot_b != 0) throw std::invalid_argument("ShiftPlan: rot_b must be 0");
  if (2 * (f - norm_b1) > 62)
    throw std::invalid_argument("ShiftPlan: norm accumulator needs 2*(frac_bits - norm_b1) <= 62");
}

ShiftPlan ShiftPlan::default_unpreconditioned(QFormat fmt) {
  // Table IV presets: 16-bit guard shifts for ~2^16 row-scaled operands
  ShiftPlan p;
  p.dot_b1 = p.axpy_b1 = p.norm_b1 = p.div_b1 = p.givens_b2 = 16;
  p.div_b2 = fmt.frac_bits() - 16;
  p.validate(fmt);
  return p;
}

ShiftPlan ShiftPlan::default_preconditioned(QFormat fmt) {
  ShiftPlan p;  // Table VI: no destructive shifts, dividend pre-shift f
  p.div_b1 = fmt.frac_bits();
  p.validate(fmt);
  return p;
}

// ===========================================================================
// csr (csr.hpp)

CsrMatrixF from_triplets(int n, std::vector<std::tuple<int, int, double>> t) {
  for (const auto& e : t) {
    const int i = std::get<0>(e), j = std::get<1>(e);
    if (i < 0 || i >= n || j < 0 || j >= n) throw std::invalid_argument("from_triplets: index out of range");
  }
  std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                            : std::get<1>(a) < std::get<1>(b);
  });
  CsrMatrixF m;
  m.n = n;
  m.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (std::size_t k = 0; k < t.size(); ++k) {
    const auto& [i, j, v] = t[k];
    const bool dup = k > 0 && std::get<0>(t[k - 1]) == i && std::get<1>(t[k - 1]) == j;
    if (dup) {
      m.vals.back() += v;
    } else {
      m.col_idx.push_back(j);
      m.vals.push_back(v);
      ++m.row_ptr[i + 1];
    }
  }
  for (int i = 0; i < n; ++i) m.row_ptr[i + 1] += m.row_ptr[i];
  return m;
}

std::vector<double> spmv_fp(const CsrMatrixF& a, const std::vector<double>& x) {
  if (static_cast<int>(x.size()) != a.n) throw std::invalid_argument("spmv_fp: dimension mismatch");
  CsrfUp up(a);
  std::vector<double> y(static_cast<std::size_t>(a.n));
  ok(igm_spmv_fp(ctx(), up.h, x.data(), y.data()));
  return y;
}

double norm2(const std::vector<double>& v) {
  double r = 0.0;
  ok(igm_norm2(ctx(), static_cast<int64_t>(v.size()), v.data(), &r));
  return r;
}

Residual residual_fp(const CsrMatrixF& a, const std::vector<double>& x, const std::vector<double>& b) {
  if (static_cast<int>(x.size()) != a.n || static_cast<int>(b.size()) != a.n)
    throw std::invalid_argument("residual_fp: dimension mismatch");
  CsrfUp up(a);
  Residual res;
  res.r.resize(static_cast<std::size_t>(a.n));
  ok(igm_residual_fp(ctx(), up.h, x.data(), b.data(), res.r.data(), &res.relnorm));
  return res;
}

// ===========================================================================
// split (split.hpp): setup on the host, SpMV on the GPU

RowScaled row_scale(const CsrMatrixF& a, int alpha_a) {
  RowScaled rs;
  rs.a = a;
  rs.scale.assign(static_cast<std::size_t>(a.n), 0.0);
  ok(igm_row_scale(a.n, a.row_ptr.data(), a.col_idx.data(), a.vals.data(), alpha_a, rs.a.vals.data(),
                   rs.scale.data()));
  return rs;
}

std::vector<double> scale_rhs(const std::vector<double>& b, const std::vector<double>& scale) {
  if (b.size() != scale.size()) throw std::invalid_argument("scale_rhs: length mismatch");
  std::vector<double> out(b.size());
  for (std::size_t i = 0; i < b.size(); ++i) out[i] = b[i] / scale[i];
  return out;
}

SplitMatrix build_split(const CsrMatrixF& a, int alpha_a, int max_components, std::vector<double> scale_diag) {
  if (max_components < 1) throw std::invalid_argument("build_split: need at least one component");
  const int nnz = static_cast<int>(a.vals.size());
  std::vector<int64_t> comp(static_cast<std::size_t>(nnz) * max_components);
  std::vector<int> alphas(static_cast<std::size_t>(max_components));
  int ncomp = 0, exact = 0;
  ok(igm_build_split(a.n, nnz, a.vals.data(), alpha_a, max_components, comp.data(), alphas.data(), &ncomp,
                     &exact));
  SplitMatrix m;
  m.n = a.n;
  m.alpha_a = alpha_a;
  m.scale_diag = std::move(scale_diag);
  m.exact = exact != 0;
  for (int l = 0; l < ncomp; ++l) {
    CsrMatrixI c;
    c.n = a.n;
    c.row_ptr = a.row_ptr;
    c.col_idx = a.col_idx;
    c.vals.assign(comp.begin() + static_cast<std::ptrdiff_t>(l) * nnz,
                  comp.begin() + static_cast<std::ptrdiff_t>(l + 1) * nnz);
    m.components.push_back(std::move(c));
    m.alphas.push_back(alphas[l]);
  }
  return m;
}

FxVector spmv(const SplitMatrix& m, int s, const FxVector& v, FxTrace* t) {
  if (s < 0 || s > m.depth()) throw std::invalid_argument("spmv: component index out of range");
  if (static_cast<int>(v.size()) != m.n) throw std::invalid_argument("spmv: dimension mismatch");
  SplitUp up(m);
  FxVector out(static_cast<std::size_t>(m.n), v.fmt);
  TraceBridge tb(t);
  const igm_status st = igm_spmv(ctx(), up.h, s, v.raw.data(), out.raw.data(), tb.ptr());
  tb.flush();
  ok(st);
  return out;
}

std::vector<double> spmv_fp(const SplitMatrix& m, int s, const std::vector<double>& x) {
  if (s < 0 || s > m.depth()) throw std::invalid_argument("spmv_fp: component index out of range");
  if (static_cast<int>(x.size()) != m.n) throw std::invalid_argument("spmv_fp: dimension mismatch");
  SplitUp up(m);
  std::vector<double> y(static_cast<std::size_t>(m.n));
  ok(igm_spmv_fp_split(ctx(), up.h, s, x.data(), y.data()));
  return y;
}

CsrMatrixF reconstruct_fp(const SplitMatrix& m, int s) {
  if (s < 0 || s > m.depth()) throw std::invalid_argument("reconstruct_fp: component index out of range");
  CsrMatrixF a;
  a.n = m.n;
  a.row_ptr = m.components[0].row_ptr;
  a.col_idx = m.components[0].col_idx;
  a.vals.assign(m.components[0].vals.size(), 0.0);
  for (int l = 0; l <= s; ++l)
    for (std::size_t k = 0; k < a.vals.size(); ++k)
      a.vals[k] += std::ldexp(static_cast<double>(m.components[l].vals[k]), -m.alphas[l]);
  return a;
}

// ===========================================================================
// ilu (ilu.hpp): factorisation on the host, substitutions on the GPU

namespace {
FpIluFactors ilu0_impl(const CsrMatrixF& a, double* merged_out);
}
FpIluFactors factorize_ilu0(const CsrMatrixF& a) { return ilu0_impl(a, nullptr); }

namespace {
// merged_out (nnz doubles, may be null): the merged L\U values on A's pattern
// before the split below (a z-slab rank hands its last plane's U rows to the
// next rank, dist.slab_ilu_local)
FpIluFactors ilu0_impl(const CsrMatrixF& a, double* merged_out) {
  const int n = a.n;
  std::vector<int> dpos(static_cast<std::size_t>(n), -1);
  for (int i = 0; i < n; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.col_idx[k] == i) dpos[i] = k;
  for (int i = 0; i < n; ++i)
    if (dpos[i] < 0)
      throw std::runtime_error("factorize_ilu0: row " + std::to_string(i) + " has no diagonal entry in the pattern");
  // IKJ elimination restricted to A's pattern, L\U merged in place
  std::vector<double> lu = a.vals;
  std::vector<int> slot(static_cast<std::size_t>(n), -1);
  for (int i = 0; i < n; ++i) {
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) slot[a.col_idx[k]] = k;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j >= i) break;
      lu[k] /= lu[dpos[j]];
      for (int kk = dpos[j] + 1; kk < a.row_ptr[j + 1]; ++kk) {
        const int at = slot[a.col_idx[kk]];
        if (at >= 0) lu[at] -= lu[k] * lu[kk];
      }
    }
    if (lu[dpos[i]] == 0.0) throw std::runtime_error("factorize_ilu0: zero pivot in row " + std::to_string(i));
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) slot[a.col_idx[k]] = -1;
  }
  if (merged_out) std::copy(lu.begin(), lu.end(), merged_out);
  FpIluFactors f;
  f.diag.resize(static_cast<std::size_t>(n));
  f.lower.n = f.upper.n = n;
  f.lower.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  f.upper.row_ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (int i = 0; i < n; ++i) {
    const double d = lu[dpos[i]];
    f.diag[i] = d;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j <= i) {
        f.lower.col_idx.push_back(j);
        f.lower.vals.push_back(j < i ? lu[k] : 1.0);
      }
      if (j >= i) {
        f.upper.col_idx.push_back(j);
        f.upper.vals.push_back(j > i ? lu[k] / d : 1.0);
      }
    }
    f.lower.row_ptr[i + 1] = static_cast<int>(f.lower.col_idx.size());
    f.upper.row_ptr[i + 1] = static_cast<int>(f.upper.col_idx.size());
  }
  return f;
}
}  // namespace

IluFactors split_cast(const FpIluFactors& f) {
  const int n = f.lower.n;
  IluFactors g;
  g.lower.n = g.upper.n = n;
  g.lower.row_ptr = f.lower.row_ptr;
  g.lower.col_idx = f.lower.col_idx;
  g.upper.row_ptr = f.upper.row_ptr;
  g.upper.col_idx = f.upper.col_idx;
  g.lower.vals.resize(f.lower.vals.size());
  g.upper.vals.resize(f.upper.vals.size());
  g.diag_pos_lower.assign(static_cast<std::size_t>(n), -1);
  g.diag_pos_upper.assign(static_cast<std::size_t>(n), -1);
  std::vector<double> dl(static_cast<std::size_t>(n)), du(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    dl[i] = std::sqrt(std::fabs(f.diag[i]));
    du[i] = f.diag[i] < 0 ? -dl[i] : dl[i];
  }
  for (int i = 0; i < n; ++i) {
    for (int k = f.lower.row_ptr[i]; k < f.lower.row_ptr[i + 1]; ++k) {
      const int j = f.lower.col_idx[k];
      g.lower.vals[k] = static_cast<std::int64_t>(f.lower.vals[k] * dl[j]);
      if (j == i) g.diag_pos_lower[i] = k;
    }
    for (int k = f.upper.row_ptr[i]; k < f.upper.row_ptr[i + 1]; ++k) {
      g.upper.vals[k] = static_cast<std::int64_t>(f.upper.vals[k] * du[i]);
      if (f.upper.col_idx[k] == i) g.diag_pos_upper[i] = k;
    }
  }
  for (int i = 0; i < n; ++i)
    if (g.lower.vals[g.diag_pos_lower[i]] == 0 || g.upper.vals[g.diag_pos_upper[i]] == 0)
      throw std::runtime_error("split_cast: diagonal entry of row " + std::to_string(i) +
                               " truncates to zero; scale the matrix up before factorizing");
  return g;
}

FxVector apply_inverse(const IluFactors& f, const FxVector& y, FxTrace* t) {
  if (static_cast<int>(y.size()) != f.lower.n) throw std::invalid_argument("apply_inverse: dimension mismatch");
  IluUp up(f);
  FxVector out(y.size(), y.fmt);
  TraceBridge tb(t);
  const igm_status s = igm_apply_inverse(ctx(), up.h, y.raw.data(), out.raw.data(), tb.ptr());
  tb.flush();
  ok(s);
  return out;
}

std::vector<double> apply_inverse_fp(const IluFactors& f, const std::vector<double>& y) {
  if (static_cast<int>(y.size()) != f.lower.n) throw std::invalid_argument("apply_inverse_fp: dimension mismatch");
  IluUp up(f);
  std::vector<double> out(y.size());
  ok(igm_apply_inverse_fp(ctx(), up.h, y.data(), out.data()));
  return out;
}

std::vector<double> apply_fp(const FpIluFactors& f, const std::vector<double>& y) {
  // FP64 baseline preconditioner on the unit factors (not the int path)
  const int n = f.lower.n;
  if (static_cast<int>(y.size()) != n) throw std::invalid_argument("apply_fp: dimension mismatch");
  std::vector<double> z(static_cast<std::size_t>(n)), w(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    double acc = y[i];
    for (int k = f.lower.row_ptr[i]; k < f.lower.row_ptr[i + 1]; ++k)
      if (f.lower.col_idx[k] != i) acc -= f.lower.vals[k] * z[f.lower.col_idx[k]];
    z[i] = acc;
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = z[i] / f.diag[i];
    for (int k = f.upper.row_ptr[i]; k < f.upper.row_ptr[i + 1]; ++k)
      if (f.upper.col_idx[k] != i) acc -= f.upper.vals[k] * w[f.upper.col_idx[k]];
    w[i] = acc;
  }
  return w;
}

// ===========================================================================
// gmres_int (gmres_int.hpp)

void apply_stored_rotations(std::int64_t* h, int count, const std::int64_t* c, const std::int64_t* s,
                            int givens_b2, QFormat fmt, FxTrace* t) {
  const int f = fmt.frac_bits();
  for (int i = 0; i < count; ++i) {
    const FxScalar ci{c[i], fmt}, si{s[i], fmt}, hi{h[i], fmt}, hn{h[i + 1], fmt};
    // (c h_i + s h_{i+1}, c h_{i+1} - s h_i), products in the reference order
    const FxScalar a = fx_mul(ci, hi, 0, givens_b2, f, t);
    const FxScalar b = fx_mul(si, hn, 0, givens_b2, f, t);
    const FxScalar d = fx_mul(ci, hn, 0, givens_b2, f, t);
    const FxScalar e = fx_mul(si, hi, 0, givens_b2, f, t);
    h[i] = fx_add(a, b, t).raw;
    h[i + 1] = fx_sub(d, e, t).raw;
  }
}

std::vector<double> solve_hessenberg(const std::vector<double>& r, int ld, int dim, const std::vector<double>& g) {
  std::vector<double> y(static_cast<std::size_t>(dim));
  for (int i = dim - 1; i >= 0; --i) {
    double acc = g[i];
    for (int j = i + 1; j < dim; ++j) acc -= r[static_cast<std::size_t>(j) * ld + i] * y[j];
    const double rii = r[static_cast<std::size_t>(i) * ld + i];
    if (rii == 0.0) throw std::runtime_error("solve_hessenberg: zero diagonal");
    y[i] = acc / rii;
  }
  return y;
}

CycleResult run_cycle(const SplitMatrix& m, const CycleConfig& cfg, const std::vector<double>& b,
                      const std::vector<double>& x0, FxTrace* trace, ArnoldiState* state_out) {
  const int n = m.n;
  if (cfg.m < 1) throw std::invalid_argument("run_cycle: m must be >= 1");
  if (static_cast<int>(b.size()) != n || static_cast<int>(x0.size()) != n)
    throw std::invalid_argument("run_cycle: dimension mismatch");
  if (cfg.s < 0 || cfg.s > m.depth()) throw std::invalid_argument("run_cycle: splitting depth out of range");
  cfg.shifts.validate(cfg.fmt);
  SplitUp up(m);
  std::unique_ptr<IluUp> pre;
  if (cfg.precond) pre = std::make_unique<IluUp>(*cfg.precond);
  const int M = cfg.m;
  igm_cycle_cfg cc{M, cfg.fmt.frac_bits(), cfg.s, to_c(cfg.shifts), pre ? pre->h : nullptr,
                   cfg.collect_basis_norms ? 1 : 0};
  CycleResult res;
  res.x.resize(static_cast<std::size_t>(n));
  std::vector<double> gabs(M), cd(M), sd(M), bn(M + 1);
  std::vector<int64_t> basis, hess(static_cast<std::size_t>(M + 1) * M), g(M + 1), cr(M), sr(M);
  if (state_out) basis.resize(static_cast<std::size_t>(M + 1) * n);
  igm_cycle_out co{};
  co.g_abs = gabs.data();
  co.cos_d = cd.data();
  co.sin_d = sd.data();
  co.basis_norms = bn.data();
  co.basis = state_out ? basis.data() : nullptr;
  co.hess = hess.data();
  co.g = g.data();
  co.cos_raw = cr.data();
  co.sin_raw = sr.data();
  const std::size_t shift_cap =
      trace && trace->records_shifts()
          ? static_cast<std::size_t>(M) * (2 * (M + 1) + static_cast<std::size_t>(n) + 4 * M + 8)
          : 0;
  TraceBridge tb(trace, shift_cap);
  const igm_status st = igm_run_cycle(ctx(), up.h, &cc, b.data(), x0.data(), res.x.data(), &co, tb.ptr());
  tb.flush();
  ok(st);
  res.diag.dim = co.dim;
  res.diag.r0_norm = co.r0_norm;
  if (co.r0_norm == 0.0) {
    res.x = x0;
    return res;  // nothing to correct (gmres_int.cpp:72-73); state untouched
  }
  res.diag.g_abs.assign(gabs.begin(), gabs.begin() + co.dim);
  res.diag.cos.assign(cd.begin(), cd.begin() + co.dim);
  res.diag.sin.assign(sd.begin(), sd.begin() + co.dim);
  if (cfg.collect_basis_norms) res.diag.basis_norms.assign(bn.begin(), bn.begin() + co.n_basis_norms);
  if (state_out) {
    state_out->basis.clear();
    for (int k = 0; k < co.n_basis; ++k) {
      FxVector v;
      v.fmt = cfg.fmt;
      v.raw.assign(basis.begin() + static_cast<std::ptrdiff_t>(k) * n,
                   basis.begin() + static_cast<std::ptrdiff_t>(k + 1) * n);
      state_out->basis.push_back(std::move(v));
    }
    state_out->hess = std::move(hess);
    state_out->ld = M + 1;
    state_out->g = std::move(g);
    state_out->cos_raw = std::move(cr);
    state_out->sin_raw = std::move(sr);
    state_out->fmt = cfg.fmt;
  }
  return res;
}

// ===========================================================================
// refine (refine.hpp)

GammaScaled gamma_scale(const std::vector<double>& r) {
  GammaScaled g;
  g.b_k.resize(r.size());
  ok(igm_gamma_scale(ctx(), static_cast<int64_t>(r.size()), r.data(), &g.gamma, g.b_k.data()));
  return g;
}

namespace {
int call_schedule(void* user, int k) { return (*static_cast<const std::function<int(int)>*>(user))(k); }
}  // namespace

SolveResult solve(const SplitMatrix& m, const CsrMatrixF& a_fp, const std::vector<double>& b,
                  const RefineConfig& cfg, const IluFactors* precond, FxTrace* external_trace) {
  const int n = m.n;
  if (a_fp.n != n || static_cast<int>(b.size()) != n) throw std::invalid_argument("solve: dimension mismatch");
  if (cfg.max_refinements < 0) throw std::invalid_argument("solve: max_refinements must be >= 0");
  const auto t0 = std::chrono::steady_clock::now();
  FxTrace own(cfg.checked, false);
  FxTrace* trace = external_trace ? external_trace : &own;
  std::unique_ptr<SplitUp> up_own;
  std::unique_ptr<CsrfUp> af_own;
  std::unique_ptr<IluUp> pre_own;
  // Operators whose arrays sit where the cached upload's did are used at once;
  // their content fingerprints are checked on host threads while the GPU
  // solves, and a mismatch (arrays mutated in place) repeats the solve on a
  // fresh upload before anything is returned or thrown.
  PendingCheck chk[3];
  SplitUp* up = &cached_upload(m, up_own, &chk[0]);
  CsrfUp* af = &cached_upload(a_fp, af_own, &chk[1]);
  IluUp* pre = precond ? &cached_upload(*precond, pre_own, &chk[2]) : nullptr;
  std::future<bool> verified;
  if (chk[0].active || chk[1].active || chk[2].active)
    verified = std::async(std::launch::async, [&chk] {
      bool same = true;
      for (const PendingCheck& c : chk)
        if (c.active && fingerprint(c.data) != c.want) same = false;
      return same;
    });
  const int R = cfg.max_refinements;
  igm_refine_cfg rc{};
  rc.tol = cfg.tol;
  rc.max_refinements = R;
  rc.m = cfg.m;
  rc.frac_bits = cfg.fmt.frac_bits();
  rc.s = cfg.s;
  rc.checked = cfg.checked ? 1 : 0;
  rc.shifts = to_c(cfg.shifts);
  rc.engine = cfg.engine == Engine::floating_point ? 1 : 0;
  if (cfg.s_schedule) {
    rc.s_schedule_fn = &call_schedule;
    rc.s_schedule_user = const_cast<std::function<int(int)>*>(&cfg.s_schedule);
  }
  std::vector<int> dims(R + 1);
  std::vector<double> relres(R + 2), gam(R + 1);
  std::vector<uint64_t> ovf(R + 1);
  igm_report rep{};
  rep.inner_dims = dims.data();
  rep.relres_history = relres.data();
  rep.gamma_history = gam.data();
  rep.overflow_per_restart = ovf.data();
  const std::size_t shift_cap =
      trace->records_shifts()
          ? static_cast<std::size_t>(R) * cfg.m * (2 * (cfg.m + 1) + static_cast<std::size_t>(n) + 4 * cfg.m + 8)
          : 0;
  SolveResult res;
  res.x.resize(static_cast<std::size_t>(n));
  std::unique_ptr<TraceBridge> tb = std::make_unique<TraceBridge>(trace, std::min<std::size_t>(shift_cap, 1u << 26));
  igm_status st =
      igm_solve(ctx(), up->h, af->h, b.data(), &rc, pre ? pre->h : nullptr, res.x.data(), &rep, tb->ptr());
  if (verified.valid() && !verified.get()) {
    // some operator changed under an unchanged address: drop the stale
    // uploads, upload again (fingerprinted synchronously) and solve again;
    // the first run touched neither the caller's trace nor anything returned
    if (chk[0].active) cache_drop<SplitUp>();
    if (chk[1].active) cache_drop<CsrfUp>();
    if (chk[2].active) cache_drop<IluUp>();
    up = &cached_upload(m, up_own);
    af = &cached_upload(a_fp, af_own);
    pre = precond ? &cached_upload(*precond, pre_own) : nullptr;
    rep = igm_report{};
    rep.inner_dims = dims.data();
    rep.relres_history = relres.data();
    rep.gamma_history = gam.data();
    rep.overflow_per_restart = ovf.data();
    tb = std::make_unique<TraceBridge>(trace, std::min<std::size_t>(shift_cap, 1u << 26));
    st = igm_solve(ctx(), up->h, af->h, b.data(), &rc, pre ? pre->h : nullptr, res.x.data(), &rep, tb->ptr());
  }
  tb->flush();
  ok(st);
  SolveReport& r = res.report;
  r.converged = rep.converged != 0;
  r.refinements = rep.refinements;
  r.total_inner_iterations = static_cast<long>(rep.total_inner_iterations);
  r.inner_dims.assign(dims.begin(), dims.begin() + rep.refinements);
  r.relres_history.assign(relres.begin(), relres.begin() + rep.n_relres);
  r.gamma_history.assign(gam.begin(), gam.begin() + rep.refinements);
  r.overflow_per_restart.assign(ovf.begin(), ovf.begin() + rep.refinements);
  r.overflow_events = trace->events;
  r.overflow_total = trace->total_overflows();
  r.wall_time_sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

}  // namespace intgmres

// ===========================================================================
// host-setup entry points of the C ABI (igm.h), shared with the C++ API

namespace {
template <class F>
igm_status setup_guard(F&& fn) {
  try {
    fn();
    return IGM_OK;
  } catch (const std::invalid_argument& e) {
    igm_internal_set_error(e.what());
    return IGM_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    igm_internal_set_error(e.what());
    return IGM_DOMAIN_ERROR;
  } catch (const std::overflow_error& e) {
    igm_internal_set_error(e.what());
    return IGM_OVERFLOW_ERROR;
  } catch (const std::logic_error& e) {
    igm_internal_set_error(e.what());
    return IGM_LOGIC_ERROR;
  } catch (const std::runtime_error& e) {
    igm_internal_set_error(e.what());
    return IGM_RUNTIME_ERROR;
  }
}
}  // namespace

extern "C" igm_status igm_factorize_split_cast(int n, const int* rp, const int* ci, const double* vals,
                                               int* lrp, int* lci, int64_t* lv, int* ldp, int* urp,
                                               int* uci, int64_t* uv, int* udp) {
  return igm_factorize_split_cast_lu(n, rp, ci, vals, lrp, lci, lv, ldp, urp, uci, uv, udp, nullptr);
}

extern "C" igm_status igm_factorize_split_cast_lu(int n, const int* rp, const int* ci, const double* vals,
                                                  int* lrp, int* lci, int64_t* lv, int* ldp, int* urp,
                                                  int* uci, int64_t* uv, int* udp, double* lu_out) {
  return setup_guard([&] {
    intgmres::CsrMatrixF a;
    a.n = n;
    a.row_ptr.assign(rp, rp + n + 1);
    a.col_idx.assign(ci, ci + rp[n]);
    a.vals.assign(vals, vals + rp[n]);
    const intgmres::IluFactors g = intgmres::split_cast(intgmres::ilu0_impl(a, lu_out));
    std::copy(g.lower.row_ptr.begin(), g.lower.row_ptr.end(), lrp);
    std::copy(g.lower.col_idx.begin(), g.lower.col_idx.end(), lci);
    std::copy(g.lower.vals.begin(), g.lower.vals.end(), lv);
    std::copy(g.diag_pos_lower.begin(), g.diag_pos_lower.end(), ldp);
    std::copy(g.upper.row_ptr.begin(), g.upper.row_ptr.end(), urp);
    std::copy(g.upper.col_idx.begin(), g.upper.col_idx.end(), uci);
    std::copy(g.upper.vals.begin(), g.upper.vals.end(), uv);
    std::copy(g.diag_pos_upper.begin(), g.diag_pos_upper.end(), udp);
  });
}

extern "C" igm_status igm_row_scale(int n, const int* row_ptr, const int* /*col_idx*/, const double* vals,
                                    int alpha_a, double* vals_out, double* scale_out) {
  // d_i = 2^-alpha_a * max_j |a_ij|; every scaled row max is exactly 2^alpha_a
  for (int i = 0; i < n; ++i) {
    double mx = 0.0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) mx = intgmres::absmax_update(mx, vals[k]);
    if (mx == 0.0) {
      igm_internal_set_error("row_scale: row " + std::to_string(i) + " has no nonzero entry");
      return IGM_RUNTIME_ERROR;
    }
    const double d = std::ldexp(mx, -alpha_a);
    scale_out[i] = d;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) vals_out[k] = vals[k] / d;
  }
  return IGM_OK;
}

extern "C" igm_status igm_build_split(int /*n*/, int nnz, const double* vals, int alpha_a, int max_components,
                                      int64_t* comp_vals_out, int* alphas_out, int* ncomp_out, int* exact_out) {
  if (max_components < 1) {
    igm_internal_set_error("build_split: need at least one component");
    return IGM_INVALID_ARGUMENT;
  }
  // layer 0 = truncation; each later layer rescales the exact remainder so
  // its largest entry lands in [2^alpha_a, 2^(alpha_a+1))
  std::vector<double> rest(static_cast<std::size_t>(nnz));
  for (int k = 0; k < nnz; ++k) {
    const int64_t q = static_cast<int64_t>(vals[k]);
    comp_vals_out[k] = q;
    rest[k] = vals[k] - static_cast<double>(q);
  }
  auto rest_max = [&] {
    double mx = 0.0;
    for (double r : rest) mx = intgmres::absmax_update(mx, r);
    return mx;
  };
  int layers = 1;
  alphas_out[0] = 0;
  while (layers < max_components) {
    const double mx = rest_max();
    if (mx == 0.0) break;
    const int alpha = alpha_a - std::ilogb(mx);
    if (alpha <= alphas_out[layers - 1]) {
      igm_internal_set_error("build_split: exponents must increase");
      return IGM_LOGIC_ERROR;
    }
    int64_t* layer = comp_vals_out + static_cast<std::size_t>(layers) * nnz;
    for (int k = 0; k < nnz; ++k) {
      const int64_t q = static_cast<int64_t>(std::ldexp(rest[k], alpha));
      layer[k] = q;
      rest[k] -= std::ldexp(static_cast<double>(q), -alpha);
    }
    alphas_out[layers++] = alpha;
  }
  *exact_out = rest_max() == 0.0 ? 1 : 0;
  *ncomp_out = layers;
  return IGM_OK;
}

// ===========================================================================
// refsolve (refsolve.hpp): the FP64 GMRES comparator on the device

#include "intgmres/refsolve.hpp"

namespace intgmres {
namespace {
int call_precond(void* user, int64_t n, const double* in, double* out) {
  const PrecondFn& f = *static_cast<const PrecondFn*>(user);
  const std::vector<double> r = f(std::vector<double>(in, in + n));
  if (static_cast<int64_t>(r.size()) != n) return 1;
  std::copy(r.begin(), r.end(), out);
  return 0;
}

FpCycleResult fp_cycle_up(const CsrfUp& up, int n, int m, const std::vector<double>& b,
                          const std::vector<double>& x0, const PrecondFn& precond) {
  FpCycleResult res;
  res.x.resize(static_cast<size_t>(n));
  std::vector<double> gabs(static_cast<size_t>(std::max(m, 1)));
  int dim = 0;
  ok(igm_fp_cycle(ctx(), up.h, m, b.data(), x0.data(), precond ? &call_precond : nullptr,
                  precond ? const_cast<PrecondFn*>(&precond) : nullptr, res.x.data(), &dim, &res.r0_norm,
                  gabs.data()));
  res.dim = dim;
  res.g_abs.assign(gabs.begin(), gabs.begin() + dim);
  return res;
}
}  // namespace

FpCycleResult fp_cycle(const CsrMatrixF& a, int m, const std::vector<double>& b, const std::vector<double>& x0,
                       const PrecondFn& precond) {
  if (m < 1) throw std::invalid_argument("fp_cycle: m must be >= 1");
  if (static_cast<int>(b.size()) != a.n || static_cast<int>(x0.size()) != a.n)
    throw std::invalid_argument("fp_cycle: dimension mismatch");
  CsrfUp up(a);
  return fp_cycle_up(up, a.n, m, b, x0, precond);
}

FpSolveResult solve_fp(const CsrMatrixF& a, const std::vector<double>& b, const FpGmresConfig& cfg,
                       const FpIluFactors* precond) {
  PrecondFn pf;
  if (precond) pf = [precond](const std::vector<double>& y) { return apply_fp(*precond, y); };
  if (cfg.m < 1) throw std::invalid_argument("fp_cycle: m must be >= 1");
  if (static_cast<int>(b.size()) != a.n) throw std::invalid_argument("fp_cycle: dimension mismatch");
  CsrfUp up(a);
  FpSolveResult res;
  res.x.assign(static_cast<size_t>(a.n), 0.0);
  double relres = residual_fp(a, res.x, b).relnorm;
  res.relres_history.push_back(relres);
  while (relres >= cfg.tol && res.restarts < cfg.max_restarts) {
    const FpCycleResult cyc = fp_cycle_up(up, a.n, cfg.m, b, res.x, pf);
    if (cyc.dim == 0) break;  // no progress possible
    res.x = cyc.x;
    res.restarts += 1;
    res.iterations += cyc.dim;
    res.cycle_dims.push_back(cyc.dim);
    relres = residual_fp(a, res.x, b).relnorm;
    res.relres_history.push_back(relres);
  }
  res.converged = relres < cfg.tol;
  return res;
}

}  // namespace intgmres
