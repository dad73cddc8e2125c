// ref_capi.cpp -- extern "C" adapter over the REFERENCE library itself.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources under /root/reference/proj/core/src (renamed to
// namespace intgmres_ref via -Dintgmres=intgmres_ref) into
// oracle/_ref/libintgmres_ref.so.  It exposes the same call shapes as
// igm_oracle.h (ref_* instead of ora_*) so tests can replay the restatement
// and the CUDA path against the unmodified reference.  No reference source is
// copied into this repository.
#include "igm_oracle.h"

#include "intgmres/fxp.hpp"
#include "intgmres/gmres_int.hpp"
#include "intgmres/ilu.hpp"
#include "intgmres/refine.hpp"
#include "intgmres/split.hpp"

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

using namespace intgmres_ref;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& fn) {
  try {
    fn();
    return ORA_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORA_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return ORA_DOMAIN_ERROR;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return ORA_OVERFLOW_ERROR;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ORA_LOGIC_ERROR;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return ORA_RUNTIME_ERROR;
  }
}

int kernel_id(const std::string& k) {
  static const char* names[] = {"",        "spmv",   "precond", "dot",
                                "axpy",    "norm",   "vec_div", "givens",
                                "givens_norm", "givens_div", "rot"};
  for (int i = 0; i < 11; ++i)
    if (k == names[i]) return i;
  return -1;
}

int op_id(const std::string& o) {
  if (o == "add") return ORA_OP_ADD;
  if (o == "sub") return ORA_OP_SUB;
  if (o == "mul") return ORA_OP_MUL;
  if (o == "shl") return ORA_OP_SHL;
  if (o == "div") return ORA_OP_DIV;
  return 0;
}

// Holds a reference FxTrace for the duration of a call and copies it back.
struct TraceBridge {
  ora_trace* out;
  FxTrace tr;
  explicit TraceBridge(ora_trace* o)
      : out(o), tr(o ? o->checked != 0 : false, o ? o->record_shifts != 0 : false) {}
  FxTrace* ptr() { return out ? &tr : nullptr; }
  void flush() {
    if (!out) return;
    out->total += tr.total_overflows();
    for (const auto& e : tr.events) {
      if (out->n_events >= out->cap_events || !out->events) break;
      int32_t* d = out->events + 4 * out->n_events;
      d[0] = kernel_id(e.kernel); d[1] = op_id(e.op); d[2] = e.restart; d[3] = e.step;
      out->n_events++;
    }
    for (const auto& s : tr.shifts) {
      if (out->n_shifts < out->cap_shifts && out->shifts) {
        int32_t* d = out->shifts + 3 * out->n_shifts;
        d[0] = kernel_id(s.kernel); d[1] = s.b1; d[2] = s.b2;
      }
      out->n_shifts++;
    }
  }
};

SplitMatrix to_split(const ora_split* m) {
  SplitMatrix s;
  s.n = m->n;
  for (int l = 0; l < m->ncomp; ++l) {
    CsrMatrixI c;
    c.n = m->n;
    c.row_ptr.assign(m->row_ptr, m->row_ptr + m->n + 1);
    c.col_idx.assign(m->col_idx, m->col_idx + m->nnz);
    c.vals.assign(m->vals + static_cast<std::size_t>(l) * m->nnz,
                  m->vals + static_cast<std::size_t>(l + 1) * m->nnz);
    s.components.push_back(std::move(c));
    s.alphas.push_back(m->alphas[l]);
  }
  return s;
}

CsrMatrixF to_csrf(const ora_csrf* a) {
  CsrMatrixF c;
  c.n = a->n;
  c.row_ptr.assign(a->row_ptr, a->row_ptr + a->n + 1);
  const int nnz = a->row_ptr[a->n];
  c.col_idx.assign(a->col_idx, a->col_idx + nnz);
  c.vals.assign(a->vals, a->vals + nnz);
  return c;
}

IluFactors to_ilu(const ora_ilu* f) {
  IluFactors g;
  const int n = f->n;
  g.lower.n = g.upper.n = n;
  g.lower.row_ptr.assign(f->l_row_ptr, f->l_row_ptr + n + 1);
  g.lower.col_idx.assign(f->l_col_idx, f->l_col_idx + f->l_row_ptr[n]);
  g.lower.vals.assign(f->l_vals, f->l_vals + f->l_row_ptr[n]);
  g.upper.row_ptr.assign(f->u_row_ptr, f->u_row_ptr + n + 1);
  g.upper.col_idx.assign(f->u_col_idx, f->u_col_idx + f->u_row_ptr[n]);
  g.upper.vals.assign(f->u_vals, f->u_vals + f->u_row_ptr[n]);
  g.diag_pos_lower.assign(f->l_diag_pos, f->l_diag_pos + n);
  g.diag_pos_upper.assign(f->u_diag_pos, f->u_diag_pos + n);
  return g;
}

ShiftPlan to_plan(const ora_shifts& s) {
  ShiftPlan p;
  p.dot_b1 = s.dot_b1; p.dot_b2 = s.dot_b2; p.axpy_b1 = s.axpy_b1;
  p.norm_b1 = s.norm_b1; p.div_b1 = s.div_b1; p.div_b2 = s.div_b2;
  p.givens_b2 = s.givens_b2; p.rot_b = s.rot_b;
  return p;
}

FxVector fxv(int64_t n, const int64_t* p, int f) {
  FxVector v;
  v.raw.assign(p, p + n);
  v.fmt = QFormat(f);
  return v;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_fx_mul(int64_t a, int64_t b, int f, int b1, int b2, int out_frac,
               int64_t* out, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] {
    *out = fx_mul(FxScalar{a, QFormat(f)}, FxScalar{b, QFormat(f)}, b1, b2,
                  out_frac, tb.ptr()).raw;
  });
  tb.flush();
  return rc;
}

int ref_fx_div(int64_t a, int64_t b, int f, int b1, int b2, int64_t* out,
               ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] {
    *out = fx_div(FxScalar{a, QFormat(f)}, FxScalar{b, QFormat(f)}, b1, b2,
                  tb.ptr()).raw;
  });
  tb.flush();
  return rc;
}

int ref_fx_add(int64_t a, int64_t b, int64_t* out, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] { *out = fx_add(FxScalar{a, QFormat(30)}, FxScalar{b, QFormat(30)}, tb.ptr()).raw; });
  tb.flush();
  return rc;
}

int ref_fx_sub(int64_t a, int64_t b, int64_t* out, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] { *out = fx_sub(FxScalar{a, QFormat(30)}, FxScalar{b, QFormat(30)}, tb.ptr()).raw; });
  tb.flush();
  return rc;
}

uint64_t ref_isqrt(uint64_t v) { return isqrt(v); }

int ref_fx_sqrt(int64_t a, int fin, int out_frac, int64_t* out, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] { *out = fx_sqrt(FxScalar{a, QFormat(fin)}, out_frac, tb.ptr()).raw; });
  tb.flush();
  return rc;
}

int ref_encode(double x, int f, int64_t* out) {
  return guard([&] { *out = encode(x, QFormat(f)).raw; });
}

double ref_decode(int64_t raw, int f) { return decode(FxScalar{raw, QFormat(f)}); }

int ref_shifts_validate(const ora_shifts* sp, int f) {
  return guard([&] { to_plan(*sp).validate(QFormat(f)); });
}

int ref_fx_dot(int64_t n, const int64_t* v, const int64_t* w, int f, int b1,
               int b2, int64_t* out, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] { *out = fx_dot(fxv(n, v, f), fxv(n, w, f), b1, b2, tb.ptr()).raw; });
  tb.flush();
  return rc;
}

int ref_fx_norm(int64_t n, const int64_t* v, int f, int b1, int64_t* out,
                ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] { *out = fx_norm(fxv(n, v, f), b1, tb.ptr()).raw; });
  tb.flush();
  return rc;
}

int ref_fx_axpy_sub(int64_t n, int64_t* w, int64_t h, const int64_t* v, int f,
                    int b1, ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] {
    FxVector ww = fxv(n, w, f);
    fx_axpy_sub(ww, FxScalar{h, QFormat(f)}, fxv(n, v, f), b1, tb.ptr());
    std::memcpy(w, ww.raw.data(), sizeof(int64_t) * static_cast<std::size_t>(n));
  });
  tb.flush();
  return rc;
}

int ref_spmv(const ora_split* m, int s, const int64_t* v, int64_t* out,
             ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] {
    const SplitMatrix sm = to_split(m);
    const FxVector r = spmv(sm, s, fxv(m->n, v, 30), tb.ptr());
    std::memcpy(out, r.raw.data(), sizeof(int64_t) * static_cast<std::size_t>(m->n));
  });
  tb.flush();
  return rc;
}

int ref_apply_inverse(const ora_ilu* f, const int64_t* y, int64_t* out,
                      ora_trace* t) {
  TraceBridge tb(t);
  int rc = guard([&] {
    const IluFactors g = to_ilu(f);
    const FxVector r = apply_inverse(g, fxv(f->n, y, 30), tb.ptr());
    std::memcpy(out, r.raw.data(), sizeof(int64_t) * static_cast<std::size_t>(f->n));
  });
  tb.flush();
  return rc;
}

int ref_apply_inverse_fp(const ora_ilu* f, const double* y, double* out) {
  return guard([&] {
    const IluFactors g = to_ilu(f);
    const std::vector<double> r = apply_inverse_fp(g, std::vector<double>(y, y + f->n));
    std::memcpy(out, r.data(), sizeof(double) * static_cast<std::size_t>(f->n));
  });
}

double ref_norm2(int64_t n, const double* v) {
  return norm2(std::vector<double>(v, v + n));
}

double ref_residual_fp(const ora_csrf* a, const double* x, const double* b,
                       double* r) {
  const CsrMatrixF c = to_csrf(a);
  const Residual res = residual_fp(c, std::vector<double>(x, x + a->n),
                                   std::vector<double>(b, b + a->n));
  std::memcpy(r, res.r.data(), sizeof(double) * static_cast<std::size_t>(a->n));
  return res.relnorm;
}

int ref_spmv_fp_split(const ora_split* m, int s, const double* x, double* y) {
  return guard([&] {
    const std::vector<double> r = spmv_fp(to_split(m), s, std::vector<double>(x, x + m->n));
    std::memcpy(y, r.data(), sizeof(double) * static_cast<std::size_t>(m->n));
  });
}

int ref_row_scale(const ora_csrf* a, int alpha_a, double* vals_out,
                  double* scale_out) {
  return guard([&] {
    const RowScaled rs = row_scale(to_csrf(a), alpha_a);
    std::memcpy(vals_out, rs.a.vals.data(), sizeof(double) * rs.a.vals.size());
    std::memcpy(scale_out, rs.scale.data(), sizeof(double) * rs.scale.size());
  });
}

int ref_build_split(const ora_csrf* a, int alpha_a, int max_components,
                    int64_t* comp_vals_out, int* alphas_out, int* ncomp_out,
                    int* exact_out) {
  return guard([&] {
    const SplitMatrix m = build_split(to_csrf(a), alpha_a, max_components);
    const std::size_t nnz = static_cast<std::size_t>(a->row_ptr[a->n]);
    for (std::size_t l = 0; l < m.components.size(); ++l) {
      std::memcpy(comp_vals_out + l * nnz, m.components[l].vals.data(), sizeof(int64_t) * nnz);
      alphas_out[l] = m.alphas[l];
    }
    *ncomp_out = static_cast<int>(m.components.size());
    *exact_out = m.exact ? 1 : 0;
  });
}

int ref_factorize_split_cast(const ora_csrf* a, int* lrp, int* lci,
                             int64_t* lv, int* ldp, int* urp, int* uci,
                             int64_t* uv, int* udp) {
  return guard([&] {
    const IluFactors g = split_cast(factorize_ilu0(to_csrf(a)));
    std::memcpy(lrp, g.lower.row_ptr.data(), sizeof(int) * g.lower.row_ptr.size());
    std::memcpy(lci, g.lower.col_idx.data(), sizeof(int) * g.lower.col_idx.size());
    std::memcpy(lv, g.lower.vals.data(), sizeof(int64_t) * g.lower.vals.size());
    std::memcpy(ldp, g.diag_pos_lower.data(), sizeof(int) * g.diag_pos_lower.size());
    std::memcpy(urp, g.upper.row_ptr.data(), sizeof(int) * g.upper.row_ptr.size());
    std::memcpy(uci, g.upper.col_idx.data(), sizeof(int) * g.upper.col_idx.size());
    std::memcpy(uv, g.upper.vals.data(), sizeof(int64_t) * g.upper.vals.size());
    std::memcpy(udp, g.diag_pos_upper.data(), sizeof(int) * g.diag_pos_upper.size());
  });
}

int ref_run_cycle(const ora_split* m, const ora_cycle_cfg* cfg, const double* b,
                  const double* x0, double* x_out, ora_cycle_out* out,
                  ora_trace* t) {
  TraceBridge tb(t);
  IluFactors ilu;
  if (cfg->precond) ilu = to_ilu(cfg->precond);
  int rc = guard([&] {
    const SplitMatrix sm = to_split(m);
    CycleConfig cc;
    cc.m = cfg->m;
    cc.fmt = QFormat(cfg->frac_bits);
    cc.shifts = to_plan(cfg->shifts);
    cc.s = cfg->s;
    cc.precond = cfg->precond ? &ilu : nullptr;
    cc.collect_basis_norms = cfg->collect_basis_norms != 0;
    ArnoldiState st;
    const CycleResult r = run_cycle(sm, cc, std::vector<double>(b, b + m->n),
                                    std::vector<double>(x0, x0 + m->n), tb.ptr(), &st);
    std::memcpy(x_out, r.x.data(), sizeof(double) * static_cast<std::size_t>(m->n));
    out->dim = r.diag.dim;
    out->r0_norm = r.diag.r0_norm;
    for (std::size_t j = 0; j < r.diag.g_abs.size(); ++j) {
      out->g_abs[j] = r.diag.g_abs[j];
      out->cos_d[j] = r.diag.cos[j];
      out->sin_d[j] = r.diag.sin[j];
    }
    out->n_basis_norms = static_cast<int>(r.diag.basis_norms.size());
    if (out->basis_norms)
      for (std::size_t j = 0; j < r.diag.basis_norms.size(); ++j)
        out->basis_norms[j] = r.diag.basis_norms[j];
    out->n_basis = static_cast<int>(st.basis.size());
    if (out->basis)
      for (std::size_t k = 0; k < st.basis.size(); ++k)
        std::memcpy(out->basis + k * static_cast<std::size_t>(m->n), st.basis[k].raw.data(),
                    sizeof(int64_t) * static_cast<std::size_t>(m->n));
    if (out->hess && !st.hess.empty()) std::memcpy(out->hess, st.hess.data(), sizeof(int64_t) * st.hess.size());
    if (out->g && !st.g.empty()) std::memcpy(out->g, st.g.data(), sizeof(int64_t) * st.g.size());
    if (out->cos_raw && !st.cos_raw.empty()) std::memcpy(out->cos_raw, st.cos_raw.data(), sizeof(int64_t) * st.cos_raw.size());
    if (out->sin_raw && !st.sin_raw.empty()) std::memcpy(out->sin_raw, st.sin_raw.data(), sizeof(int64_t) * st.sin_raw.size());
  });
  tb.flush();
  return rc;
}

int ref_solve_engine(const ora_split* m, const ora_csrf* a_fp, const double* b,
                     const ora_refine_cfg* cfg, const ora_ilu* precond, double* x_out,
                     ora_report* rep, ora_trace* ext, int engine);

int ref_solve(const ora_split* m, const ora_csrf* a_fp, const double* b,
              const ora_refine_cfg* cfg, const ora_ilu* precond, double* x_out,
              ora_report* rep, ora_trace* ext) {
  return ref_solve_engine(m, a_fp, b, cfg, precond, x_out, rep, ext, 0);
}

// engine: 0 = Engine::fixed_point, 1 = Engine::floating_point (refine.hpp:22)
int ref_solve_engine(const ora_split* m, const ora_csrf* a_fp, const double* b,
                     const ora_refine_cfg* cfg, const ora_ilu* precond, double* x_out,
                     ora_report* rep, ora_trace* ext, int engine) {
  TraceBridge tb(ext);
  IluFactors ilu;
  if (precond) ilu = to_ilu(precond);
  int rc = guard([&] {
    const SplitMatrix sm = to_split(m);
    const CsrMatrixF af = to_csrf(a_fp);
    RefineConfig rc2;
    rc2.tol = cfg->tol;
    rc2.max_refinements = cfg->max_refinements;
    rc2.m = cfg->m;
    rc2.fmt = QFormat(cfg->frac_bits);
    rc2.shifts = to_plan(cfg->shifts);
    rc2.s = cfg->s;
    rc2.checked = cfg->checked != 0;
    rc2.engine = engine ? Engine::floating_point : Engine::fixed_point;
    if (cfg->s_schedule) {
      const int* sched = cfg->s_schedule;
      rc2.s_schedule = [sched](int k) { return sched[k]; };
    }
    const SolveResult r = solve(sm, af, std::vector<double>(b, b + m->n), rc2,
                                precond ? &ilu : nullptr, tb.ptr());
    std::memcpy(x_out, r.x.data(), sizeof(double) * static_cast<std::size_t>(m->n));
    const SolveReport& s = r.report;
    rep->converged = s.converged;
    rep->refinements = s.refinements;
    rep->total_inner_iterations = s.total_inner_iterations;
    for (std::size_t k = 0; k < s.inner_dims.size(); ++k) rep->inner_dims[k] = s.inner_dims[k];
    rep->n_relres = static_cast<int>(s.relres_history.size());
    for (std::size_t k = 0; k < s.relres_history.size(); ++k) rep->relres_history[k] = s.relres_history[k];
    for (std::size_t k = 0; k < s.gamma_history.size(); ++k) rep->gamma_history[k] = s.gamma_history[k];
    for (std::size_t k = 0; k < s.overflow_per_restart.size(); ++k)
      rep->overflow_per_restart[k] = s.overflow_per_restart[k];
    rep->overflow_total = s.overflow_total;
    rep->wall_time_sec = s.wall_time_sec;
  });
  tb.flush();
  return rc;
}

}  // extern "C"

// ---- the reference's FP64 comparator (refsolve.cpp), for the device
// implementation's tests: fp_cycle / solve_fp on a CsrMatrixF, optionally
// preconditioned with apply_fp(factorize_ilu0(a)).
#include "intgmres/refsolve.hpp"

extern "C" {

int ref_fp_cycle(const ora_csrf* a, int m, const double* b, const double* x0, int use_ilu, double* x_out,
                 int* dim, double* r0_norm, double* g_abs) {
  return guard([&] {
    const CsrMatrixF af = to_csrf(a);
    PrecondFn pf;
    FpIluFactors f;
    if (use_ilu) {
      f = factorize_ilu0(af);
      pf = [&f](const std::vector<double>& y) { return apply_fp(f, y); };
    }
    const FpCycleResult r = fp_cycle(af, m, std::vector<double>(b, b + a->n), std::vector<double>(x0, x0 + a->n), pf);
    std::memcpy(x_out, r.x.data(), sizeof(double) * static_cast<std::size_t>(a->n));
    *dim = r.dim;
    *r0_norm = r.r0_norm;
    for (std::size_t i = 0; i < r.g_abs.size(); ++i) g_abs[i] = r.g_abs[i];
  });
}

int ref_solve_fp(const ora_csrf* a, const double* b, int m, double tol, int max_restarts, int use_ilu,
                 double* x_out, int* restarts, long* iterations, int* converged) {
  return guard([&] {
    const CsrMatrixF af = to_csrf(a);
    FpGmresConfig cfg;
    cfg.m = m;
    cfg.tol = tol;
    cfg.max_restarts = max_restarts;
    FpIluFactors f;
    if (use_ilu) f = factorize_ilu0(af);
    const FpSolveResult r = solve_fp(af, std::vector<double>(b, b + a->n), cfg, use_ilu ? &f : nullptr);
    std::memcpy(x_out, r.x.data(), sizeof(double) * static_cast<std::size_t>(a->n));
    *restarts = r.restarts;
    *iterations = r.iterations;
    *converged = r.converged;
  });
}

}  // extern "C"

// ---- the reference's experiment path (experiment.cpp), for the drop-in's test
#include "intgmres/experiment.hpp"

extern "C" {

int ref_run_experiment(const char* path, int solver, int precond, int m, double tol, int max_ref, char* csv,
                       int csv_cap, char* summary, int summary_cap) {
  return guard([&] {
    ExperimentSpec spec;
    spec.matrix_path = path;
    spec.solver = solver ? SolverKind::fp64 : SolverKind::integer;
    spec.precond = precond ? PrecondKind::ilu0 : PrecondKind::none;
    spec.m = m;
    spec.tol = tol;
    spec.max_refinements = max_ref;
    const ExperimentResult r = run_experiment(spec);
    std::snprintf(csv, static_cast<std::size_t>(csv_cap), "%s", r.csv.c_str());
    std::snprintf(summary, static_cast<std::size_t>(summary_cap), "%s", r.summary.c_str());
  });
}

}  // extern "C"
