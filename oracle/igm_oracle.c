/*
 * igm_oracle.c -- CPU restatement of the reference int-GMRES hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see igm_oracle.h).  The product never links this.
 * All citations are into /root/reference/proj/core/.
 */
#include "igm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char g_err[256];

const char* ora_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------------ */
/* FxTrace (fxp.hpp:51-103)                                                  */

static int checking(const ora_trace* t) { return t != NULL && t->checked; }

static void record_overflow(ora_trace* t, int op) {
  /* fxp.hpp:76-80: total always counts, the event list caps */
  t->total++;
  if (t->n_events < t->cap_events && t->events) {
    int32_t* e = t->events + 4 * t->n_events;
    e[0] = t->kernel; e[1] = op; e[2] = t->restart; e[3] = t->step;
    t->n_events++;
  }
}

static void record_shift(ora_trace* t, int b1, int b2) {
  /* fxp.hpp:81-83; callers guard with `if (t)` */
  if (!t || !t->record_shifts) return;
  if (t->n_shifts < t->cap_shifts && t->shifts) {
    int32_t* s = t->shifts + 3 * t->n_shifts;
    s[0] = t->kernel; s[1] = b1; s[2] = b2;
  }
  t->n_shifts++;
}

static void set_kernel(ora_trace* t, int k) { if (t) t->kernel = k; }

/* ------------------------------------------------------------------------ */
/* detail:: primitives (fxp.hpp:105-163)                                     */

int64_t ora_asr(int64_t x, int s) { /* fxp.hpp:108-111 */
  if (s >= 63) return x >> 63;
  return x >> s;
}

int64_t ora_wrap_shl(int64_t x, int s) { /* fxp.hpp:114-117 */
  if (s >= 64) return 0;
  return (int64_t)((uint64_t)x << s);
}

static int64_t add_c(int64_t a, int64_t b, ora_trace* t) { /* fxp.hpp:121-125 */
  int64_t r;
  if (__builtin_add_overflow(a, b, &r) && checking(t)) record_overflow(t, ORA_OP_ADD);
  return r;
}

static int64_t sub_c(int64_t a, int64_t b, ora_trace* t) { /* fxp.hpp:127-131 */
  int64_t r;
  if (__builtin_sub_overflow(a, b, &r) && checking(t)) record_overflow(t, ORA_OP_SUB);
  return r;
}

static int64_t mul_c(int64_t a, int64_t b, ora_trace* t) { /* fxp.hpp:133-137 */
  int64_t r;
  if (__builtin_mul_overflow(a, b, &r) && checking(t)) record_overflow(t, ORA_OP_MUL);
  return r;
}

static int64_t shl_c(int64_t x, int s, ora_trace* t) { /* fxp.hpp:139-143 */
  int64_t r = ora_wrap_shl(x, s);
  if (ora_asr(r, s) != x && checking(t)) record_overflow(t, ORA_OP_SHL);
  return r;
}

static int64_t div_c(int64_t num, int64_t den, ora_trace* t) { /* fxp.hpp:145-152 */
  if (num == INT64_MIN && den == -1) {
    if (checking(t)) record_overflow(t, ORA_OP_DIV);
    return num;
  }
  return num / den;
}

static int shift_range(int b, const char* who) { /* fxp.hpp:159-163 */
  if (b < 0 || b > 63) {
    snprintf(g_err, sizeof g_err, "%s: shift out of [0, 63]", who);
    return ORA_INVALID_ARGUMENT;
  }
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* scalar conversions and ops                                                */

int ora_encode(double x, int f, int64_t* out) { /* fxp.hpp:171-176 */
  const int int_bits = 64 - 1 - f;
  if (!(fabs(x) < ldexp(1.0, int_bits)))
    return fail(ORA_OVERFLOW_ERROR, "encode: value outside representable range");
  *out = (int64_t)ldexp(x, f);
  return ORA_OK;
}

double ora_decode(int64_t raw, int f) { /* fxp.hpp:180-182 */
  return ldexp((double)raw, -f);
}

int ora_fx_add(int64_t a, int64_t b, int64_t* out, ora_trace* t) {
  *out = add_c(a, b, t); /* fxp.hpp:189-193 */
  return ORA_OK;
}

int ora_fx_sub(int64_t a, int64_t b, int64_t* out, ora_trace* t) {
  *out = sub_c(a, b, t); /* fxp.hpp:195-199 */
  return ORA_OK;
}

int ora_fx_mul(int64_t a, int64_t b, int f, int b1, int b2, int out_frac,
               int64_t* out, ora_trace* t) { /* fxp.hpp:203-216 */
  int rc;
  if ((rc = shift_range(b1, "fx_mul")) || (rc = shift_range(b2, "fx_mul"))) return rc;
  if (out_frac < 0 || out_frac > 62)
    return fail(ORA_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 62]");
  const int post = 2 * f - b1 - b2 - out_frac;
  if (post < 0)
    return fail(ORA_INVALID_ARGUMENT, "fx_mul: shifts exceed available precision");
  if (t) record_shift(t, b1, b2);
  const int64_t p = mul_c(ora_asr(a, b1), ora_asr(b, b2), t);
  *out = ora_asr(p, post);
  return ORA_OK;
}

int ora_fx_div(int64_t a, int64_t b, int f, int b1, int b2, int64_t* out,
               ora_trace* t) { /* fxp.hpp:220-234 */
  int rc;
  if ((rc = shift_range(b1, "fx_div")) || (rc = shift_range(b2, "fx_div"))) return rc;
  if (t) record_shift(t, b1, b2);
  const int64_t num = shl_c(a, b1, t);
  const int64_t den = ora_asr(b, b2);
  if (den == 0) return fail(ORA_DOMAIN_ERROR, "fx_div: shifted divisor is zero");
  const int64_t q = div_c(num, den, t);
  const int e = f - b1 - b2;
  *out = e >= 0 ? shl_c(q, e, t) : ora_asr(q, -e);
  return ORA_OK;
}

uint64_t ora_isqrt(uint64_t v) { /* fxp.cpp:20-33: Newton from 2^ceil(bits/2) */
  if (v == 0) return 0;
  const int bits = 64 - __builtin_clzll(v);
  uint64_t x = (uint64_t)1 << ((bits + 1) / 2);
  for (;;) {
    const uint64_t nx = (x + v / x) / 2;
    if (nx >= x) break;
    x = nx;
  }
  while ((unsigned __int128)x * x > v) --x;
  return x;
}

int ora_fx_sqrt(int64_t a, int fin, int out_frac, int64_t* out,
                ora_trace* t) { /* fxp.cpp:35-47 */
  if (a < 0) return fail(ORA_DOMAIN_ERROR, "fx_sqrt: negative input");
  if (fin % 2 != 0)
    return fail(ORA_INVALID_ARGUMENT, "fx_sqrt: input frac_bits must be even");
  if (out_frac < 0 || out_frac > 62)
    return fail(ORA_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 62]");
  const int64_t r = (int64_t)ora_isqrt((uint64_t)a);
  const int e = out_frac - fin / 2;
  *out = e >= 0 ? shl_c(r, e, t) : ora_asr(r, -e);
  return ORA_OK;
}

int ora_shifts_validate(const ora_shifts* p, int f) { /* fxp.cpp:106-127 */
#define RIGHT(b, name)                                                       \
  if ((b) < 0 || ((b) > 0 && (b) >= f))                                      \
    return fail(ORA_INVALID_ARGUMENT, "ShiftPlan: " name " must lie in [0, frac_bits)");
  RIGHT(p->dot_b1, "dot_b1");
  RIGHT(p->dot_b2, "dot_b2");
  RIGHT(p->axpy_b1, "axpy_b1");
  RIGHT(p->norm_b1, "norm_b1");
  RIGHT(p->div_b2, "div_b2");
  RIGHT(p->givens_b2, "givens_b2");
#undef RIGHT
  if (p->div_b1 < 0 || p->div_b1 > f)
    return fail(ORA_INVALID_ARGUMENT, "ShiftPlan: div_b1 must lie in [0, frac_bits]");
  if (p->rot_b != 0) return fail(ORA_INVALID_ARGUMENT, "ShiftPlan: rot_b must be 0");
  if (2 * (f - p->norm_b1) > 62)
    return fail(ORA_INVALID_ARGUMENT,
                "ShiftPlan: norm accumulator needs 2*(frac_bits - norm_b1) <= 62");
  return ORA_OK;
}

void ora_shifts_default_unpreconditioned(int f, ora_shifts* p) { /* fxp.cpp:129-141 */
  memset(p, 0, sizeof *p);
  p->dot_b1 = 16; p->dot_b2 = 0; p->axpy_b1 = 16; p->norm_b1 = 16;
  p->div_b1 = 16; p->div_b2 = f - 16; p->givens_b2 = 16; p->rot_b = 0;
}

void ora_shifts_default_preconditioned(int f, ora_shifts* p) { /* fxp.cpp:143-148 */
  memset(p, 0, sizeof *p);
  p->div_b1 = f;
}

/* ------------------------------------------------------------------------ */
/* vector kernels (fxp.cpp:49-104)                                           */

int ora_fx_dot(int64_t n, const int64_t* v, const int64_t* w, int f, int b1,
               int b2, int64_t* out, ora_trace* t) { /* fxp.cpp:49-67 */
  int rc;
  if ((rc = shift_range(b1, "fx_dot")) || (rc = shift_range(b2, "fx_dot"))) return rc;
  if (t) record_shift(t, b1, b2);
  int64_t acc = 0;
  for (int64_t l = 0; l < n; ++l) {
    const int64_t p = mul_c(ora_asr(v[l], b1), ora_asr(w[l], b2), t);
    acc = add_c(acc, p, t);
  }
  const int e = f - b1 - b2;
  *out = e >= 0 ? ora_asr(acc, e) : shl_c(acc, -e, t);
  return ORA_OK;
}

int ora_fx_norm(int64_t n, const int64_t* v, int f, int b1, int64_t* out,
                ora_trace* t) { /* fxp.cpp:69-86 */
  int rc;
  if ((rc = shift_range(b1, "fx_norm"))) return rc;
  const int acc_frac = 2 * (f - b1);
  if (acc_frac < 0 || acc_frac > 62)
    return fail(ORA_INVALID_ARGUMENT,
                "fx_norm: accumulator format not representable (need 2*(f-b1) in "
                "[0, 62])");
  if (t) record_shift(t, b1, b1);
  int64_t acc = 0;
  for (int64_t l = 0; l < n; ++l) {
    const int64_t s = ora_asr(v[l], b1);
    acc = add_c(acc, mul_c(s, s, t), t);
  }
  if (acc < 0) return fail(ORA_DOMAIN_ERROR, "fx_norm: accumulator wrapped negative");
  return ora_fx_sqrt(acc, acc_frac, f, out, t);
}

int ora_fx_axpy_sub(int64_t n, int64_t* w, int64_t h, const int64_t* v, int f,
                    int b1, ora_trace* t) { /* fxp.cpp:88-104 */
  int rc;
  if ((rc = shift_range(b1, "fx_axpy_sub"))) return rc;
  const int post = f - b1;
  if (post < 0) return fail(ORA_INVALID_ARGUMENT, "fx_axpy_sub: b1 exceeds frac_bits");
  if (t) record_shift(t, b1, 0);
  const int64_t hs = ora_asr(h, b1);
  for (int64_t l = 0; l < n; ++l) {
    const int64_t p = mul_c(hs, v[l], t);
    w[l] = sub_c(w[l], ora_asr(p, post), t);
  }
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* operators                                                                 */

int ora_spmv(const ora_split* m, int s, const int64_t* v, int64_t* out,
             ora_trace* t) { /* split.cpp:137-157 */
  if (s < 0 || s > m->ncomp - 1)
    return fail(ORA_INVALID_ARGUMENT, "spmv: component index out of range");
  for (int i = 0; i < m->n; ++i) out[i] = 0;
  for (int l = 0; l <= s; ++l) {
    const int64_t* vals = m->vals + (int64_t)l * m->nnz;
    const int alpha = m->alphas[l];
    for (int i = 0; i < m->n; ++i) {
      int64_t acc = 0;
      for (int k = m->row_ptr[i]; k < m->row_ptr[i + 1]; ++k)
        acc = add_c(acc, mul_c(vals[k], v[m->col_idx[k]], t), t);
      out[i] = add_c(out[i], ora_asr(acc, alpha), t);
    }
  }
  return ORA_OK;
}

int ora_apply_inverse(const ora_ilu* f, const int64_t* y, int64_t* out,
                      ora_trace* t) { /* ilu.cpp:122-155 */
  const int n = f->n;
  int64_t* z = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) { /* forward */
    int64_t acc = y[i];
    for (int k = f->l_row_ptr[i]; k < f->l_row_ptr[i + 1]; ++k) {
      const int j = f->l_col_idx[k];
      if (j == i) continue;
      acc = sub_c(acc, mul_c(f->l_vals[k], z[j], t), t);
    }
    z[i] = div_c(acc, f->l_vals[f->l_diag_pos[i]], t);
  }
  for (int i = n - 1; i >= 0; --i) { /* backward */
    int64_t acc = z[i];
    for (int k = f->u_row_ptr[i]; k < f->u_row_ptr[i + 1]; ++k) {
      const int j = f->u_col_idx[k];
      if (j == i) continue;
      acc = sub_c(acc, mul_c(f->u_vals[k], out[j], t), t);
    }
    out[i] = div_c(acc, f->u_vals[f->u_diag_pos[i]], t);
  }
  free(z);
  return ORA_OK;
}

int ora_apply_inverse_fp(const ora_ilu* f, const double* y,
                         double* out) { /* ilu.cpp:157-180 */
  const int n = f->n;
  double* z = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    double acc = y[i];
    for (int k = f->l_row_ptr[i]; k < f->l_row_ptr[i + 1]; ++k) {
      const int j = f->l_col_idx[k];
      if (j != i) acc -= (double)f->l_vals[k] * z[j];
    }
    z[i] = acc / (double)f->l_vals[f->l_diag_pos[i]];
  }
  for (int i = n - 1; i >= 0; --i) {
    double acc = z[i];
    for (int k = f->u_row_ptr[i]; k < f->u_row_ptr[i + 1]; ++k) {
      const int j = f->u_col_idx[k];
      if (j != i) acc -= (double)f->u_vals[k] * out[j];
    }
    out[i] = acc / (double)f->u_vals[f->u_diag_pos[i]];
  }
  free(z);
  return ORA_OK;
}

void ora_spmv_fp_csr(const ora_csrf* a, const double* x, double* y) { /* split.cpp:37-43 */
  for (int i = 0; i < a->n; ++i) {
    y[i] = 0.0;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
      y[i] += a->vals[k] * x[a->col_idx[k]];
  }
}

int ora_spmv_fp_split(const ora_split* m, int s, const double* x,
                      double* y) { /* split.cpp:159-175 */
  if (s < 0 || s > m->ncomp - 1)
    return fail(ORA_INVALID_ARGUMENT, "spmv_fp: component index out of range");
  for (int i = 0; i < m->n; ++i) y[i] = 0.0;
  for (int l = 0; l <= s; ++l) {
    const int64_t* vals = m->vals + (int64_t)l * m->nnz;
    const double scale = ldexp(1.0, -m->alphas[l]);
    for (int i = 0; i < m->n; ++i) {
      double acc = 0.0;
      for (int k = m->row_ptr[i]; k < m->row_ptr[i + 1]; ++k)
        acc += (double)vals[k] * x[m->col_idx[k]];
      y[i] += scale * acc;
    }
  }
  return ORA_OK;
}

double ora_norm2(int64_t n, const double* v) { /* split.cpp:45-49: serial chain */
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += v[i] * v[i];
  return sqrt(acc);
}

double ora_residual_fp(const ora_csrf* a, const double* x, const double* b,
                       double* r) { /* split.cpp:51-59 */
  ora_spmv_fp_csr(a, x, r);
  for (int i = 0; i < a->n; ++i) r[i] = b[i] - r[i];
  const double nb = ora_norm2(a->n, b);
  return nb == 0.0 ? ora_norm2(a->n, r) : ora_norm2(a->n, r) / nb;
}

int ora_gamma_scale(int64_t n, const double* r, double* gamma,
                    double* b_k) { /* refine.cpp:11-19 */
  double g = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double a = fabs(r[i]);
    g = (g < a) ? a : g; /* std::max(g, a) */
  }
  if (g == 0.0) return fail(ORA_INVALID_ARGUMENT, "gamma_scale: zero residual");
  for (int64_t i = 0; i < n; ++i) b_k[i] = r[i] / g;
  *gamma = g;
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* host setup                                                                */

int ora_row_scale(const ora_csrf* a, int alpha_a, double* vals_out,
                  double* scale_out) { /* split.cpp:61-79 */
  for (int i = 0; i < a->n; ++i) {
    double mx = 0.0;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
      const double v = fabs(a->vals[k]);
      mx = (mx < v) ? v : mx;
    }
    if (mx == 0.0) {
      snprintf(g_err, sizeof g_err, "row_scale: row %d has no nonzero entry", i);
      return ORA_RUNTIME_ERROR;
    }
    const double d = ldexp(mx, -alpha_a);
    scale_out[i] = d;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
      vals_out[k] = a->vals[k] / d;
  }
  return ORA_OK;
}

int ora_build_split(int n, int nnz, const double* vals, int alpha_a,
                    int max_components, int64_t* comp_vals_out, int* alphas_out,
                    int* ncomp_out, int* exact_out) { /* split.cpp:90-135 */
  (void)n;
  if (max_components < 1)
    return fail(ORA_INVALID_ARGUMENT, "build_split: need at least one component");
  double* rem = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  for (int k = 0; k < nnz; ++k) {
    comp_vals_out[k] = (int64_t)vals[k];
    rem[k] = vals[k] - (double)comp_vals_out[k];
  }
  int nc = 1;
  alphas_out[0] = 0;
  while (nc < max_components) {
    double mx = 0.0;
    for (int k = 0; k < nnz; ++k) { const double r = fabs(rem[k]); mx = (mx < r) ? r : mx; }
    if (mx == 0.0) break;
    const int alpha = alpha_a - ilogb(mx);
    if (alpha <= alphas_out[nc - 1]) {
      free(rem);
      return fail(ORA_LOGIC_ERROR, "build_split: exponents must increase");
    }
    int64_t* cv = comp_vals_out + (int64_t)nc * nnz;
    for (int k = 0; k < nnz; ++k) {
      const double scaled = ldexp(rem[k], alpha);
      cv[k] = (int64_t)scaled;
      rem[k] -= ldexp((double)cv[k], -alpha);
    }
    alphas_out[nc] = alpha;
    nc++;
  }
  double mx = 0.0;
  for (int k = 0; k < nnz; ++k) { const double r = fabs(rem[k]); mx = (mx < r) ? r : mx; }
  *exact_out = mx == 0.0;
  *ncomp_out = nc;
  free(rem);
  return ORA_OK;
}

int ora_factorize_split_cast(const ora_csrf* a, int* lrp, int* lci,
                             int64_t* lv, int* ldp, int* urp, int* uci,
                             int64_t* uv, int* udp) { /* ilu.cpp:25-120 */
  const int n = a->n;
  const int nnz = a->row_ptr[n];
  int* diag = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    diag[i] = -1;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k)
      if (a->col_idx[k] == i) diag[i] = k;
  }
  for (int i = 0; i < n; ++i)
    if (diag[i] < 0) {
      free(diag);
      snprintf(g_err, sizeof g_err,
               "factorize_ilu0: row %d has no diagonal entry in the pattern", i);
      return ORA_RUNTIME_ERROR;
    }
  double* lu = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  memcpy(lu, a->vals, sizeof(double) * (size_t)nnz);
  int* iw = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) iw[i] = -1;
  for (int i = 0; i < n; ++i) { /* ilu.cpp:31-48 */
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) iw[a->col_idx[k]] = k;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
      const int j = a->col_idx[k];
      if (j >= i) break;
      lu[k] /= lu[diag[j]];
      for (int kk = diag[j] + 1; kk < a->row_ptr[j + 1]; ++kk) {
        const int pos = iw[a->col_idx[kk]];
        if (pos >= 0) lu[pos] -= lu[k] * lu[kk];
      }
    }
    if (lu[diag[i]] == 0.0) {
      free(diag); free(lu); free(iw);
      snprintf(g_err, sizeof g_err, "factorize_ilu0: zero pivot in row %d", i);
      return ORA_RUNTIME_ERROR;
    }
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) iw[a->col_idx[k]] = -1;
  }
  /* split (ilu.cpp:52-77) fused with split_cast (ilu.cpp:80-120) */
  int nl = 0, nu = 0;
  lrp[0] = urp[0] = 0;
  for (int i = 0; i < n; ++i) {
    const double d = lu[diag[i]];
    const double r = sqrt(fabs(d));
    const double du = d < 0 ? -r : r;
    ldp[i] = udp[i] = -1;
    for (int k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
      const int j = a->col_idx[k];
      if (j < i) { /* lower multiplier, column-scaled by dl_j */
        const double dj = lu[diag[j]];
        lci[nl] = j;
        lv[nl] = (int64_t)(lu[k] * sqrt(fabs(dj)));
        nl++;
      } else if (j == i) {
        lci[nl] = i; lv[nl] = (int64_t)(1.0 * r); ldp[i] = nl; nl++;
        uci[nu] = i; uv[nu] = (int64_t)(1.0 * du); udp[i] = nu; nu++;
      } else {
        uci[nu] = j;
        uv[nu] = (int64_t)((lu[k] / d) * du);
        nu++;
      }
    }
    lrp[i + 1] = nl;
    urp[i + 1] = nu;
  }
  for (int i = 0; i < n; ++i) {
    if (lv[ldp[i]] == 0 || uv[udp[i]] == 0) {
      free(diag); free(lu); free(iw);
      snprintf(g_err, sizeof g_err,
               "split_cast: diagonal entry of row %d truncates to zero; scale the "
               "matrix up before factorizing", i);
      return ORA_RUNTIME_ERROR;
    }
  }
  free(diag); free(lu); free(iw);
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* Givens / Hessenberg (gmres_int.cpp:8-40)                                  */

int ora_apply_stored_rotations(int64_t* h, int count, const int64_t* c,
                               const int64_t* s, int gb2, int f, ora_trace* t) {
  for (int i = 0; i < count; ++i) { /* gmres_int.cpp:12-24 */
    int64_t a, b, d, e, rc;
    if ((rc = ora_fx_mul(c[i], h[i], f, 0, gb2, f, &a, t))) return (int)rc;
    if ((rc = ora_fx_mul(s[i], h[i + 1], f, 0, gb2, f, &b, t))) return (int)rc;
    if ((rc = ora_fx_mul(c[i], h[i + 1], f, 0, gb2, f, &d, t))) return (int)rc;
    if ((rc = ora_fx_mul(s[i], h[i], f, 0, gb2, f, &e, t))) return (int)rc;
    h[i] = add_c(a, b, t);
    h[i + 1] = sub_c(d, e, t);
  }
  return ORA_OK;
}

int ora_solve_hessenberg(const double* r, int ld, int dim, const double* g,
                         double* y) { /* gmres_int.cpp:27-40 */
  for (int i = dim - 1; i >= 0; --i) {
    double acc = g[i];
    for (int j = i + 1; j < dim; ++j) acc -= r[j * ld + i] * y[j];
    const double rii = r[i * ld + i];
    if (rii == 0.0) return fail(ORA_RUNTIME_ERROR, "solve_hessenberg: zero diagonal");
    y[i] = acc / rii;
  }
  return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* run_cycle (gmres_int.cpp:42-196)                                          */

int ora_run_cycle(const ora_split* m, const ora_cycle_cfg* cfg, const double* b,
                  const double* x0, double* x, ora_cycle_out* out,
                  ora_trace* t) {
  const int n = m->n;
  const int M = cfg->m;
  const int f = cfg->frac_bits;
  const ora_shifts* sp = &cfg->shifts;
  int rc = ORA_OK;
  if (M < 1) return fail(ORA_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
  if (cfg->s < 0 || cfg->s > m->ncomp - 1)
    return fail(ORA_INVALID_ARGUMENT, "run_cycle: splitting depth out of range");
  if (f < 0 || f > 62) return fail(ORA_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 62]");
  if ((rc = ora_shifts_validate(sp, f))) return rc;

  for (int i = 0; i < n; ++i) x[i] = x0[i];
  out->dim = 0;
  out->r0_norm = 0.0;
  out->n_basis = 0;
  out->n_basis_norms = 0;

  /* r0 in floating point (gmres_int.cpp:61-70) */
  double* r0 = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) r0[i] = b[i];
  int x0_nonzero = 0;
  for (int i = 0; i < n; ++i) x0_nonzero = x0_nonzero || x0[i] != 0.0;
  if (x0_nonzero) {
    double* ax = (double*)malloc(sizeof(double) * (size_t)n);
    ora_spmv_fp_split(m, cfg->s, x0, ax);
    for (int i = 0; i < n; ++i) r0[i] -= ax[i];
    free(ax);
  }
  if (cfg->precond) {
    double* z = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    ora_apply_inverse_fp(cfg->precond, r0, z);
    free(r0);
    r0 = z;
  }
  const double r0n = ora_norm2(n, r0);
  out->r0_norm = r0n;
  if (r0n == 0.0) { free(r0); return ORA_OK; }

  const int ld = M + 1;
  int64_t* basis = (int64_t*)calloc((size_t)(M + 1) * (size_t)n + 1, sizeof(int64_t));
  int nb = 0;
  for (int i = 0; i < n; ++i) { /* gmres_int.cpp:77-81 */
    if ((rc = ora_encode(r0[i] / r0n, f, &basis[i]))) { free(r0); free(basis); return rc; }
  }
  nb = 1;
  free(r0);

  int64_t* hess = (int64_t*)calloc((size_t)ld * M, sizeof(int64_t));
  int64_t* g = (int64_t*)calloc((size_t)ld, sizeof(int64_t));
  int64_t* cr = (int64_t*)calloc((size_t)M, sizeof(int64_t));
  int64_t* sr = (int64_t*)calloc((size_t)M, sizeof(int64_t));
  int64_t* w = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t* w2 = cfg->precond ? (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1)) : NULL;
  g[0] = (int64_t)1 << f;

  int dim = 0;
  for (int j = 0; j < M; ++j) { /* gmres_int.cpp:90-160 */
    if (t) t->step = j;
    int64_t* col = &hess[(size_t)j * ld];
    const int64_t* vj = basis + (size_t)j * n;

    set_kernel(t, ORA_K_SPMV);
    if ((rc = ora_spmv(m, cfg->s, vj, w, t))) goto done;
    if (cfg->precond) {
      set_kernel(t, ORA_K_PRECOND);
      ora_apply_inverse(cfg->precond, w, w2, t);
      memcpy(w, w2, sizeof(int64_t) * (size_t)n);
    }
    for (int i = 0; i <= j; ++i) {
      const int64_t* vi = basis + (size_t)i * n;
      int64_t hij;
      set_kernel(t, ORA_K_DOT);
      if ((rc = ora_fx_dot(n, w, vi, f, sp->dot_b1, sp->dot_b2, &hij, t))) goto done;
      col[i] = hij;
      set_kernel(t, ORA_K_AXPY);
      if ((rc = ora_fx_axpy_sub(n, w, hij, vi, f, sp->axpy_b1, t))) goto done;
    }
    set_kernel(t, ORA_K_NORM);
    int64_t hnext;
    if ((rc = ora_fx_norm(n, w, f, sp->norm_b1, &hnext, t))) goto done;
    col[j + 1] = hnext;
    const int happy = hnext == 0;
    if (!happy) {
      set_kernel(t, ORA_K_VEC_DIV);
      int64_t* vn = basis + (size_t)(j + 1) * n;
      for (int l = 0; l < n; ++l)
        if ((rc = ora_fx_div(w[l], hnext, f, sp->div_b1, sp->div_b2, &vn[l], t))) goto done;
      nb++;
    }
    set_kernel(t, ORA_K_GIVENS);
    if ((rc = ora_apply_stored_rotations(col, j, cr, sr, sp->givens_b2, f, t))) goto done;

    set_kernel(t, ORA_K_GIVENS_NORM);
    int64_t pair[2] = {col[j], col[j + 1]};
    int64_t tmp;
    if ((rc = ora_fx_norm(2, pair, f, sp->norm_b1, &tmp, t))) goto done;
    if (tmp == 0) break;

    set_kernel(t, ORA_K_GIVENS_DIV);
    int64_t c, s;
    if ((rc = ora_fx_div(col[j], tmp, f, sp->div_b1, sp->div_b2, &c, t))) goto done;
    if ((rc = ora_fx_div(col[j + 1], tmp, f, sp->div_b1, sp->div_b2, &s, t))) goto done;
    cr[j] = c;
    sr[j] = s;
    col[j] = tmp;
    col[j + 1] = 0;

    set_kernel(t, ORA_K_ROT);
    const int64_t g_old = g[j];
    const int64_t neg_s = sub_c(0, s, t);
    if ((rc = ora_fx_mul(neg_s, g_old, f, sp->rot_b, sp->rot_b, f, &g[j + 1], t))) goto done;
    if ((rc = ora_fx_mul(c, g_old, f, sp->rot_b, sp->rot_b, f, &g[j], t))) goto done;

    dim = j + 1;
    out->g_abs[j] = fabs(ora_decode(g[j + 1], f));
    out->cos_d[j] = ora_decode(c, f);
    out->sin_d[j] = ora_decode(s, f);
    if (happy) break;
  }
  out->dim = dim;

  if (dim > 0) { /* gmres_int.cpp:163-180 */
    double* rcols = (double*)calloc((size_t)ld * dim, sizeof(double));
    double* gd = (double*)malloc(sizeof(double) * (size_t)dim);
    double* y = (double*)malloc(sizeof(double) * (size_t)dim);
    for (int j = 0; j < dim; ++j) {
      for (int i = 0; i <= j; ++i)
        rcols[(size_t)j * ld + i] = ora_decode(hess[(size_t)j * ld + i], f);
      gd[j] = ora_decode(g[j], f);
    }
    rc = ora_solve_hessenberg(rcols, ld, dim, gd, y);
    if (!rc) {
      for (int j = 0; j < dim; ++j) {
        const int64_t* vj = basis + (size_t)j * n;
        const double wj = r0n * y[j];
        for (int l = 0; l < n; ++l) x[l] += wj * ora_decode(vj[l], f);
      }
    }
    free(rcols); free(gd); free(y);
    if (rc) goto done;
  }

  if (cfg->collect_basis_norms && out->basis_norms) {
    double* dv = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int k = 0; k < nb; ++k) {
      for (int l = 0; l < n; ++l) dv[l] = ora_decode(basis[(size_t)k * n + l], f);
      out->basis_norms[k] = ora_norm2(n, dv);
    }
    out->n_basis_norms = nb;
    free(dv);
  }
  out->n_basis = nb;
  if (out->basis) memcpy(out->basis, basis, sizeof(int64_t) * (size_t)nb * n);
  if (out->hess) memcpy(out->hess, hess, sizeof(int64_t) * (size_t)ld * M);
  if (out->g) memcpy(out->g, g, sizeof(int64_t) * (size_t)ld);
  if (out->cos_raw) memcpy(out->cos_raw, cr, sizeof(int64_t) * (size_t)M);
  if (out->sin_raw) memcpy(out->sin_raw, sr, sizeof(int64_t) * (size_t)M);

done:
  free(basis); free(hess); free(g); free(cr); free(sr); free(w); free(w2);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* solve (refine.cpp:21-106), fixed_point engine                             */

int ora_solve(const ora_split* m, const ora_csrf* a_fp, const double* b,
              const ora_refine_cfg* cfg, const ora_ilu* precond, double* x,
              ora_report* rep, ora_trace* ext) {
  const int n = m->n;
  if (a_fp->n != n) return fail(ORA_INVALID_ARGUMENT, "solve: dimension mismatch");
  if (cfg->max_refinements < 0)
    return fail(ORA_INVALID_ARGUMENT, "solve: max_refinements must be >= 0");
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);

  ora_trace own;
  memset(&own, 0, sizeof own);
  own.checked = cfg->checked;
  ora_trace* t = ext ? ext : &own;

  rep->converged = 0;
  rep->refinements = 0;
  rep->total_inner_iterations = 0;
  rep->n_relres = 0;
  for (int i = 0; i < n; ++i) x[i] = 0.0;

  double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* bk = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* zeros = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* corr = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  const int M = cfg->m > 0 ? cfg->m : 1;
  double* gabs = (double*)malloc(sizeof(double) * (size_t)M);
  double* cd = (double*)malloc(sizeof(double) * (size_t)M);
  double* sd = (double*)malloc(sizeof(double) * (size_t)M);
  int rc = ORA_OK;

  double relnorm = ora_residual_fp(a_fp, x, b, r);
  rep->relres_history[rep->n_relres++] = relnorm;

  for (int k = 0; k < cfg->max_refinements && relnorm >= cfg->tol; ++k) {
    double rmax = 0.0;
    for (int i = 0; i < n; ++i) { const double a = fabs(r[i]); rmax = (rmax < a) ? a : rmax; }
    if (rmax == 0.0) break;
    double gamma;
    if ((rc = ora_gamma_scale(n, r, &gamma, bk))) break;
    t->restart = k;
    const uint64_t before = t->total;
    const int depth = cfg->s_schedule ? cfg->s_schedule[k] : cfg->s;

    ora_cycle_cfg cc;
    memset(&cc, 0, sizeof cc);
    cc.m = cfg->m; cc.frac_bits = cfg->frac_bits; cc.s = depth;
    cc.shifts = cfg->shifts; cc.precond = precond;
    ora_cycle_out co;
    memset(&co, 0, sizeof co);
    co.g_abs = gabs; co.cos_d = cd; co.sin_d = sd;
    if ((rc = ora_run_cycle(m, &cc, bk, zeros, corr, &co, t))) break;
    const int dim = co.dim;
    if (dim == 0) break;

    for (int i = 0; i < n; ++i) x[i] += gamma * corr[i];
    rep->refinements = k + 1;
    rep->total_inner_iterations += dim;
    rep->inner_dims[k] = dim;
    rep->gamma_history[k] = gamma;
    rep->overflow_per_restart[k] = t->total - before;

    relnorm = ora_residual_fp(a_fp, x, b, r);
    rep->relres_history[rep->n_relres++] = relnorm;
  }
  rep->converged = relnorm < cfg->tol;
  rep->overflow_total = t->total;
  clock_gettime(CLOCK_MONOTONIC, &t1);
  rep->wall_time_sec = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(r); free(bk); free(zeros); free(corr); free(gabs); free(cd); free(sd);
  return rc;
}
