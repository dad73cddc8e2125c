/*
 * igm_oracle32.c -- CPU restatement of the int-GMRES hot path at WORD LENGTH
 * 32 (BASELINE.json config 3, "WL=32 fixed point").
 *
 * TEST INFRASTRUCTURE ONLY (see igm_oracle.h).  The product never links this.
 *
 * PARITY UNPINNED: the reference hard-wires WL = 64 (fxp.hpp:22; WL != 64 is
 * a SPEC.md:149 non-goal), so no reference code or test pins this file.  It
 * restates the reference's WL = 64 algorithm (the citations below, into
 * /root/reference/proj/core/) with every word an int32 and every wrap mod
 * 2^32, which is the paper's intWL arithmetic for WL = 32 (PAPER.md
 * "Basic Arithmetic of Fixed-Point Numbers": shifts, products and sums all
 * in the intWL type).  Its WL = 64-shaped structure is checked against the
 * pinned WL = 64 restatement by tests/test_wl32.py (same control flow).
 * Floating-point parts (residual, norm2, gamma scaling, Hessenberg solve,
 * x update) are the WL = 64 ones, word-length independent.
 */
#include "igm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- intWL primitives at WL = 32 (fxp.hpp:105-163 with 64 -> 32) ---- */
static int32_t asr32(int32_t x, int s) { /* fxp.hpp:108-111 */
  if (s >= 31) return x >> 31;
  return x >> s;
}
static int32_t shl32(int32_t x, int s) { /* fxp.hpp:114-117 */
  if (s >= 32) return 0;
  return (int32_t)((uint32_t)x << s);
}
typedef struct { uint64_t n; } cnt32; /* overflow events (checked mode) */
/* diagnostics: events by kernel of the last run_cycle (spmv, dot, axpy, norm, div, givens, rot) */
static uint64_t g_k32[8];
static int g_kk = 0;
uint64_t ora32_kernel_events(int k) { return k >= 0 && k < 8 ? g_k32[k] : 0; }
#define KSET(k) (g_kk = (k))
static int32_t add32(int32_t a, int32_t b, cnt32* c) {
  int32_t r;
  if (__builtin_add_overflow(a, b, &r) && c) { c->n++; g_k32[g_kk]++; }
  return r;
}
static int32_t sub32(int32_t a, int32_t b, cnt32* c) {
  int32_t r;
  if (__builtin_sub_overflow(a, b, &r) && c) { c->n++; g_k32[g_kk]++; }
  return r;
}
static int32_t mul32(int32_t a, int32_t b, cnt32* c) {
  int32_t r;
  if (__builtin_mul_overflow(a, b, &r) && c) { c->n++; g_k32[g_kk]++; }
  return r;
}
static int32_t shlc32(int32_t x, int s, cnt32* c) { /* fxp.hpp:139-143 */
  const int32_t r = shl32(x, s);
  if (asr32(r, s) != x && c) { c->n++; g_k32[g_kk]++; }
  return r;
}
static int32_t div32(int32_t num, int32_t den, cnt32* c) { /* fxp.hpp:145-152 */
  if (num == INT32_MIN && den == -1) {
    if (c) { c->n++; g_k32[g_kk]++; }
    return num;
  }
  return num / den;
}

static char g_err32[256];
const char* ora32_last_error(void) { return g_err32; }
static int fail32(int code, const char* msg) {
  snprintf(g_err32, sizeof g_err32, "%s", msg);
  return code;
}

int ora32_encode(double x, int f, int32_t* out) { /* fxp.hpp:171-176 */
  if (!(fabs(x) < ldexp(1.0, 32 - 1 - f)))
    return fail32(ORA_OVERFLOW_ERROR, "encode: value outside representable range");
  *out = (int32_t)ldexp(x, f);
  return ORA_OK;
}
double ora32_decode(int32_t raw, int f) { return ldexp((double)raw, -f); } /* fxp.hpp:180-182 */

uint32_t ora32_isqrt(uint32_t v) { /* fxp.cpp:20-33 (floor sqrt is unique) */
  if (v == 0) return 0;
  uint64_t x = (uint64_t)sqrt((double)v);
  while (x * x > v) --x;
  while ((x + 1) * (x + 1) <= v) ++x;
  return (uint32_t)x;
}

static int32_t fx_mul32(int32_t a, int32_t b, int f, int b1, int b2, cnt32* c) { /* fxp.hpp:203-216, out = f */
  const int post = 2 * f - b1 - b2 - f;
  return asr32(mul32(asr32(a, b1), asr32(b, b2), c), post);
}
static int fx_div32(int32_t a, int32_t b, int f, int b1, int b2, int32_t* out, cnt32* c) { /* fxp.hpp:220-234 */
  const int32_t num = shlc32(a, b1, c);
  const int32_t den = asr32(b, b2);
  if (den == 0) return fail32(ORA_DOMAIN_ERROR, "fx_div: shifted divisor is zero");
  const int32_t q = div32(num, den, c);
  const int e = f - b1 - b2;
  *out = e >= 0 ? shlc32(q, e, c) : asr32(q, -e);
  return ORA_OK;
}
static int fx_sqrt32(int32_t a, int fin, int f, int32_t* out, cnt32* c) { /* fxp.cpp:35-47 */
  if (a < 0) return fail32(ORA_DOMAIN_ERROR, "fx_sqrt: negative input");
  const int32_t r = (int32_t)ora32_isqrt((uint32_t)a);
  const int e = f - fin / 2;
  *out = e >= 0 ? shlc32(r, e, c) : asr32(r, -e);
  return ORA_OK;
}

int ora32_shifts_validate(const ora_shifts* p, int f) { /* fxp.cpp:106-127 at WL = 32 */
  if (f < 0 || f > 30) return fail32(ORA_INVALID_ARGUMENT, "QFormat: frac_bits must be in [0, 30]");
#define RIGHT(b, name)                      \
  if ((b) < 0 || ((b) > 0 && (b) >= f)) return fail32(ORA_INVALID_ARGUMENT, "ShiftPlan: " name " must lie in [0, frac_bits)");
  RIGHT(p->dot_b1, "dot_b1");
  RIGHT(p->dot_b2, "dot_b2");
  RIGHT(p->axpy_b1, "axpy_b1");
  RIGHT(p->norm_b1, "norm_b1");
  RIGHT(p->div_b2, "div_b2");
  RIGHT(p->givens_b2, "givens_b2");
#undef RIGHT
  if (p->div_b1 < 0 || p->div_b1 > f) return fail32(ORA_INVALID_ARGUMENT, "ShiftPlan: div_b1 must lie in [0, frac_bits]");
  /* WL = 32 departs from the WL = 64 rule rot_b == 0 (fxp.cpp:125): two Q.f
   * words of magnitude ~1 multiply to 2^(2f), which needs rot_b >= f - 15 */
  if (p->rot_b < 0 || (p->rot_b > 0 && p->rot_b >= f))
    return fail32(ORA_INVALID_ARGUMENT, "ShiftPlan: rot_b must lie in [0, frac_bits)");
  if (2 * (f - p->norm_b1) > 30)
    return fail32(ORA_INVALID_ARGUMENT, "ShiftPlan: norm accumulator needs 2*(frac_bits - norm_b1) <= 30");
  return ORA_OK;
}

/* ---- vector kernels (fxp.cpp:49-104 at WL = 32) ---- */
static int32_t fx_dot32(int64_t n, const int32_t* v, const int32_t* w, int f, int b1, int b2, cnt32* c) {
  int32_t acc = 0;
  for (int64_t l = 0; l < n; ++l) acc = add32(acc, mul32(asr32(v[l], b1), asr32(w[l], b2), c), c);
  const int e = f - b1 - b2;
  return e >= 0 ? asr32(acc, e) : shlc32(acc, -e, c);
}
static int fx_norm32(int64_t n, const int32_t* v, int f, int b1, int32_t* out, cnt32* c) {
  int32_t acc = 0;
  for (int64_t l = 0; l < n; ++l) {
    const int32_t s = asr32(v[l], b1);
    acc = add32(acc, mul32(s, s, c), c);
  }
  if (acc < 0) return fail32(ORA_DOMAIN_ERROR, "fx_norm: accumulator wrapped negative");
  return fx_sqrt32(acc, 2 * (f - b1), f, out, c);
}
static void fx_axpy32(int64_t n, int32_t* w, int32_t h, const int32_t* v, int f, int b1, cnt32* c) {
  const int post = f - b1;
  const int32_t hs = asr32(h, b1);
  for (int64_t l = 0; l < n; ++l) w[l] = sub32(w[l], asr32(mul32(hs, v[l], c), post), c);
}
/* split.cpp:137-157 at WL = 32 */
int ora32_spmv(int n, const int* rp, const int* ci, const int32_t* vals, int nnz, int ncomp, const int* alphas, int s,
               const int32_t* v, int32_t* out, uint64_t* ovf) {
  cnt32 c = {0};
  for (int i = 0; i < n; ++i) out[i] = 0;
  for (int l = 0; l <= s && l < ncomp; ++l) {
    const int32_t* cv = vals + (int64_t)l * nnz;
    for (int i = 0; i < n; ++i) {
      int32_t acc = 0;
      for (int k = rp[i]; k < rp[i + 1]; ++k) acc = add32(acc, mul32(cv[k], v[ci[k]], &c), &c);
      out[i] = add32(out[i], asr32(acc, alphas[l]), &c);
    }
  }
  if (ovf) *ovf = c.n;
  return ORA_OK;
}

/* run_cycle (gmres_int.cpp:42-196), unpreconditioned, at WL = 32.  x += the
 * correction.  Outputs: dim, r0 norm, the basis (n_basis x n int32), H
 * (column-major, ld = m+1), g, cos, sin (raw), overflow events (total). */
typedef struct {
  int m, f, s, checked;
  ora_shifts sh;
} ora32_cycle_cfg;

int ora32_run_cycle(int n, const int* rp, const int* ci, const int32_t* vals, int nnz, int ncomp, const int* alphas,
                    const ora32_cycle_cfg* cfg, const double* b, double* x, int* dim_out, double* r0n_out,
                    int32_t* basis_out, int* nbasis_out, int32_t* hess_out, int32_t* g_out, int32_t* cos_out,
                    int32_t* sin_out, uint64_t* ovf_out) {
  const int M = cfg->m, f = cfg->f;
  const ora_shifts* sp = &cfg->sh;
  int rc;
  if (M < 1) return fail32(ORA_INVALID_ARGUMENT, "run_cycle: m must be >= 1");
  if ((rc = ora32_shifts_validate(sp, f))) return rc;
  cnt32 cc = {0};
  cnt32* c = cfg->checked ? &cc : NULL;
  *dim_out = 0;
  *nbasis_out = 0;
  /* r0 = b (x0 = 0 in the refinement loop), gmres_int.cpp:61-70 */
  const double r0n = ora_norm2(n, b);
  *r0n_out = r0n;
  if (r0n == 0.0) return ORA_OK;
  const int ld = M + 1;
  int32_t* basis = (int32_t*)calloc((size_t)(M + 1) * (size_t)n + 1, sizeof(int32_t));
  int32_t* hess = (int32_t*)calloc((size_t)ld * M, sizeof(int32_t));
  int32_t* g = (int32_t*)calloc((size_t)ld, sizeof(int32_t));
  int32_t* cr = (int32_t*)calloc((size_t)M, sizeof(int32_t));
  int32_t* sr = (int32_t*)calloc((size_t)M, sizeof(int32_t));
  int32_t* w = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) /* gmres_int.cpp:77-81 */
    if ((rc = ora32_encode(b[i] / r0n, f, &basis[i]))) goto done;
  int nb = 1;
  g[0] = (int32_t)1 << f;
  int dim = 0;
  for (int j = 0; j < M; ++j) { /* gmres_int.cpp:90-160 */
    int32_t* col = &hess[(size_t)j * ld];
    uint64_t so = 0;
    if (j == 0) memset(g_k32, 0, sizeof g_k32);
    KSET(0);
    ora32_spmv(n, rp, ci, vals, nnz, ncomp, alphas, cfg->s, basis + (size_t)j * n, w, &so);
    if (c) c->n += so;
    g_k32[0] += so;
    for (int i = 0; i <= j; ++i) {
      const int32_t* vi = basis + (size_t)i * n;
      KSET(1);
      const int32_t hij = fx_dot32(n, w, vi, f, sp->dot_b1, sp->dot_b2, c);
      col[i] = hij;
      KSET(2);
      fx_axpy32(n, w, hij, vi, f, sp->axpy_b1, c);
    }
    int32_t hnext;
    KSET(3);
    if ((rc = fx_norm32(n, w, f, sp->norm_b1, &hnext, c))) goto done;
    col[j + 1] = hnext;
    const int happy = hnext == 0;
    KSET(4);
    if (!happy) {
      int32_t* vn = basis + (size_t)(j + 1) * n;
      for (int l = 0; l < n; ++l)
        if ((rc = fx_div32(w[l], hnext, f, sp->div_b1, sp->div_b2, &vn[l], c))) goto done;
      nb++;
    }
    KSET(5);
    for (int i = 0; i < j; ++i) { /* apply_stored_rotations, gmres_int.cpp:8-25 */
      const int32_t a = fx_mul32(cr[i], col[i], f, 0, sp->givens_b2, c);
      const int32_t bb = fx_mul32(sr[i], col[i + 1], f, 0, sp->givens_b2, c);
      const int32_t d = fx_mul32(cr[i], col[i + 1], f, 0, sp->givens_b2, c);
      const int32_t e = fx_mul32(sr[i], col[i], f, 0, sp->givens_b2, c);
      col[i] = add32(a, bb, c);
      col[i + 1] = sub32(d, e, c);
    }
    int32_t pair[2] = {col[j], col[j + 1]};
    int32_t tmp;
    if ((rc = fx_norm32(2, pair, f, sp->norm_b1, &tmp, c))) goto done; /* gmres_int.cpp:133-137 */
    if (tmp == 0) break;
    int32_t cc2, s2;
    if ((rc = fx_div32(col[j], tmp, f, sp->div_b1, sp->div_b2, &cc2, c))) goto done;
    if ((rc = fx_div32(col[j + 1], tmp, f, sp->div_b1, sp->div_b2, &s2, c))) goto done;
    cr[j] = cc2;
    sr[j] = s2;
    col[j] = tmp;
    col[j + 1] = 0;
    KSET(6);
    const int32_t g_old = g[j]; /* gmres_int.cpp:150-153 */
    const int32_t neg_s = sub32(0, s2, c);
    g[j + 1] = fx_mul32(neg_s, g_old, f, sp->rot_b, sp->rot_b, c);
    g[j] = fx_mul32(cc2, g_old, f, sp->rot_b, sp->rot_b, c);
    dim = j + 1;
    if (happy) break;
  }
  *dim_out = dim;
  if (dim > 0) { /* gmres_int.cpp:163-180 */
    double* rcols = (double*)calloc((size_t)ld * dim, sizeof(double));
    double* gd = (double*)malloc(sizeof(double) * (size_t)dim);
    double* y = (double*)malloc(sizeof(double) * (size_t)dim);
    for (int j = 0; j < dim; ++j) {
      for (int i = 0; i <= j; ++i) rcols[(size_t)j * ld + i] = ora32_decode(hess[(size_t)j * ld + i], f);
      gd[j] = ora32_decode(g[j], f);
    }
    rc = ora_solve_hessenberg(rcols, ld, dim, gd, y);
    if (!rc) {
      double* corr = (double*)calloc((size_t)n, sizeof(double));
      for (int j = 0; j < dim; ++j) {
        const int32_t* vj = basis + (size_t)j * n;
        const double wj = r0n * y[j];
        for (int l = 0; l < n; ++l) corr[l] += wj * ora32_decode(vj[l], f);
      }
      for (int l = 0; l < n; ++l) x[l] = corr[l];
      free(corr);
    }
    free(rcols);
    free(gd);
    free(y);
  }
  *nbasis_out = nb;
  if (basis_out) memcpy(basis_out, basis, sizeof(int32_t) * (size_t)nb * n);
  if (hess_out) memcpy(hess_out, hess, sizeof(int32_t) * (size_t)ld * M);
  if (g_out) memcpy(g_out, g, sizeof(int32_t) * (size_t)ld);
  if (cos_out) memcpy(cos_out, cr, sizeof(int32_t) * (size_t)M);
  if (sin_out) memcpy(sin_out, sr, sizeof(int32_t) * (size_t)M);
done:
  if (ovf_out) *ovf_out = cc.n;
  free(basis);
  free(hess);
  free(g);
  free(cr);
  free(sr);
  free(w);
  return rc;
}

/* solve (refine.cpp:21-106) with the WL = 32 cycle.  relres / gamma / dims
 * histories (capacity max_ref + 1 / max_ref / max_ref). */
int ora32_solve(int n, const int* rp, const int* ci, const int32_t* vals, int nnz, int ncomp, const int* alphas,
                const ora_csrf* a_fp, const double* b, double tol, int max_ref, const ora32_cycle_cfg* cfg, double* x,
                double* relres, double* gammas, int* dims, int* nref, int* converged, uint64_t* ovf_total) {
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* bk = (double*)malloc(sizeof(double) * (size_t)n);
  double* corr = (double*)malloc(sizeof(double) * (size_t)n);
  int rc = ORA_OK;
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  *ovf_total = 0;
  double rel = ora_residual_fp(a_fp, x, b, r);
  relres[0] = rel;
  int k = 0;
  for (; k < max_ref && rel >= tol; ++k) {
    double gamma;
    if ((rc = ora_gamma_scale(n, r, &gamma, bk))) break;
    int dim, nbv;
    double r0n;
    uint64_t ov = 0;
    rc = ora32_run_cycle(n, rp, ci, vals, nnz, ncomp, alphas, cfg, bk, corr, &dim, &r0n, NULL, &nbv, NULL, NULL, NULL,
                         NULL, &ov);
    *ovf_total += ov;
    if (rc) break;
    if (dim == 0) break;
    for (int i = 0; i < n; ++i) x[i] += gamma * corr[i]; /* refine.cpp:87 */
    gammas[k] = gamma;
    dims[k] = dim;
    rel = ora_residual_fp(a_fp, x, b, r);
    relres[k + 1] = rel;
  }
  *nref = k;
  *converged = rel < tol;
  free(r);
  free(bk);
  free(corr);
  return rc;
}
