/*
 * igm_oracle.h -- CPU restatement of the reference int-GMRES hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2009_07495_b200/)
 * may include, link or call this.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker.
 *
 * Every function restates the reference algorithm in plain C99 (+ gcc's
 * __builtin_*_overflow and __int128), citing the reference file:line it
 * follows (paths relative to /root/reference/proj/core).  Floating-point code
 * is compiled with -ffp-contract=off and no -march, i.e. the same SSE2
 * mulsd/addsd sequence the reference library is built to.
 *
 * Pinning: tests/test_oracle_kats.py checks this file against every known-
 * answer value in the reference's own unit tests (tests/golden/kats.json) and
 * tests/test_oracle_vs_ref.py replays it against the reference library itself
 * compiled from /root/reference into oracle/_ref/ (see oracle/Makefile).
 */
#ifndef IGM_ORACLE_H
#define IGM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes mirror the reference's exception types */
enum {
  ORA_OK = 0,
  ORA_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  ORA_DOMAIN_ERROR = 2,     /* std::domain_error */
  ORA_OVERFLOW_ERROR = 3,   /* std::overflow_error */
  ORA_RUNTIME_ERROR = 4,    /* std::runtime_error */
  ORA_LOGIC_ERROR = 5       /* std::logic_error */
};

/* kernel tags set by run_cycle (gmres_int.cpp:91-149) */
enum {
  ORA_K_NONE = 0, ORA_K_SPMV = 1, ORA_K_PRECOND = 2, ORA_K_DOT = 3,
  ORA_K_AXPY = 4, ORA_K_NORM = 5, ORA_K_VEC_DIV = 6, ORA_K_GIVENS = 7,
  ORA_K_GIVENS_NORM = 8, ORA_K_GIVENS_DIV = 9, ORA_K_ROT = 10
};
/* primitive op tags (fxp.hpp:121-152) */
enum { ORA_OP_ADD = 1, ORA_OP_SUB = 2, ORA_OP_MUL = 3, ORA_OP_SHL = 4, ORA_OP_DIV = 5 };

/* FxTrace restated (fxp.hpp:51-103). */
typedef struct {
  int checked;
  int record_shifts;
  int kernel, restart, step; /* current location */
  uint64_t total;            /* total overflow events */
  int n_events, cap_events;  /* events stored (<= cap) */
  int32_t* events;           /* 4 ints each: kernel, op, restart, step */
  int64_t n_shifts;          /* shift records seen (may exceed cap) */
  int cap_shifts;
  int32_t* shifts;           /* 3 ints each: kernel, b1, b2 */
} ora_trace;

typedef struct {
  int dot_b1, dot_b2, axpy_b1, norm_b1, div_b1, div_b2, givens_b2, rot_b;
} ora_shifts;

typedef struct { /* CsrMatrixF (csr.hpp:10-18) */
  int n;
  const int* row_ptr;
  const int* col_idx;
  const double* vals;
} ora_csrf;

typedef struct { /* SplitMatrix (split.hpp:28-37): components share one pattern */
  int n, nnz, ncomp;
  const int* row_ptr;
  const int* col_idx;
  const int64_t* vals; /* ncomp * nnz, component-major */
  const int* alphas;   /* ncomp */
} ora_split;

typedef struct { /* IluFactors (ilu.hpp:27-32) */
  int n;
  const int *l_row_ptr, *l_col_idx, *l_diag_pos;
  const int64_t* l_vals;
  const int *u_row_ptr, *u_col_idx, *u_diag_pos;
  const int64_t* u_vals;
} ora_ilu;

const char* ora_last_error(void);

/* ---- scalar fixed point (fxp.hpp:105-234, fxp.cpp:20-47) ---- */
int64_t ora_asr(int64_t x, int s);
int64_t ora_wrap_shl(int64_t x, int s);
int ora_encode(double x, int frac_bits, int64_t* out);
double ora_decode(int64_t raw, int frac_bits);
int ora_fx_add(int64_t a, int64_t b, int64_t* out, ora_trace* t);
int ora_fx_sub(int64_t a, int64_t b, int64_t* out, ora_trace* t);
int ora_fx_mul(int64_t a, int64_t b, int f, int b1, int b2, int out_frac,
               int64_t* out, ora_trace* t);
int ora_fx_div(int64_t a, int64_t b, int f, int b1, int b2, int64_t* out,
               ora_trace* t);
uint64_t ora_isqrt(uint64_t v);
int ora_fx_sqrt(int64_t a, int fin, int out_frac, int64_t* out, ora_trace* t);
int ora_shifts_validate(const ora_shifts* sp, int f);
void ora_shifts_default_unpreconditioned(int f, ora_shifts* out);
void ora_shifts_default_preconditioned(int f, ora_shifts* out);

/* ---- vector kernels (fxp.cpp:49-104) ---- */
int ora_fx_dot(int64_t n, const int64_t* v, const int64_t* w, int f, int b1,
               int b2, int64_t* out, ora_trace* t);
int ora_fx_norm(int64_t n, const int64_t* v, int f, int b1, int64_t* out,
                ora_trace* t);
int ora_fx_axpy_sub(int64_t n, int64_t* w, int64_t h, const int64_t* v, int f,
                    int b1, ora_trace* t);

/* ---- operators (split.cpp, ilu.cpp) ---- */
int ora_spmv(const ora_split* m, int s, const int64_t* v, int64_t* out,
             ora_trace* t);
int ora_apply_inverse(const ora_ilu* f, const int64_t* y, int64_t* out,
                      ora_trace* t);
int ora_apply_inverse_fp(const ora_ilu* f, const double* y, double* out);
void ora_spmv_fp_csr(const ora_csrf* a, const double* x, double* y);
int ora_spmv_fp_split(const ora_split* m, int s, const double* x, double* y);
double ora_norm2(int64_t n, const double* v);
double ora_residual_fp(const ora_csrf* a, const double* x, const double* b,
                       double* r);
int ora_gamma_scale(int64_t n, const double* r, double* gamma, double* b_k);

/* ---- host setup (split.cpp:61-135, ilu.cpp:25-120) ---- */
int ora_row_scale(const ora_csrf* a, int alpha_a, double* vals_out,
                  double* scale_out);
/* comp_vals_out: max_components * nnz; returns ncomp, exact */
int ora_build_split(int n, int nnz, const double* vals, int alpha_a,
                    int max_components, int64_t* comp_vals_out,
                    int* alphas_out, int* ncomp_out, int* exact_out);
/* Lower/upper patterns are A's entries with j<=i / j>=i (diag stored).
 * Outputs sized: l_row_ptr/u_row_ptr n+1; l_col/l_vals/u_col/u_vals nnz(A)
 * upper bounds; diag_fp n. */
int ora_factorize_split_cast(const ora_csrf* a, int* l_row_ptr, int* l_col_idx,
                             int64_t* l_vals, int* l_diag_pos, int* u_row_ptr,
                             int* u_col_idx, int64_t* u_vals, int* u_diag_pos);

/* ---- Givens / Hessenberg (gmres_int.cpp:8-40) ---- */
int ora_apply_stored_rotations(int64_t* h_col, int count, const int64_t* c,
                               const int64_t* s, int givens_b2, int f,
                               ora_trace* t);
int ora_solve_hessenberg(const double* r_cols, int ld, int dim, const double* g,
                         double* y);

/* ---- one int-GMRES(m) cycle (gmres_int.cpp:42-196) ---- */
typedef struct {
  int m, frac_bits, s;
  ora_shifts shifts;
  const ora_ilu* precond; /* NULL = none */
  int collect_basis_norms;
} ora_cycle_cfg;

typedef struct { /* CycleDiagnostics + ArnoldiState, caller-allocated */
  int dim;
  double r0_norm;
  double* g_abs;       /* m */
  double* cos_d;       /* m */
  double* sin_d;       /* m */
  double* basis_norms; /* m+1 or NULL */
  int n_basis_norms;
  /* ArnoldiState: any may be NULL */
  int64_t* basis; /* (m+1)*n */
  int n_basis;
  int64_t* hess;  /* (m+1)*m column-major, ld=m+1 */
  int64_t* g;     /* m+1 */
  int64_t* cos_raw, *sin_raw; /* m */
} ora_cycle_out;

int ora_run_cycle(const ora_split* m, const ora_cycle_cfg* cfg, const double* b,
                  const double* x0, double* x_out, ora_cycle_out* out,
                  ora_trace* t);

/* ---- iterative refinement (refine.cpp:21-106) ---- */
typedef struct {
  double tol;
  int max_refinements, m, frac_bits, s, checked;
  ora_shifts shifts;
  const int* s_schedule; /* NULL or max_refinements entries */
} ora_refine_cfg;

typedef struct { /* SolveReport, caller-allocated arrays of max_refinements(+1) */
  int converged, refinements;
  int64_t total_inner_iterations;
  int* inner_dims;
  double* relres_history; /* max_refinements + 1 */
  int n_relres;
  double* gamma_history;
  uint64_t* overflow_per_restart;
  uint64_t overflow_total;
  double wall_time_sec;
} ora_report;

int ora_solve(const ora_split* m, const ora_csrf* a_fp, const double* b,
              const ora_refine_cfg* cfg, const ora_ilu* precond, double* x_out,
              ora_report* rep, ora_trace* external_trace);

#ifdef __cplusplus
}
#endif
#endif
