/*
 * igm.h -- C ABI of the B200-native int-GMRES hot path (libigm_b200.so).
 *
 * Plain C: opaque handles, plain pointers and sizes, status codes.  No torch,
 * no C++ types.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core/).  The C++ drop-in API in
 * include/intgmres/ (*.hpp) is implemented on top of these calls.
 *
 * Memory: every vector/array argument may be HOST memory or DEVICE memory of
 * the context's GPU; the library detects which (cudaPointerGetAttributes) and
 * stages host buffers through its own device workspace.  Results are written
 * back into the same space the output pointer lives in.  Device buffers are
 * accessed on the context's stream (igm_ctx_stream): the caller orders any
 * producer stream before the call; every call returns with the stream
 * synchronised unless documented otherwise (igm_spmv_mgs with h_out == NULL,
 * igm_mgs_pass).
 *
 * Errors: every call returns igm_status; igm_last_error() returns the message
 * of the last failure on the calling thread.  Status codes map 1:1 onto the
 * reference's exception types; the C++ shim re-throws them.
 *
 * Threading: a context owns one CUDA stream; calls on one context must be
 * serialised by the caller (the reference is single-threaded, FxTrace is not
 * thread-safe).  Uploaded split and FP64 matrices are immutable and may be
 * shared by contexts on the same device; an ILU handle also carries its
 * substitutions' device scratch (wavefront tickets, tagged exported values,
 * magnitude bounds) and must be used by one context at a time.
 */
#ifndef IGM_H
#define IGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IGM_OK = 0,
  IGM_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  IGM_DOMAIN_ERROR = 2,     /* std::domain_error */
  IGM_OVERFLOW_ERROR = 3,   /* std::overflow_error */
  IGM_RUNTIME_ERROR = 4,    /* std::runtime_error */
  IGM_LOGIC_ERROR = 5,      /* std::logic_error */
  IGM_CUDA_ERROR = 6,       /* device / driver failure (no reference analogue) */
  IGM_NCCL_ERROR = 7
} igm_status;

typedef struct igm_ctx igm_ctx;     /* device, stream, workspaces */
typedef struct igm_split igm_split; /* device-resident SplitMatrix */
typedef struct igm_csrf igm_csrf;   /* device-resident CsrMatrixF */
typedef struct igm_ilu igm_ilu;     /* device-resident IluFactors + schedule */

/* ShiftPlan (fxp.hpp:262-278) */
typedef struct {
  int dot_b1, dot_b2, axpy_b1, norm_b1, div_b1, div_b2, givens_b2, rot_b;
} igm_shifts;

/* FxTrace (fxp.hpp:51-103), caller-owned; survives failed calls with its
 * counts updated (test_refine.cpp:175-203).  `exact` is set to 0 when a
 * reduction MAY have wrapped in its running sum, in which case `total`
 * counts the order-free events (mul/sub/shl/div and per-row adds) only. */
typedef struct {
  int checked;       /* in: record overflow events */
  int record_shifts; /* in: log (kernel, b1, b2) per shifted call */
  int kernel, restart, step; /* in/out: current location */
  uint64_t total;    /* in/out: accumulates */
  int n_events, cap_events;
  int32_t* events;   /* 4 ints each: kernel, op, restart, step */
  int64_t n_shifts;
  int cap_shifts;
  int32_t* shifts;   /* 3 ints each: kernel, b1, b2 */
  int exact;         /* out */
} igm_trace;

/* ---- context ---------------------------------------------------------- */
igm_status igm_ctx_create(int device, igm_ctx** out);
void igm_ctx_destroy(igm_ctx* ctx);
igm_status igm_ctx_synchronize(igm_ctx* ctx);
/* CUDA stream (cudaStream_t) the context launches on. */
void* igm_ctx_stream(igm_ctx* ctx);
/* number of kernels this context has launched so far */
uint64_t igm_ctx_launch_count(igm_ctx* ctx);
/* Exact running-sum ("add") overflow events for the fx_dot / fx_norm
 * reductions in checked mode: after every reduction
 * whose sum|term| certificate fails, an exact int128 prefix scan counts the
 * sequential order's wrap crossings, so igm_trace.total / igm_report
 * overflow counts are the reference's in every case (overflow_exact = 1).
 * Off by default (the certificate already proves zero events in configured
 * runs); on, the cycle runs the separate pass kernels. */
igm_status igm_set_exact_overflow_counts(igm_ctx* ctx, int on);
const char* igm_last_error(void);
const char* igm_version(void);
/* Opt-in per-kernel-class device timing (CUDA events around each launch).
 * Classes: 0 spmv_int, 1 ilu_int, 2 ilu_fp, 3 mgs, 4 vec_div, 5 step_scalar,
 * 6 norm2_serial, 7 residual_fp, 8 x_update, 9 encode, 10 other.
 * collect() fills ms[11] and count[11], resets, returns the class count. */
void igm_profile_enable(int on);
int igm_profile_collect(double* ms, uint64_t* count);

/* ---- uploads (the hot path's inputs) ----------------------------------- */
/* SplitMatrix (split.hpp:28-37): ncomp components sharing one CSR pattern;
 * comp_vals is ncomp*nnz int64, component-major; alphas[0] == 0. */
igm_status igm_upload_split(igm_ctx* ctx, int n, int nnz, const int* row_ptr,
                            const int* col_idx, int ncomp,
                            const int64_t* comp_vals, const int* alphas,
                            igm_split** out);
void igm_split_free(igm_split* m);
/* CsrMatrixF (csr.hpp:10-18), the FP64 system matrix of residual_fp. */
igm_status igm_upload_csrf(igm_ctx* ctx, int n, const int* row_ptr,
                           const int* col_idx, const double* vals,
                           igm_csrf** out);
void igm_csrf_free(igm_csrf* a);
/* IluFactors (ilu.hpp:27-32): lower = L*D_l, upper = D_u*U, diagonal stored
 * at diag_pos.  Builds the wavefront schedule and per-row reciprocals. */
igm_status igm_upload_ilu(igm_ctx* ctx, int n, const int* l_row_ptr,
                          const int* l_col_idx, const int64_t* l_vals,
                          const int* l_diag_pos, const int* u_row_ptr,
                          const int* u_col_idx, const int64_t* u_vals,
                          const int* u_diag_pos, igm_ilu** out);
void igm_ilu_free(igm_ilu* f);
/* levels of the forward / backward substitution DAGs (diagnostics) */
int igm_ilu_levels(const igm_ilu* f, int backward);
/* schedule diagnostics: ntiles, nseg, nlevels, maxdeps, grid x/y/z,
 * brick (x*1e6 + y*1e3 + z) */
void igm_ilu_schedule_info(const igm_ilu* f, int backward, int* out8);
/* CPU-only: build + structurally validate the wavefront schedule of one
 * factor (host arrays); returns 0 if valid (info as igm_ilu_schedule_info) */
int igm_debug_tri_schedule(int n, const int* row_ptr, const int* col_idx,
                           const int64_t* vals, const int* diag_pos, int upper,
                           int num_sms, int* out8);
/* bricks of the pencil wavefront that apply_inverse uses for this
 * substitution: the 7-point one (csrc/pencil.hpp, tri_pencil2.cuh) or, for
 * factors of a 27-point stencil, the 27-point one (csrc/pencil27.cuh: selected
 * only when all of its bricks can be resident at once, launched
 * cooperatively); 0 = the generic wavefront */
int igm_ilu_pencil(const igm_ilu* f, int backward);
/* CPU-only: build the pencil record stream of one factor on a gx*gy*gz grid
 * (host arrays); returns 1 if the factor has the 7-point structure, then
 * out4 = {bricks, steps per warp, bricks in x, bricks in y} */
int igm_debug_pencil_stream(int n, const int* row_ptr, const int* col_idx, const int64_t* vals,
                            const int* diag_pos, int upper, int gx, int gy, int gz, int* out4);
/* CPU-only: the 27-point pencil stream (csrc/pencil27.cuh) of one factor on
 * a gx*gy*gz grid; returns 1 if every entry is one of the 13 lower 27-point
 * neighbours, then out2 = {bricks, stream bytes / 64} */
int igm_debug_pencil27_stream(int n, const int* row_ptr, const int* col_idx, const int64_t* vals,
                              const int* diag_pos, int upper, int gx, int gy, int gz, long long* out2);
/* debug: per-segment phase timestamps of one ILU tile (8 u64 per segment) */
void igm_debug_tri_trace(int tile, unsigned long long* device_buf);
/* debug: per-CTA phase timestamps (ns) of Arnoldi step j of the register
 * resident MGS kernel; out == NULL arms, then out reads cap words and disarms;
 * returns the slots per CTA */
int igm_debug_arn_ts(int j, unsigned long long* out, int cap);
/* debug: the device fast paths of the scalar fixed-point helpers on n input
 * pairs (a_i, b_i): out[4i..4i+3] = isqrt(a), division magic of b,
 * trunc(a / b) as int64, floor(((a mod b) * 2^64 + (~a ^ b)) / b); 0 = ok */
int igm_debug_fx_selftest(int n, const uint64_t* a, const uint64_t* b, uint64_t* out);

/* ---- primitives (parity entry points) ---------------------------------- */
/* replaces intgmres::spmv (split.hpp:48-49, split.cpp:137-157) */
igm_status igm_spmv(igm_ctx* ctx, const igm_split* m, int s, const int64_t* v,
                    int64_t* out, igm_trace* t);
/* replaces intgmres::apply_inverse (ilu.hpp:40-41, ilu.cpp:122-155) */
igm_status igm_apply_inverse(igm_ctx* ctx, const igm_ilu* f, const int64_t* y,
                             int64_t* out, igm_trace* t);
/* replaces intgmres::apply_inverse_fp (ilu.hpp:44-45, ilu.cpp:157-180) */
igm_status igm_apply_inverse_fp(igm_ctx* ctx, const igm_ilu* f,
                                const double* y, double* out);
/* replaces intgmres::fx_dot / fx_norm / fx_axpy_sub (fxp.hpp:248-257) */
igm_status igm_fx_dot(igm_ctx* ctx, int64_t n, const int64_t* v,
                      const int64_t* w, int frac_bits, int b1, int b2,
                      int64_t* out, igm_trace* t);
igm_status igm_fx_norm(igm_ctx* ctx, int64_t n, const int64_t* v,
                       int frac_bits, int b1, int64_t* out, igm_trace* t);
igm_status igm_fx_axpy_sub(igm_ctx* ctx, int64_t n, int64_t* w, int64_t h,
                           const int64_t* v, int frac_bits, int b1,
                           igm_trace* t);
/* replaces intgmres::spmv_fp(CsrMatrixF) and residual_fp (csr.hpp:36-44) */
igm_status igm_spmv_fp(igm_ctx* ctx, const igm_csrf* a, const double* x,
                       double* y);
igm_status igm_residual_fp(igm_ctx* ctx, const igm_csrf* a, const double* x,
                           const double* b, double* r, double* relnorm);
/* replaces intgmres::spmv_fp(SplitMatrix, s, x) (split.hpp:53-54) */
igm_status igm_spmv_fp_split(igm_ctx* ctx, const igm_split* m, int s,
                             const double* x, double* y);
/* replaces intgmres::norm2 (csr.hpp:31): the sequential FP64 chain */
igm_status igm_norm2(igm_ctx* ctx, int64_t n, const double* v, double* out);
/* replaces intgmres::gamma_scale (refine.hpp:61, refine.cpp:11-19) */
igm_status igm_gamma_scale(igm_ctx* ctx, int64_t n, const double* r,
                           double* gamma, double* b_k);

/* ---- the cycle and the solve ------------------------------------------- */
/* CycleConfig (gmres_int.hpp:18-25) */
typedef struct {
  int m, frac_bits, s;
  igm_shifts shifts;
  const igm_ilu* precond; /* NULL = unpreconditioned */
  int collect_basis_norms;
} igm_cycle_cfg;

/* CycleDiagnostics + ArnoldiState (gmres_int.hpp:27-44); host arrays sized
 * by the caller, any may be NULL. */
typedef struct {
  int dim;
  double r0_norm;
  double* g_abs;       /* m */
  double* cos_d;       /* m */
  double* sin_d;       /* m */
  double* basis_norms; /* m+1 */
  int n_basis_norms;
  int64_t* basis;      /* (m+1)*n */
  int n_basis;
  int64_t* hess;       /* (m+1)*m, column-major, ld = m+1 */
  int64_t* g;          /* m+1 */
  int64_t* cos_raw;    /* m */
  int64_t* sin_raw;    /* m */
} igm_cycle_out;

/* replaces intgmres::run_cycle (gmres_int.hpp:51-54, gmres_int.cpp:42-196) */
igm_status igm_run_cycle(igm_ctx* ctx, const igm_split* m,
                         const igm_cycle_cfg* cfg, const double* b,
                         const double* x0, double* x_out, igm_cycle_out* out,
                         igm_trace* t);

/* RefineConfig (refine.hpp:24-34).  The per-refinement depth schedule (a
 * std::function in the reference, consulted once per refinement that runs,
 * refine.cpp:61) is either a callback or an array indexed by refinement;
 * with neither, the constant s is used. */
typedef int (*igm_schedule_fn)(void* user, int k);
typedef struct {
  double tol;
  int max_refinements, m, frac_bits, s, checked;
  igm_shifts shifts;
  const int* s_schedule;         /* NULL or max_refinements entries */
  igm_schedule_fn s_schedule_fn; /* NULL or callback, wins over the array */
  void* s_schedule_user;
  int engine; /* 0 = Engine::fixed_point, 1 = Engine::floating_point (refine.hpp:22):
                 FP64 GMRES(m) on reconstruct_fp(m, s) (refsolve.cpp:9-105) */
} igm_refine_cfg;

/* SolveReport (refine.hpp:36-47); arrays sized max_refinements (+1). */
typedef struct {
  int converged, refinements;
  int64_t total_inner_iterations;
  int* inner_dims;
  double* relres_history;
  int n_relres;
  double* gamma_history;
  uint64_t* overflow_per_restart;
  uint64_t overflow_total;
  double wall_time_sec;
  int overflow_exact; /* 0 if a reduction may have wrapped (see igm_trace) */
} igm_report;

/* replaces intgmres::solve (refine.hpp:67-70, refine.cpp:21-106) */
igm_status igm_solve(igm_ctx* ctx, const igm_split* m, const igm_csrf* a_fp,
                     const double* b, const igm_refine_cfg* cfg,
                     const igm_ilu* precond, double* x_out, igm_report* rep,
                     igm_trace* external_trace);

/* ---- config 3's WL = 32 variant ----------------------------------------- */
/* The int-GMRES cycle with 32-bit words (BASELINE.json config 3, "WL=32 fixed
 * point").  The reference has no WL != 64 code (fxp.hpp:22, a SPEC.md:149
 * non-goal), so these entries replace no reference function: they are the
 * reference's unpreconditioned run_cycle / solve (gmres_int.cpp:42-196,
 * refine.cpp:21-106) with every word an int32 and every wrap mod 2^32, checked
 * against the CPU restatement oracle/igm_oracle32.c (parity unpinned).  One
 * departure from the WL = 64 ShiftPlan rules: rot_b may be > 0 (two Q.f words
 * of magnitude ~1 multiply to 2^(2f), which needs rot_b >= f - 15). */
typedef struct igm_split32 igm_split32;
/* the int64 components of an uploaded split narrowed to int32 (the CSR
 * pattern is shared); IGM_OVERFLOW_ERROR if a value does not fit */
igm_status igm_split32_from_split(igm_ctx* ctx, const igm_split* m, igm_split32** out);
void igm_split32_free(igm_split32* m);
typedef struct {
  int m, frac_bits, s, checked;
  igm_shifts shifts;
} igm_cycle32_cfg;
/* the builder's WL = 32 shift plan for n rows, matrix scaling alpha_a (the
 * split's) and frac_bits: each shift keeps its operands and sums inside 31
 * bits with the headroom of a sum of n terms */
igm_status igm_shifts32_plan(long long n, int alpha_a, int frac_bits, igm_shifts* out);
/* one cycle from x0 = 0; any output may be NULL: basis ((m+1)*n), hess
 * ((m+1)*m, column-major), g (m+1), cos_raw / sin_raw (m) */
igm_status igm_run_cycle32(igm_ctx* ctx, const igm_split32* m, const igm_cycle32_cfg* cfg, const double* b,
                           double* x_out, int* dim, double* r0_norm, int32_t* basis, int* n_basis, int32_t* hess,
                           int32_t* g, int32_t* cos_raw, int32_t* sin_raw, uint64_t* overflows);
/* the refinement loop (refine.cpp:21-106) around the WL = 32 cycle; report
 * arrays as in igm_solve (overflow_exact = 0 when a reduction may have wrapped) */
igm_status igm_solve32(igm_ctx* ctx, const igm_split32* m, const igm_csrf* a_fp, const double* b, double tol,
                       int max_refinements, const igm_cycle32_cfg* cfg, double* x_out, igm_report* rep);

/* replaces intgmres::fp_cycle (refsolve.hpp:26-29, refsolve.cpp:9-105): one
 * FP64 GMRES(m) cycle from x0 on a, with an optional LEFT preconditioner
 * given as a host callback (in/out host buffers of n doubles; returns 0 on
 * success).  Outputs: x_out (n), dim, r0_norm (preconditioned), g_abs (m,
 * may be NULL).  SpMV, norms, scalings and updates follow the reference's
 * order; the MGS dots are deterministic tree reductions. */
typedef int (*igm_fp_precond_fn)(void* user, int64_t n, const double* in, double* out);
igm_status igm_fp_cycle(igm_ctx* ctx, const igm_csrf* a, int m, const double* b,
                        const double* x0, igm_fp_precond_fn precond, void* user,
                        double* x_out, int* dim, double* r0_norm, double* g_abs);

/* ---- kernel microbench (BASELINE config 5) ------------------------------ */
/* One call = w = spmv(m, s, v_in); then for i in 0..k-1:
 * h_i = fx_dot(w, basis_i, dot_b1, dot_b2); fx_axpy_sub(w, h_i, basis_i,
 * axpy_b1) -- unchecked (FxTrace* = nullptr).  basis is k*n device int64,
 * v_in/w device.  h_out: k host int64 (may be NULL). */
igm_status igm_spmv_mgs(igm_ctx* ctx, const igm_split* m, int s,
                        const int64_t* v_in, const int64_t* basis, int k,
                        int frac_bits, int dot_b1, int dot_b2, int axpy_b1,
                        int64_t* w, int64_t* h_out);

/* One fused MGS pass of the config-5 / multi-GPU path on DEVICE pointers,
 * enqueued on the context stream and NOT synchronised (the distributed
 * driver all-reduces *acc_out between passes):
 *   mode 0: *acc_out += sum_l wrap(asr(w_l, dot_b1) * asr(vcur_l, dot_b2))
 *   mode 1: w -= asr(wrap(h * vprev), f - axpy_b1) elementwise with
 *           h = asr(fx_dot finalisation of *hacc, axpy_b1), then mode 0
 *   mode 3: the axpy of mode 1 only
 * (fxp.cpp:49-67, 88-104).  acc_out must be zeroed by the caller; the sum is
 * the wrapping u64 accumulator, so partial sums of row blocks add exactly. */
igm_status igm_mgs_pass(igm_ctx* ctx, int64_t n, int mode, int64_t* w, const int64_t* vprev,
                        const int64_t* vcur, const uint64_t* hacc, uint64_t* acc_out, int f,
                        int dot_b1, int dot_b2, int axpy_b1);

/* ---- row-block (z-slab) partition: rank-local building blocks ----------
 * SURVEY.md 8(e).  The distributed driver (paper_2009_07495_b200/dist.py:
 * solve_sharded) owns the rank's vectors (device pointers) and the
 * collectives (halo planes, exact u64 sums, the relayed norm2 chain, the
 * ILU pipeline hand-offs); each entry below enqueues the same kernels as
 * igm_solve / igm_run_cycle on the context stream and returns WITHOUT
 * synchronising, so a whole cycle is enqueued with no host round trip.
 * igm_dstate holds the replicated per-cycle scalars (Ctl, H, g, cos, sin)
 * and the per-step reduction slots:
 *   RED  step j: (m+2) slots x 3 u64 {wrapped accumulator, sum|t| hi, lo};
 *        slot i <= j: MGS pass i (fx_dot, fxp.cpp:49-67), slot j+1: fx_norm
 *        (fxp.cpp:69-86).  A pass's 3 words are summed over ranks (SUM of
 *        u64 mod 2^64: exact in any order) before the next pass reads them.
 *   LCNT step j: overflow counters of the rank-local kernels [K][OP]; summed
 *        over ranks after the norm pass, before igm_dc_step reads it.
 *   VCNT all steps: vec_div counters, summed once per cycle.
 *   RMAX ctl's max|r| as IEEE bits (int64 MAX over ranks = gamma_scale's max).
 *   CHAIN 4 doubles of scratch for the norm2 relay. */
typedef struct igm_dstate igm_dstate;
enum { IGM_DS_RED = 0, IGM_DS_LCNT = 1, IGM_DS_VCNT = 2, IGM_DS_RMAX = 3, IGM_DS_CHAIN = 4 };
typedef struct {
  int dim, stop, nbasis, add_inexact;
  double r0_norm, relnorm, nb, nr, gamma;
  uint64_t overflows; /* this cycle's events (all-reduced counters + scalar events) */
} igm_dc_info;
igm_status igm_dstate_create(igm_ctx* ctx, int m, igm_dstate** out);
void igm_dstate_free(igm_dstate* d);
igm_status igm_dstate_buffer(igm_dstate* d, int which, int j, void** ptr, int64_t* bytes);
/* ctl := 0 (start of a solve) */
igm_status igm_dc_reset(igm_ctx* ctx, igm_dstate* d);
/* r = b - A x over the rank's rows (A: own rows x extended columns), max|r|
 * into RMAX (residual_fp, split.cpp:51-59; gamma_scale, refine.cpp:11-19) */
igm_status igm_dc_residual(igm_ctx* ctx, igm_dstate* d, const igm_csrf* a, const double* x_ext,
                           const double* b, double* r);
/* norm2 (split.cpp:45-49) continued from *start (device, NULL = 0.0) over n
 * terms; mode 5: *out = running sum; 1: ||b|| (ctl.nb); 2: ||r|| and the
 * relative norm; 3: ||r0|| (stops the cycle when 0) */
igm_status igm_dc_norm2(igm_ctx* ctx, igm_dstate* d, int64_t n, const double* v, const double* start,
                        double* out, int mode);
/* zero the per-cycle state, g_0 = 2^f (gmres_int.cpp:83-89) */
igm_status igm_dc_begin(igm_ctx* ctx, igm_dstate* d, int frac_bits);
/* out = r / gamma (refine.cpp:17-18) */
igm_status igm_dc_scale(igm_ctx* ctx, igm_dstate* d, int64_t n, const double* r, double* out);
/* one FP64 / integer substitution of the (extended-local) factors
 * (ilu.cpp:157-180 / 122-155) */
igm_status igm_dc_tri_fp(igm_ctx* ctx, igm_dstate* d, const igm_ilu* f, int backward, const double* in,
                         double* out);
igm_status igm_dc_tri(igm_ctx* ctx, igm_dstate* d, const igm_ilu* f, int backward, const int64_t* in,
                      int64_t* out, int j, int checked);
/* ---- pipelined z-slab substitutions (the row-partitioned solve)
 * The global ILU(0) on z-slabs: instead of handing a whole boundary plane to
 * the next rank after the substitution finished, every rank's pencil
 * wavefront streams its last own plane, pencil by pencil, as tagged 16-byte
 * words (value, epoch + idx; idx = natural j * gx + i) into the neighbour's
 * import buffer -- a device buffer of the neighbour mapped with CUDA IPC (P2P
 * over NVLink) -- and imports its own halo plane the same way, so rank p's
 * wavefront starts as soon as rank p-1's first pencils finish (the critical
 * path stays the global DAG's, ilu.cpp:122-155).  zimp: this rank's import
 * buffer (NULL: the halo rows' right-hand sides are in `in`); zexp: the
 * neighbour's buffer (NULL: nothing exported); kexp: the solve-order plane
 * exported; epoch: the same value on both ranks for one substitution.
 * Both pencil wavefronts stream: the 7-point one (k_tri_pencil2) and the
 * 27-point one (k_tri27; BASELINE config 4).  IGM_INVALID_ARGUMENT when the
 * rank-local factor is neither (the caller then relays whole planes). */
igm_status igm_dc_tri_piped(igm_ctx* ctx, igm_dstate* d, const igm_ilu* f, int backward, const int64_t* in,
                            int64_t* out, int j, int checked, const void* zimp, void* zexp, int kexp,
                            uint64_t epoch);
/* device buffers shared across processes (CUDA IPC) */
igm_status igm_dev_alloc(igm_ctx* ctx, uint64_t bytes, void** out);
void igm_dev_free(void* p);
igm_status igm_ipc_handle(const void* dptr, unsigned char handle[64]);
igm_status igm_ipc_open(igm_ctx* ctx, const unsigned char handle[64], void** dptr);
void igm_ipc_close(void* dptr);

/* ---- one-shot P2P mailbox reductions -------------------
 * The partitioned cycle needs, after every MGS / norm pass, the SUM over ranks
 * of 3 u64 words (fx_dot / fx_norm accumulators, fxp.cpp:49-86: wrapping sums
 * are exact in any order) before the next pass can derive h_i -- a latency-,
 * not bandwidth-bound exchange.  A mailbox is a device buffer of
 * 2 (parity) x world (sender) x max_words 16-byte words; every rank maps all
 * peers' mailboxes (CUDA IPC between processes, peer access inside one
 * process).  A reduction is two small kernels on the context stream:
 *   publish: stores each word as (value, tag ^ value), tag = f(sequence
 *            number, word index), with one 128-bit store into slot [rank] of
 *            EVERY rank's mailbox (NVLink P2P stores; no reads cross the link);
 *   collect: polls this rank's own mailbox until all `world` senders' words
 *            of this sequence number have arrived (a stale or torn word fails
 *            the tag check), reduces them (lanes = senders, warp shuffles) and
 *            overwrites `words` with the result -- identical on every rank.
 * Ranks issue the same reductions in the same order (the sequence number is
 * counted per mailbox).  Two parities suffice: rank A can publish sequence
 * k+2 only after collecting k+1, which needed B's publish of k+1, which B
 * enqueued after its collect of k.  A sender that never arrives makes the
 * collect give up after `IGM_MBOX_TIMEOUT_MS` (default 20 000): the error is
 * reported by igm_mbox_status / the next igm_mbox_allreduce. */
typedef struct igm_mbox igm_mbox;
enum { IGM_MBOX_SUM = 0 /* u64 mod 2^64 */, IGM_MBOX_MAX = 1 /* signed int64 */ };
enum { IGM_MBOX_MAX_WORLD = 32, IGM_MBOX_MAX_WORDS = 4096 };
igm_status igm_mbox_create(igm_ctx* ctx, int rank, int world, int max_words, igm_mbox** out);
void igm_mbox_free(igm_mbox* m);
/* CUDA IPC handle of this rank's mailbox (to be exchanged out of band) */
igm_status igm_mbox_handle(igm_mbox* m, unsigned char handle[64]);
/* one process per GPU: handles = world x 64 bytes, rank-major (own entry ignored) */
igm_status igm_mbox_connect_ipc(igm_mbox* m, const unsigned char* handles);
/* one process, several contexts / devices: all = the world's mailboxes by
 * rank (peer access is enabled between their devices) */
igm_status igm_mbox_connect_local(igm_mbox* m, igm_mbox* const* all);
/* the two halves, asynchronous on ctx's stream; n <= max_words device words */
igm_status igm_mbox_publish(igm_ctx* ctx, igm_mbox* m, const uint64_t* words, int n);
igm_status igm_mbox_collect(igm_ctx* ctx, igm_mbox* m, uint64_t* words, int n, int op);
/* publish + collect, any n (chunks of max_words) */
igm_status igm_mbox_allreduce(igm_ctx* ctx, igm_mbox* m, uint64_t* words, int n, int op);
/* synchronises ctx's stream; IGM_CUDA_ERROR if a collect timed out */
igm_status igm_mbox_status(igm_ctx* ctx, igm_mbox* m);

/* v0 = encode(r0 / ||r0||) (gmres_int.cpp:71-81) */
igm_status igm_dc_encode(igm_ctx* ctx, igm_dstate* d, int64_t n, const double* r0, int64_t* v0,
                         int frac_bits);
/* out = spmv(A, s, v) over the rank's rows (split.cpp:137-157) */
igm_status igm_dc_spmv(igm_ctx* ctx, igm_dstate* d, const igm_split* m, int s, const int64_t* v_ext,
                       int64_t* out, int j, int checked);
/* MGS pass i of step j: i == 0 dot_0; 0 < i <= j axpy_{i-1} then dot_i;
 * i == j+1 axpy_j then the norm sum (gmres_int.cpp:101-116) */
igm_status igm_dc_mgs_pass(igm_ctx* ctx, igm_dstate* d, int64_t n, int j, int i, int64_t* w,
                           const int64_t* vprev, const int64_t* vcur, int frac_bits,
                           const igm_shifts* shifts, int checked);
/* the step's scalar work, replicated on every rank (gmres_int.cpp:101-159) */
igm_status igm_dc_step(igm_ctx* ctx, igm_dstate* d, int j, int frac_bits, const igm_shifts* shifts,
                       const int64_t* w, int checked);
/* v_{j+1} = w / h_{j+1,j} (gmres_int.cpp:117-125) */
igm_status igm_dc_vec_div(igm_ctx* ctx, igm_dstate* d, int64_t n, int j, const int64_t* w, int64_t* vout,
                          int frac_bits, const igm_shifts* shifts, int checked);
/* least squares + x += gamma * (0 + sum_j w_j v_j) (gmres_int.cpp:163-180,
 * refine.cpp:87) over the rank's rows */
igm_status igm_dc_finish(igm_ctx* ctx, igm_dstate* d, int frac_bits, int64_t n, const int64_t* basis,
                         double* x);
/* synchronise and read the cycle/refinement scalars; returns the device
 * error of the cycle (domain_error, ...) with the reference's message */
igm_status igm_dc_fetch(igm_ctx* ctx, igm_dstate* d, igm_dc_info* info);

/* ---- host setup (not on the GPU hot path; inputs of the calls above) ---- */
/* replaces intgmres::row_scale (split.cpp:61-79) */
igm_status igm_row_scale(int n, const int* row_ptr, const int* col_idx,
                         const double* vals, int alpha_a, double* vals_out,
                         double* scale_out);
/* replaces intgmres::build_split (split.cpp:90-135); comp_vals_out holds
 * max_components*nnz */
igm_status igm_build_split(int n, int nnz, const double* vals, int alpha_a,
                           int max_components, int64_t* comp_vals_out,
                           int* alphas_out, int* ncomp_out, int* exact_out);
/* replaces intgmres::split_cast(factorize_ilu0(a)) (ilu.cpp:25-120);
 * L/U arrays hold up to nnz(A) entries, row_ptr n+1 */
igm_status igm_factorize_split_cast(int n, const int* row_ptr,
                                    const int* col_idx, const double* vals,
                                    int* l_row_ptr, int* l_col_idx,
                                    int64_t* l_vals, int* l_diag_pos,
                                    int* u_row_ptr, int* u_col_idx,
                                    int64_t* u_vals, int* u_diag_pos);

/* the same, also returning the merged L, U values of ilu.cpp:29-49 on A's
 * pattern (lu_out: nnz doubles, may be NULL).  A z-slab rank factorises its
 * own planes from the previous rank's last plane of merged U rows and hands
 * its own last plane on (dist.slab_ilu_local). */
igm_status igm_factorize_split_cast_lu(int n, const int* row_ptr, const int* col_idx, const double* vals,
                                       int* l_row_ptr, int* l_col_idx, int64_t* l_vals, int* l_diag_pos,
                                       int* u_row_ptr, int* u_col_idx, int64_t* u_vals, int* u_diag_pos,
                                       double* lu_out);

/* ---- device-side setup -------------------------- *
 * The same three functions on the GPU, bit-identical to the host versions
 * above (per-row / per-entry IEEE sequences in the reference's order; the
 * ILU(0) factorisation runs one DAG level per launch, a thread per row).
 * Array arguments may be host or device pointers; outputs are written where
 * they point.  Errors (types and texts) are the reference's; the reported row
 * is the first one the sequential code would meet. */
/* replaces intgmres::row_scale (split.cpp:61-79) */
igm_status igm_row_scale_dev(igm_ctx* ctx, int n, const int* row_ptr, const double* vals, int alpha_a,
                             double* vals_out, double* scale_out);
/* replaces intgmres::build_split (split.cpp:90-135); alphas_out (host) holds
 * max_components ints, comp_vals_out max_components*nnz */
igm_status igm_build_split_dev(igm_ctx* ctx, int nnz, const double* vals, int alpha_a, int max_components,
                               int64_t* comp_vals_out, int* alphas_out, int* ncomp_out, int* exact_out);
/* replaces intgmres::split_cast(factorize_ilu0(a)) (ilu.cpp:25-120) */
igm_status igm_factorize_split_cast_dev(igm_ctx* ctx, int n, const int* row_ptr, const int* col_idx,
                                        const double* vals, int* l_row_ptr, int* l_col_idx, int64_t* l_vals,
                                        int* l_diag_pos, int* u_row_ptr, int* u_col_idx, int64_t* u_vals,
                                        int* u_diag_pos);

/* igm_factorize_split_cast_lu on the device (lu_out: host or device, may be NULL) */
igm_status igm_factorize_split_cast_dev_lu(igm_ctx* ctx, int n, const int* row_ptr, const int* col_idx,
                                           const double* vals, int* l_row_ptr, int* l_col_idx, int64_t* l_vals,
                                           int* l_diag_pos, int* u_row_ptr, int* u_col_idx, int64_t* u_vals,
                                           int* u_diag_pos, double* lu_out);

#ifdef __cplusplus
}
#endif
#endif
