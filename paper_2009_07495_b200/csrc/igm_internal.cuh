// igm_internal.cuh -- device-side data layout of the B200 int-GMRES path.
//
// HBM layout:
//   * SplitMatrix: one CSR pattern (int32 row_ptr/col_idx) shared by all
//     components; int64 values component-major (comp l at vals + l*nnz).
//   * CsrMatrixF: int32 pattern (aliased to the split's when identical) +
//     FP64 values.
//   * IluFactors: per factor the STRICT off-diagonal CSR in natural row order,
//     the raw diagonal, per-row exact reciprocals of the diagonal, and the
//     wavefront schedule (rows grouped into contiguous tiles, each tile's rows
//     bucketed by DAG level).
//   * Krylov basis: (m+1) contiguous int64 vectors of n words.
#pragma once

#include "fx_core.cuh"
#include "schedule.hpp"
#include "../../include/igm.h"

#include <cuda_runtime.h>
#include <atomic>
#include <stdexcept>

#include <cstdint>
#include <string>
#include <vector>

namespace igm {

// Device error-message ids (mapped to the reference's exception texts).
enum ErrMsg {
  EM_NONE = 0,
  EM_NORM_NEG = 1,     // "fx_norm: accumulator wrapped negative"
  EM_DIV_ZERO = 2,     // "fx_div: shifted divisor is zero"
  EM_ENCODE = 3,       // "encode: value outside representable range"
  EM_HESS_ZERO = 4,    // "solve_hessenberg: zero diagonal"
  EM_GAMMA_ZERO = 5,   // "gamma_scale: zero residual"
};

// Per-context control block in device memory.  Written by single-thread
// kernels, read by every kernel of a cycle to early-exit after a break or
// an error (so a whole cycle can be enqueued without host round trips).
struct Ctl {
  int err;        // igm_status of the first error
  int err_msg;    // ErrMsg
  int err_step;
  int stop;       // cycle ended (t_mp == 0, happy breakdown, r0 == 0)
  int dim;
  int nbasis;
  int do_vecdiv;  // the current step produces v_{j+1}
  int add_inexact;
  i64 hnext;
  u64 div_m;      // SDivMagic of the current vec_div divisor
  int div_sh1, div_sh2, div_neg, div_m1;
  double r0n;
  // refinement state
  u64 rmax_bits;  // max |r_i| as IEEE bits (non-negative doubles order as u64)
  double nb, nr, relnorm;
  double scalar;  // scratch result of norm2 kernels
  // grid-barrier arrivals of the persistent Arnoldi kernel (reset per cycle),
  // on a cache line of its own: every CTA polls it while CTA 0's scalar step
  // reads and writes the fields above
  alignas(128) unsigned gbar;
  unsigned gbar_pad[31];
};

struct DevSplit {
  int n = 0, nnz = 0, ncomp = 0;
  int* row_ptr = nullptr;
  int* col_idx = nullptr;
  i64* vals = nullptr;   // ncomp * nnz
  int* alphas = nullptr; // ncomp (device)
  std::vector<int> h_alphas;
  std::vector<int> h_row_ptr_hash;  // not used for identity, kept small
  int device = 0;
  int max_row = 0;  // longest row (selects the staged SpMV for long rows)
  u64 max_abs0 = ~0ull;  // max |value| of component 0 (the SpMV's magnitude certificate)
  // long rows (17..32 entries: 27-point stencils): component 0 once more in a
  // sliced-ELL layout (32-row slices, slot-major, sell_w slots per row, zero
  // padded) for coalesced matrix AND vector loads with one thread per row
  i64* sell_vals = nullptr;
  int* sell_cols = nullptr;
  int sell_w = 0;
};

struct DevCsrf {
  int n = 0, nnz = 0;
  int* row_ptr = nullptr;
  int* col_idx = nullptr;
  double* vals = nullptr;
  int device = 0;
};

// One triangular factor prepared for the wavefront kernels (see
// schedule.hpp): records in schedule order (tile-major, level, row).
struct DevTri {
  int n = 0, maxd = 0, stride = 4, ntiles = 0, nseg = 0, nlevels = 0, tile_cap = 0, max_tile_segs = 0;
  int grid[3] = {0, 0, 0}, brick[3] = {0, 0, 0};
  int *tile_pbase = nullptr, *tile_seg = nullptr, *seg_level = nullptr, *seg_rows = nullptr;
  int *seg_wptr = nullptr, *seg_wt = nullptr;
  int *p_row = nullptr, *p_nd = nullptr, *p_dep = nullptr, *p_xrp = nullptr, *p_xdep = nullptr;
  i64 *p_val = nullptr, *p_xval = nullptr, *p_diag = nullptr;
  u64* p_mag = nullptr;
  int* p_info = nullptr;
  unsigned char* p_rec = nullptr;  // packed records, rec_bytes each
  int rec_bytes = 0;
  bool compact = false;            // compact records (schedule.hpp)
  ulonglong2* xz = nullptr;        // n tagged exported values (128-bit each)
  void* yperm = nullptr;           // n+2 right-hand-side values in schedule order (8 bytes each)
  u64* stats = nullptr;            // [max|y|, max|z|] of the current integer apply (device)
  u64 maxabs_l = 0;                // max |factor value| of the stripped factor (host)
  int *seg_xptr = nullptr, *seg_xrow = nullptr;
  int max_seg_ext = 0;
  int *c_rp = nullptr, *c_ci = nullptr;
  i64 *c_val = nullptr, *c_diag = nullptr;
  unsigned long long epoch = 0;    // launches so far (tag of the next one)
  bool acyclic = false;   // tile graph acyclic in ticket order (lookahead wavefront allowed)
  int* prog = nullptr;    // ntiles progress words
  // structured 7-point factors: the pencil wavefront's stream (pencil.hpp)
  bool pen = false;
  int pen_gx = 0, pen_gy = 0, pen_gz = 0, pen_nbx = 0, pen_nby = 0, pen_nbricks = 0, pen_S = 0, pen_pad = 0;
  void* pen_blk = nullptr;
  // structured 27-point factors: the 27-point pencil wavefront (pencil27.cuh)
  bool pen27 = false;
  int p27_gx = 0, p27_gy = 0, p27_gz = 0, p27_nbx = 0, p27_nbricks = 0;
  void* p27_rec = nullptr;
  void* p27_rec_fp = nullptr;  // the FP64 substitution's stream (diagonal as a double)
  void* pen_blk_fp = nullptr;  // the FP64 substitution's stream (diagonal as a double)
  int* pen_bot = nullptr;
  int pen_cy = 1;  // bricks per thread-block cluster along y in the stream's ticket order (tri_pencil2.cuh)
  int* ticket = nullptr;  // 1
};

// config 3's WL = 32 variant (wl32.cu): the split's values as int32
struct Dev32Split {
  int n = 0, nnz = 0, ncomp = 0;
  int* row_ptr = nullptr;
  int* col_idx = nullptr;
  int32_t* vals = nullptr;  // ncomp * nnz
  int* alphas = nullptr;    // ncomp (device)
  std::vector<int> h_alphas;
  bool own_pattern = true;
  int device = 0;
  int max_row = 0;  // longest row (rows of <= 16 entries use the register-batched SpMV)
};
// per-cycle buffers of the WL = 32 cycle; `small` .. small + small_bytes is
// zeroed before every cycle (accumulators, certificates, counters, H, g, cs, sn)
struct Wl32Work {
  long long n = 0;
  int M = 0;
  int32_t* basis = nullptr;  // (M+1) * n
  int32_t* w = nullptr;      // n
  void* small = nullptr;
  size_t small_bytes = 0;
  uint32_t* acc = nullptr;   // M * (M+1): per step j, the j+1 dot accumulators
  u64* abs = nullptr;        // M * (M+1): their sum |term| certificates
  uint32_t* nacc = nullptr;  // M norm accumulators
  u64* nabs = nullptr;       // M
  int32_t* hess = nullptr;   // (M+1) * M column-major
  int32_t* g = nullptr;      // M+1
  int32_t* cs = nullptr;     // M
  int32_t* sn = nullptr;     // M
  u64* cnt = nullptr;        // M * K_COUNT * OP_COUNT overflow counters
  double* y = nullptr;       // M
  double* wts = nullptr;     // M
};

struct DevIlu {
  int n = 0;
  DevTri lower, upper;
  int device = 0;
};

}  // namespace igm

struct igm_split : igm::DevSplit {};
struct igm_csrf : igm::DevCsrf {};
struct igm_ilu : igm::DevIlu {};

namespace igm {

struct KParams;  // fwd

// --- kernel launchers (kernels.cu) -----------------------------------------
struct ShiftsD {
  int dot_b1, dot_b2, axpy_b1, norm_b1, div_b1, div_b2, givens_b2, rot_b;
};

int device_max_row(cudaStream_t st, int n, const int* rp);
u64 device_max_abs(cudaStream_t st, long long n, const i64* a);
void launch_build_sell(cudaStream_t st, int n, int w, const int* rp, const int* ci, const i64* vals, i64* sv, int* sc);
void launch_spmv_int(cudaStream_t st, const DevSplit& m, int s, const i64* v,
                     i64* out, u64* cnt, const Ctl* ctl, bool checked,
                     const u64* vb = nullptr);
// Work::vmx: kVmxRows rows of (m + 2) words -- row c < grid: CTA c's max |v_i|
// per basis vector; the last row: the maximum over all CTAs (atomicMax)
constexpr int kVmxRows = 1024;
void launch_spmv_fp_split(cudaStream_t st, const DevSplit& m, int s,
                          const double* x, const double* b, double* y,
                          const Ctl* ctl);
void launch_residual(cudaStream_t st, const DevCsrf& a, const double* x,
                     const double* b, double* r, Ctl* ctl, bool track_max);
int pencil27_max_resident(int device);  // CTAs of k_tri27 that fit on the GPU at once
struct PenZ {  // z-slab pipelining of the pencil wavefront (PenArgs::zimp ...)
  const ulonglong2* imp = nullptr;
  ulonglong2* exp = nullptr;
  int kexp = -1;
  unsigned long long epoch = 0;
};
// trace_order.cu: reference-order event lists (locate passes of one call;
// each appends at most `room` op tags to out and returns the call's total)
struct LocateScratch;
LocateScratch* locate_scratch_new();
void locate_scratch_free(LocateScratch* s);
long long locate_spmv(cudaStream_t st, LocateScratch& S, const DevSplit& m, int s, const i64* v, long long room,
                      std::vector<unsigned char>& out);
long long locate_tri(cudaStream_t st, LocateScratch& S, const DevTri& t, bool backward, const i64* y, const i64* z,
                     long long room, std::vector<unsigned char>& out);
long long locate_red(cudaStream_t st, LocateScratch& S, long long n, const i64* w, const i64* v, int b1, int b2,
                     long long room, std::vector<unsigned char>& out);
long long locate_axpy(cudaStream_t st, LocateScratch& S, long long n, const i64* w, const i64* v, i64 hs, int post,
                      long long room, std::vector<unsigned char>& out);
long long locate_vec_div(cudaStream_t st, LocateScratch& S, long long n, const i64* w, i64 den, int b1, int e,
                         long long room, std::vector<unsigned char>& out);
int debug_arn_ts(int j, unsigned long long* out, int cap);
int debug_fx_selftest(int n, const u64* a, const u64* b, u64* out);
bool launch_tri_int_piped(cudaStream_t st, const DevTri& t, bool backward, const i64* y, i64* out, u64* cnt,
                          const Ctl* ctl, bool checked, const PenZ& z);
void launch_tri_int(cudaStream_t st, const DevTri& t, bool backward,
                    const i64* y, i64* out, u64* cnt, const Ctl* ctl,
                    bool checked, bool defer_count = false);
void launch_tri_count_pair(cudaStream_t st, const DevTri& lo, const DevTri& up, const i64* y, const i64* mid,
                           const i64* z, u64* cnt, const Ctl* ctl);
void launch_tri_fp(cudaStream_t st, const DevTri& t, bool backward,
                   const double* y, double* out, const Ctl* ctl,
                   const double* prescale /* divide y by *prescale or null */);
// exact sequential-order norm2 (split.cpp:45-49); scratch: norm2_scratch_bytes(n)
size_t norm2_scratch_bytes(long long n);
// start: device pointer to the chain's starting value (null = 0.0); mode 5
// writes the running sum itself to *out (one rank's leg of a relayed chain)
void launch_norm2_serial(cudaStream_t st, long long n, const double* v,
                         double* out, Ctl* ctl, int mode, void* scratch,
                         const double* start = nullptr);
void launch_mgs_pass(cudaStream_t st, long long n, int mode, i64* w,
                     const i64* vprev, const i64* vcur, const u64* hacc,
                     u64* acc_out, u64* abs_out, int f, ShiftsD sh,
                     u64* cnt_axpy, u64* cnt_red, const Ctl* ctl,
                     bool checked);
void launch_vec_div(cudaStream_t st, long long n, const i64* w, i64* out,
                    int f, ShiftsD sh, u64* cnt, const Ctl* ctl,
                    bool checked, u64* vmax_out = nullptr);
void launch_step_scalar(cudaStream_t st, int j, int f, ShiftsD sh,
                        const u64* acc_col, const u64* abs_col, const u64* nacc,
                        const u64* nabs, i64* hess, int ld, i64* g, i64* cs,
                        i64* sn, i64* gabs, const i64* w, u64* cnt_step,
                        Ctl* ctl, int checked /* 2: add events counted exactly */, int acc_st = 1,
                        int abs_st = 2, const u64* norm_mul = nullptr /* cnt_step's slot */);
// exact add-event count of one fx_dot (mode 0, terms asr(w,b1)*asr(v,b2)) or
// fx_norm (mode 1, asr(w,b1)^2) reduction into *cnt_add; a no-op when the
// certificate cert = {sum|t| hi, lo} is below 2^63
size_t exact_adds_scratch_bytes(long long n);
void launch_exact_adds(cudaStream_t st, long long n, int mode, const i64* w, const i64* v, int b1, int b2,
                       const u64* cert, const Ctl* ctl, u64* cnt_add, void* scratch);
void launch_cycle_init(cudaStream_t st, Ctl* ctl, i64* g, int f);
void launch_encode(cudaStream_t st, long long n, const double* r0, i64* v0,
                   int f, Ctl* ctl);
void launch_cycle_finish(cudaStream_t st, int m, int f, const i64* hess,
                         const i64* g, double* y, double* wts, Ctl* ctl);
void launch_xupdate(cudaStream_t st, long long n, int m, int f,
                    const i64* basis, const double* wts, const double* x0,
                    double* x, const Ctl* ctl, int mode);
void launch_scale_div(cudaStream_t st, long long n, const double* r,
                      double* out, const Ctl* ctl);
void launch_fx_red(cudaStream_t st, long long n, int mode, const i64* v,
                   const i64* w, int b1, int b2, u64* acc, u64* abs_out,
                   u64* cnt, bool checked);
void launch_axpy_only(cudaStream_t st, long long n, i64* w, i64 h,
                      const i64* v, int f, int b1, u64* cnt, bool checked);
void launch_gamma(cudaStream_t st, long long n, const double* r, Ctl* ctl);
// FP64 engine pieces (refsolve.cpp)
void launch_recon_vals(cudaStream_t st, const DevSplit& m, int s, double* out);
void launch_fdot_axpy(cudaStream_t st, long long n, double* w, const double* v, double* part, double* h);
void launch_fscale(cudaStream_t st, long long n, const double* w, double* out, const double* d);
void launch_fxupdate(cudaStream_t st, long long n, int dim, const double* basis, const double* wts, double gamma,
                     double* x, int mode);
int fdot_blocks();
// persistent Arnoldi step (passes + scalar + vec_div in one cooperative launch)
long long arnoldi_slice(long long n, int device);
// one WL = 32 cycle (wl32.cu); xmode 0: x = correction, 1: x += gamma * correction
void enqueue_cycle32(cudaStream_t st, const Wl32Work& b, const Dev32Split& m, int M, int f, int s, ShiftsD sh,
                     const double* r0, Ctl* ctl, bool checked, int xmode, double* x);
void launch_vals_to32(cudaStream_t st, long long cnt, const i64* in, int32_t* out, int* bad);
int arnoldi_barriers(int j, long long S);
void launch_arnoldi(cudaStream_t st, long long n, int j, long long S, const i64* w, i64* basis, u64* accj,
                    u64* absj, u64* nacc, u64* nabs, int f, ShiftsD sh, u64* cstep, i64* hess, int ld, i64* g,
                    i64* cs, i64* sn, i64* gabs, Ctl* ctl, unsigned gbase, bool checked, u64* vmx, u64* snapj);
void launch_basis_norms(cudaStream_t st, long long n, int nb, int f,
                        const i64* basis, void* scratch, double* out, Ctl* ctl);

// device-side setup (setup.cu)
void launch_row_scale(cudaStream_t st, int n, const int* rp, const double* v, int alpha, double* out,
                      double* scale, int* err_row);
void launch_split_layer(cudaStream_t st, long long nnz, const double* v, double* rem, int alpha, i64* comp,
                        u64* mx_out, bool first);
void launch_ilu_pattern(cudaStream_t st, int n, const int* rp, const int* ci, int* diag, int* lcnt, int* ucnt,
                        int* err_row);
void launch_ilu_level(cudaStream_t st, int cnt, const int* rows, const int* rp, const int* ci, const int* diag,
                      double* lu, int* err_row);
void launch_split_cast(cudaStream_t st, int n, const int* rp, const int* ci, const int* diag, const double* lu,
                       const int* lrp, const int* urp, int* lci, i64* lv, int* ldp, int* uci, i64* uv, int* udp,
                       int* err_row);

int num_sms(int device);
int cur_device();  // cudaGetDevice
// once-per-device guard (cudaFuncSetAttribute applies per device)
struct PerDevice {
  std::atomic<unsigned long long> bits{0};
  bool first(int device);
};
// a kernel launch failed (configuration error or sticky fault): the C ABI
// returns IGM_CUDA_ERROR with this message
struct LaunchFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void tri_trace_setup(int tile, unsigned long long* buf);
extern unsigned long long g_launches;  // kernels launched by this library

// Opt-in per-kernel-class timing (CUDA events around each launch on the
// launching stream); used by bench.py for the roofline figures.
enum KClass {
  KC_SPMV = 0, KC_TRI_INT, KC_TRI_FP, KC_MGS, KC_VEC_DIV, KC_SCALAR, KC_NORM2, KC_RESIDUAL,
  KC_XUPDATE, KC_ENCODE, KC_OTHER, KC_COUNT
};
void prof_enable(bool on);
void prof_collect(double* ms, unsigned long long* count);  // KC_COUNT each; resets
struct ProfScope {
  cudaStream_t st;
  int cls;
  ProfScope(cudaStream_t s, int c);
  ~ProfScope();
};

}  // namespace igm
