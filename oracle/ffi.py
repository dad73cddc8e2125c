"""ctypes front-end of the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two back-ends with one call shape:
  * ``Oracle()``    -> oracle/libigm_oracle.so, the C restatement (igm_oracle.c)
  * ``Reference()`` -> oracle/_ref/libintgmres_ref.so, the unmodified reference
                       library compiled from /root/reference (oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libigm_oracle.so"
REF_SO = HERE / "_ref" / "libintgmres_ref.so"

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

KERNELS = ["", "spmv", "precond", "dot", "axpy", "norm", "vec_div", "givens", "givens_norm",
           "givens_div", "rot"]
OPS = ["", "add", "sub", "mul", "shl", "div"]


class Trace(C.Structure):
    _fields_ = [("checked", C.c_int), ("record_shifts", C.c_int), ("kernel", C.c_int),
                ("restart", C.c_int), ("step", C.c_int), ("total", C.c_uint64),
                ("n_events", C.c_int), ("cap_events", C.c_int), ("events", i32p),
                ("n_shifts", C.c_int64), ("cap_shifts", C.c_int), ("shifts", i32p)]


class Shifts(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("dot_b1", "dot_b2", "axpy_b1", "norm_b1", "div_b1", "div_b2", "givens_b2", "rot_b")]


class Csrf(C.Structure):
    _fields_ = [("n", C.c_int), ("row_ptr", i32p), ("col_idx", i32p), ("vals", f64p)]


class Split(C.Structure):
    _fields_ = [("n", C.c_int), ("nnz", C.c_int), ("ncomp", C.c_int), ("row_ptr", i32p),
                ("col_idx", i32p), ("vals", i64p), ("alphas", i32p)]


class Ilu(C.Structure):
    _fields_ = [("n", C.c_int), ("l_row_ptr", i32p), ("l_col_idx", i32p), ("l_diag_pos", i32p),
                ("l_vals", i64p), ("u_row_ptr", i32p), ("u_col_idx", i32p), ("u_diag_pos", i32p),
                ("u_vals", i64p)]


class CycleCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("frac_bits", C.c_int), ("s", C.c_int), ("shifts", Shifts),
                ("precond", C.POINTER(Ilu)), ("collect_basis_norms", C.c_int)]


class CycleOut(C.Structure):
    _fields_ = [("dim", C.c_int), ("r0_norm", C.c_double), ("g_abs", f64p), ("cos_d", f64p),
                ("sin_d", f64p), ("basis_norms", f64p), ("n_basis_norms", C.c_int),
                ("basis", i64p), ("n_basis", C.c_int), ("hess", i64p), ("g", i64p),
                ("cos_raw", i64p), ("sin_raw", i64p)]


class RefineCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_refinements", C.c_int), ("m", C.c_int),
                ("frac_bits", C.c_int), ("s", C.c_int), ("checked", C.c_int), ("shifts", Shifts),
                ("s_schedule", i32p)]


class Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("refinements", C.c_int),
                ("total_inner_iterations", C.c_int64), ("inner_dims", i32p),
                ("relres_history", f64p), ("n_relres", C.c_int), ("gamma_history", f64p),
                ("overflow_per_restart", u64p), ("overflow_total", C.c_uint64),
                ("wall_time_sec", C.c_double)]


class CheckerError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _p(a, t):
    return a.ctypes.data_as(t)


def ensure_built():
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-C", str(HERE), "all"], check=True, capture_output=True)


class PyTrace:
    """Python-side view of a checker trace."""

    def __init__(self, checked=True, record_shifts=False, cap_events=1024, cap_shifts=1 << 20):
        self._ev = np.zeros(4 * cap_events + 4, dtype=np.int32)
        self._sh = np.zeros(3 * (cap_shifts if record_shifts else 1) + 3, dtype=np.int32)
        self.c = Trace(1 if checked else 0, 1 if record_shifts else 0, 0, 0, 0, 0, 0, cap_events,
                       _p(self._ev, i32p), 0, cap_shifts if record_shifts else 0, _p(self._sh, i32p))

    @property
    def total(self):
        return int(self.c.total)

    @property
    def events(self):
        return [(KERNELS[self._ev[4 * i]] if self._ev[4 * i] >= 0 else "?", OPS[self._ev[4 * i + 1]],
                 int(self._ev[4 * i + 2]), int(self._ev[4 * i + 3])) for i in range(self.c.n_events)]

    @property
    def shifts(self):
        n = min(self.c.n_shifts, self.c.cap_shifts)
        return [(KERNELS[self._sh[3 * i]], int(self._sh[3 * i + 1]), int(self._sh[3 * i + 2])) for i in range(n)]


class _Backend:
    prefix = "ora_"

    def __init__(self, path):
        self.lib = C.CDLL(str(path))
        self._keep = []

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def err(self):
        f = self.fn("last_error")
        f.restype = C.c_char_p
        return f().decode()

    def _rc(self, rc):
        if rc != 0:
            raise CheckerError(rc, self.err())

    # ---- scalar ops
    def fx_mul(self, a, b, f, b1, b2, out_frac, trace=None):
        out = C.c_int64()
        self._rc(self.fn("fx_mul")(C.c_int64(a), C.c_int64(b), f, b1, b2, out_frac, C.byref(out),
                                   C.byref(trace.c) if trace else None))
        return out.value

    def fx_div(self, a, b, f, b1, b2, trace=None):
        out = C.c_int64()
        self._rc(self.fn("fx_div")(C.c_int64(a), C.c_int64(b), f, b1, b2, C.byref(out),
                                   C.byref(trace.c) if trace else None))
        return out.value

    def fx_add(self, a, b, trace=None):
        out = C.c_int64()
        self._rc(self.fn("fx_add")(C.c_int64(a), C.c_int64(b), C.byref(out), C.byref(trace.c) if trace else None))
        return out.value

    def fx_sub(self, a, b, trace=None):
        out = C.c_int64()
        self._rc(self.fn("fx_sub")(C.c_int64(a), C.c_int64(b), C.byref(out), C.byref(trace.c) if trace else None))
        return out.value

    def isqrt(self, v):
        f = self.fn("isqrt")
        f.restype = C.c_uint64
        f.argtypes = [C.c_uint64]
        return int(f(v))

    def fx_sqrt(self, a, fin, out_frac, trace=None):
        out = C.c_int64()
        self._rc(self.fn("fx_sqrt")(C.c_int64(a), fin, out_frac, C.byref(out), C.byref(trace.c) if trace else None))
        return out.value

    def encode(self, x, f):
        out = C.c_int64()
        self._rc(self.fn("encode")(C.c_double(x), f, C.byref(out)))
        return out.value

    def decode(self, raw, f):
        fn = self.fn("decode")
        fn.restype = C.c_double
        fn.argtypes = [C.c_int64, C.c_int]
        return fn(raw, f)

    def shifts_validate(self, sh, f):
        return self.fn("shifts_validate")(C.byref(sh), f)

    # ---- vector kernels
    def fx_dot(self, v, w, f, b1, b2, trace=None):
        v = np.ascontiguousarray(v, np.int64); w = np.ascontiguousarray(w, np.int64)
        out = C.c_int64()
        self._rc(self.fn("fx_dot")(C.c_int64(len(v)), _p(v, i64p), _p(w, i64p), f, b1, b2, C.byref(out),
                                   C.byref(trace.c) if trace else None))
        return out.value

    def fx_norm(self, v, f, b1, trace=None):
        v = np.ascontiguousarray(v, np.int64)
        out = C.c_int64()
        self._rc(self.fn("fx_norm")(C.c_int64(len(v)), _p(v, i64p), f, b1, C.byref(out),
                                    C.byref(trace.c) if trace else None))
        return out.value

    def fx_axpy_sub(self, w, h, v, f, b1, trace=None):
        w = np.array(w, dtype=np.int64, copy=True); v = np.ascontiguousarray(v, np.int64)
        self._rc(self.fn("fx_axpy_sub")(C.c_int64(len(w)), _p(w, i64p), C.c_int64(h), _p(v, i64p), f, b1,
                                        C.byref(trace.c) if trace else None))
        return w

    # ---- structs
    def split(self, rp, ci, comp, alphas):
        rp = np.ascontiguousarray(rp, np.int32); ci = np.ascontiguousarray(ci, np.int32)
        comp = np.ascontiguousarray(np.atleast_2d(comp), np.int64)
        al = np.ascontiguousarray(alphas, np.int32)
        self._keep += [rp, ci, comp, al]
        return Split(len(rp) - 1, comp.shape[1], comp.shape[0], _p(rp, i32p), _p(ci, i32p), _p(comp, i64p),
                     _p(al, i32p))

    def csrf(self, rp, ci, v):
        rp = np.ascontiguousarray(rp, np.int32); ci = np.ascontiguousarray(ci, np.int32)
        v = np.ascontiguousarray(v, np.float64)
        self._keep += [rp, ci, v]
        return Csrf(len(rp) - 1, _p(rp, i32p), _p(ci, i32p), _p(v, f64p))

    def ilu(self, lower, upper):
        arrs = []
        for (rp, ci, v, dp) in (lower, upper):
            arrs.append((np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32),
                         np.ascontiguousarray(dp, np.int32), np.ascontiguousarray(v, np.int64)))
        self._keep += [a for t in arrs for a in t]
        (lrp, lci, ldp, lv), (urp, uci, udp, uv) = arrs
        return Ilu(len(lrp) - 1, _p(lrp, i32p), _p(lci, i32p), _p(ldp, i32p), _p(lv, i64p),
                   _p(urp, i32p), _p(uci, i32p), _p(udp, i32p), _p(uv, i64p))

    # ---- operators
    def spmv(self, sp, s, v, trace=None):
        v = np.ascontiguousarray(v, np.int64)
        out = np.zeros(sp.n, np.int64)
        self._rc(self.fn("spmv")(C.byref(sp), s, _p(v, i64p), _p(out, i64p), C.byref(trace.c) if trace else None))
        return out

    def apply_inverse(self, il, y, trace=None):
        y = np.ascontiguousarray(y, np.int64)
        out = np.zeros(il.n, np.int64)
        self._rc(self.fn("apply_inverse")(C.byref(il), _p(y, i64p), _p(out, i64p),
                                          C.byref(trace.c) if trace else None))
        return out

    def apply_inverse_fp(self, il, y):
        y = np.ascontiguousarray(y, np.float64)
        out = np.zeros(il.n)
        self._rc(self.fn("apply_inverse_fp")(C.byref(il), _p(y, f64p), _p(out, f64p)))
        return out

    def spmv_fp_split(self, sp, s, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(sp.n)
        self._rc(self.fn("spmv_fp_split")(C.byref(sp), s, _p(x, f64p), _p(out, f64p)))
        return out

    def norm2(self, v):
        v = np.ascontiguousarray(v, np.float64)
        f = self.fn("norm2")
        f.restype = C.c_double
        return f(C.c_int64(len(v)), _p(v, f64p))

    def residual_fp(self, a, x, b):
        x = np.ascontiguousarray(x, np.float64); b = np.ascontiguousarray(b, np.float64)
        r = np.zeros(a.n)
        f = self.fn("residual_fp")
        f.restype = C.c_double
        rel = f(C.byref(a), _p(x, f64p), _p(b, f64p), _p(r, f64p))
        return r, rel

    def row_scale(self, a, alpha):
        nnz = a.row_ptr[a.n]
        vals = np.zeros(nnz)
        scale = np.zeros(a.n)
        self._rc(self.fn("row_scale")(C.byref(a), alpha, _p(vals, f64p), _p(scale, f64p)))
        return vals, scale

    def factorize_split_cast(self, a):
        n = a.n
        nnz = a.row_ptr[n]
        lrp = np.zeros(n + 1, np.int32); urp = np.zeros(n + 1, np.int32)
        lci = np.zeros(nnz, np.int32); uci = np.zeros(nnz, np.int32)
        lv = np.zeros(nnz, np.int64); uv = np.zeros(nnz, np.int64)
        ldp = np.zeros(n, np.int32); udp = np.zeros(n, np.int32)
        self._rc(self.fn("factorize_split_cast")(C.byref(a), _p(lrp, i32p), _p(lci, i32p), _p(lv, i64p),
                                                 _p(ldp, i32p), _p(urp, i32p), _p(uci, i32p), _p(uv, i64p),
                                                 _p(udp, i32p)))
        nl, nu = int(lrp[-1]), int(urp[-1])
        return (lrp, lci[:nl].copy(), lv[:nl].copy(), ldp), (urp, uci[:nu].copy(), uv[:nu].copy(), udp)

    # ---- cycle / solve
    def run_cycle(self, sp, m, f, s, shifts, b, x0, precond=None, collect_basis_norms=False, trace=None):
        n = sp.n
        M = max(m, 1)
        cfg = CycleCfg(m, f, s, shifts, C.pointer(precond) if precond is not None else None,
                       1 if collect_basis_norms else 0)
        bufs = dict(g_abs=np.zeros(M), cos_d=np.zeros(M), sin_d=np.zeros(M), basis_norms=np.zeros(M + 1),
                    basis=np.zeros((M + 1) * n, np.int64), hess=np.zeros((M + 1) * M, np.int64),
                    g=np.zeros(M + 1, np.int64), cos_raw=np.zeros(M, np.int64), sin_raw=np.zeros(M, np.int64))
        out = CycleOut()
        for k, a in bufs.items():
            setattr(out, k, _p(a, f64p if a.dtype == np.float64 else i64p))
        x = np.zeros(n)
        b = np.ascontiguousarray(b, np.float64); x0 = np.ascontiguousarray(x0, np.float64)
        self._rc(self.fn("run_cycle")(C.byref(sp), C.byref(cfg), _p(b, f64p), _p(x0, f64p), _p(x, f64p),
                                      C.byref(out), C.byref(trace.c) if trace else None))
        d = out.dim
        return dict(x=x, dim=d, r0_norm=out.r0_norm, g_abs=bufs["g_abs"][:d], cos=bufs["cos_d"][:d],
                    sin=bufs["sin_d"][:d], basis_norms=bufs["basis_norms"][:out.n_basis_norms],
                    basis=bufs["basis"][: out.n_basis * n].reshape(out.n_basis, n), hess=bufs["hess"],
                    g=bufs["g"], cos_raw=bufs["cos_raw"], sin_raw=bufs["sin_raw"], n_basis=out.n_basis)

    def solve(self, sp, a, b, tol, max_ref, m, f, s, shifts, checked=True, precond=None, s_schedule=None,
              trace=None, engine=0):
        R = max(max_ref, 0)
        dims = np.zeros(R + 1, np.int32); rel = np.zeros(R + 2); gam = np.zeros(R + 1)
        ovf = np.zeros(R + 1, np.uint64)
        sched = np.ascontiguousarray(s_schedule, np.int32) if s_schedule is not None else None
        cfg = RefineCfg(tol, max_ref, m, f, s, 1 if checked else 0, shifts,
                        _p(sched, i32p) if sched is not None else None)
        rep = Report(0, 0, 0, _p(dims, i32p), _p(rel, f64p), 0, _p(gam, f64p), _p(ovf, u64p), 0, 0.0)
        x = np.zeros(sp.n)
        b = np.ascontiguousarray(b, np.float64)
        args = (C.byref(sp), C.byref(a), _p(b, f64p), C.byref(cfg),
                C.pointer(precond) if precond is not None else None, _p(x, f64p), C.byref(rep),
                C.byref(trace.c) if trace else None)
        if engine:  # the FP64 comparator engine exists only in the reference library
            fn = self.fn("solve_engine")
            fn.argtypes = None
            self._rc(fn(*args, C.c_int(engine)))
        else:
            self._rc(self.fn("solve")(*args))
        k = rep.refinements
        return x, dict(converged=bool(rep.converged), refinements=k,
                       total_inner_iterations=int(rep.total_inner_iterations),
                       inner_dims=[int(v) for v in dims[:k]], relres_history=[float(v) for v in rel[:rep.n_relres]],
                       gamma_history=[float(v) for v in gam[:k]],
                       overflow_per_restart=[int(v) for v in ovf[:k]], overflow_total=int(rep.overflow_total),
                       wall_time_sec=rep.wall_time_sec)


class Oracle(_Backend):
    prefix = "ora_"

    def __init__(self):
        ensure_built()
        super().__init__(ORACLE_SO)

    def build_split(self, vals, alpha_a, max_components):
        vals = np.ascontiguousarray(vals, np.float64)
        nnz = len(vals)
        comp = np.zeros((max(max_components, 1), nnz), np.int64)
        al = np.zeros(max(max_components, 1), np.int32)
        nc = C.c_int(); ex = C.c_int()
        self._rc(self.fn("build_split")(0, nnz, _p(vals, f64p), alpha_a, max_components, _p(comp, i64p),
                                        _p(al, i32p), C.byref(nc), C.byref(ex)))
        return comp[:nc.value].copy(), [int(a) for a in al[:nc.value]], bool(ex.value)


class Cycle32Cfg(C.Structure):
    _fields_ = [("m", C.c_int), ("f", C.c_int), ("s", C.c_int), ("checked", C.c_int), ("sh", Shifts)]


class Oracle32:
    """WL = 32 restatement (igm_oracle32.c): PARITY UNPINNED -- the reference
    has no WL != 64 code (fxp.hpp:22)."""

    def __init__(self):
        ensure_built()
        self.lib = C.CDLL(str(ORACLE_SO))
        self.lib.ora32_last_error.restype = C.c_char_p

    def _rc(self, rc):
        if rc:
            raise RuntimeError(f"oracle32 error {rc}: {self.lib.ora32_last_error().decode()}")

    @staticmethod
    def _split(rp, ci, comp32, alphas):
        rp = np.ascontiguousarray(rp, np.int32); ci = np.ascontiguousarray(ci, np.int32)
        comp32 = np.ascontiguousarray(np.atleast_2d(comp32), np.int32)
        al = np.ascontiguousarray(alphas, np.int32)
        return rp, ci, comp32, al

    def spmv(self, rp, ci, comp32, alphas, s, v):
        rp, ci, cv, al = self._split(rp, ci, comp32, alphas)
        v = np.ascontiguousarray(v, np.int32)
        out = np.zeros(len(rp) - 1, np.int32)
        ov = C.c_uint64()
        self._rc(self.lib.ora32_spmv(len(rp) - 1, _p(rp, i32p), _p(ci, i32p), _p(cv, i32p), cv.shape[1], cv.shape[0],
                                     _p(al, i32p), s, _p(v, i32p), _p(out, i32p), C.byref(ov)))
        return out, int(ov.value)

    def run_cycle(self, rp, ci, comp32, alphas, m, f, s, shifts, b, checked=True):
        rp, ci, cv, al = self._split(rp, ci, comp32, alphas)
        n = len(rp) - 1
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(n)
        basis = np.zeros((m + 1) * n, np.int32)
        hess = np.zeros((m + 1) * m, np.int32)
        g = np.zeros(m + 1, np.int32)
        cs = np.zeros(m, np.int32); sn = np.zeros(m, np.int32)
        dim = C.c_int(); nb = C.c_int(); r0 = C.c_double(); ov = C.c_uint64()
        cfg = Cycle32Cfg(m, f, s, int(checked), shifts)
        self._rc(self.lib.ora32_run_cycle(n, _p(rp, i32p), _p(ci, i32p), _p(cv, i32p), cv.shape[1], cv.shape[0],
                                          _p(al, i32p), C.byref(cfg), _p(b, f64p), _p(x, f64p), C.byref(dim),
                                          C.byref(r0), _p(basis, i32p), C.byref(nb), _p(hess, i32p), _p(g, i32p),
                                          _p(cs, i32p), _p(sn, i32p), C.byref(ov)))
        return dict(dim=dim.value, r0_norm=r0.value, basis=basis[:nb.value * n].copy(), n_basis=nb.value,
                    hess=hess, g=g, cos_raw=cs, sin_raw=sn, x=x, overflows=int(ov.value))

    def solve(self, rp, ci, comp32, alphas, a_vals, b, tol, max_ref, m, f, s, shifts, checked=True):
        rp, ci, cv, al = self._split(rp, ci, comp32, alphas)
        n = len(rp) - 1
        av = np.ascontiguousarray(a_vals, np.float64)
        a = Csrf(n, _p(rp, i32p), _p(ci, i32p), _p(av, f64p))
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(n)
        rel = np.zeros(max_ref + 1); gam = np.zeros(max(max_ref, 1)); dims = np.zeros(max(max_ref, 1), np.int32)
        nref = C.c_int(); conv = C.c_int(); ov = C.c_uint64()
        cfg = Cycle32Cfg(m, f, s, int(checked), shifts)
        self._rc(self.lib.ora32_solve(n, _p(rp, i32p), _p(ci, i32p), _p(cv, i32p), cv.shape[1], cv.shape[0],
                                      _p(al, i32p), C.byref(a), _p(b, f64p), C.c_double(tol), max_ref, C.byref(cfg),
                                      _p(x, f64p), _p(rel, f64p), _p(gam, f64p), _p(dims, i32p), C.byref(nref),
                                      C.byref(conv), C.byref(ov)))
        k = nref.value
        return x, dict(refinements=k, relres_history=[float(v) for v in rel[:k + 1]],
                       gamma_history=[float(v) for v in gam[:k]], inner_dims=[int(v) for v in dims[:k]],
                       converged=bool(conv.value), overflow_total=int(ov.value))


class Reference(_Backend):
    """The unmodified reference library (oracle/_ref); only where it was built."""
    prefix = "ref_"

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; run `make -C oracle ref`)")
        super().__init__(REF_SO)

    def build_split(self, a, alpha_a, max_components):
        nnz = a.row_ptr[a.n]
        comp = np.zeros((max(max_components, 1), nnz), np.int64)
        al = np.zeros(max(max_components, 1), np.int32)
        nc = C.c_int(); ex = C.c_int()
        self._rc(self.fn("build_split")(C.byref(a), alpha_a, max_components, _p(comp, i64p), _p(al, i32p),
                                        C.byref(nc), C.byref(ex)))
        return comp[:nc.value].copy(), [int(a) for a in al[:nc.value]], bool(ex.value)


def ref_available() -> bool:
    return REF_SO.exists()
