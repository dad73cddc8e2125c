"""B200-native int-GMRES hot path (arXiv 2009.07495) -- Python host mirror.

Thin, typed wrappers over the C ABI (include/igm.h, libigm_b200.so).  Names
and argument meaning follow the reference C++ API (proj/core/include/intgmres)
so that parity tests read like the reference's own tests:

    spmv(split, s, v, trace)            <- intgmres::spmv            (split.cpp:137)
    apply_inverse(ilu, y, trace)        <- intgmres::apply_inverse   (ilu.cpp:122)
    apply_inverse_fp(ilu, y)            <- intgmres::apply_inverse_fp(ilu.cpp:157)
    fx_dot / fx_norm / fx_axpy_sub      <- fxp.cpp:49-104
    spmv_fp / residual_fp / norm2       <- split.cpp:37-59
    gamma_scale                         <- refine.cpp:11-19
    run_cycle(split, cfg, b, x0, ...)   <- gmres_int.cpp:42-196
    solve(split, a_fp, b, cfg, precond) <- refine.cpp:21-106

Vectors may be numpy arrays (host; staged through device memory) or torch
CUDA tensors (device-resident, used in place).  Errors raise the Python
analogue of the reference's exception type.  There is no CPU fallback: every
compute call runs the sm_100a kernels of libigm_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _capi
from ._capi import KERNEL_NAMES, OP_NAMES

__all__ = [
    "Device", "SplitMatrix", "CsrMatrixF", "IluFactors", "ShiftPlan", "FxTrace",
    "CycleConfig", "RefineConfig", "spmv", "apply_inverse", "apply_inverse_fp", "fx_dot",
    "fx_norm", "fx_axpy_sub", "spmv_fp", "spmv_fp_split", "residual_fp", "norm2",
    "gamma_scale", "run_cycle", "solve", "spmv_mgs", "row_scale", "build_split",
    "factorize_split_cast", "lib",
]


def lib() -> C.CDLL:
    return _capi.load()


# ---------------------------------------------------------------- errors
class LogicError(Exception):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {1: ValueError, 2: ArithmeticError, 3: OverflowError, 4: RuntimeError, 5: LogicError,
        6: CudaError, 7: CudaError}


def _check(status: int) -> None:
    if status != 0:
        msg = lib().igm_last_error().decode()
        raise _EXC.get(status, RuntimeError)(msg)


# ---------------------------------------------------------------- buffers
def _is_torch(a) -> bool:
    return hasattr(a, "data_ptr") and hasattr(a, "is_cuda")


def _ptr(a, dtype):
    """(void*, keepalive) for a numpy array or a torch tensor.

    Device tensors are read/written on the library's own stream
    (igm_ctx_stream); work queued on torch's current stream is ordered before
    the call here (the C ABI leaves stream ordering to the caller)."""
    if a is None:
        return None, None
    if _is_torch(a):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if a.is_cuda:
            import torch
            torch.cuda.current_stream(a.device).synchronize()
        return C.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=dtype)
    return C.c_void_p(arr.ctypes.data), arr


def _out_like(template, n, dtype):
    if template is not None and _is_torch(template):
        import torch
        tdt = {np.int64: torch.int64, np.float64: torch.float64}[dtype]
        return torch.empty(n, dtype=tdt, device=template.device)
    return np.empty(n, dtype=dtype)


# ---------------------------------------------------------------- context
class Device:
    """One igm_ctx (device + stream + workspaces)."""

    _default: Optional["Device"] = None

    def __init__(self, index: int = 0):
        h = C.c_void_p()
        _check(lib().igm_ctx_create(index, C.byref(h)))
        self.h = h
        self.index = index

    @classmethod
    def default(cls) -> "Device":
        if cls._default is None:
            cls._default = Device(0)
        return cls._default

    def synchronize(self):
        _check(lib().igm_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().igm_ctx_stream(self.h) or 0

    def set_exact_overflow_counts(self, on: bool = True) -> None:
        """Exact running-sum overflow events in checked mode (8(f) row 4)."""
        _check(lib().igm_set_exact_overflow_counts(self.h, 1 if on else 0))

    @property
    def launches(self) -> int:
        return int(lib().igm_ctx_launch_count(self.h))

    def close(self):
        if self.h:
            lib().igm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev(d: Optional[Device]) -> Device:
    return d if d is not None else Device.default()


# ---------------------------------------------------------------- matrices
class SplitMatrix:
    """Device-resident SplitMatrix (split.hpp:28-37)."""

    def __init__(self, row_ptr, col_idx, comp_vals, alphas, device: Optional[Device] = None):
        self.dev = _dev(device)
        comp_vals = np.atleast_2d(np.asarray(comp_vals, dtype=np.int64))
        self.ncomp, self.nnz = comp_vals.shape
        self.n = len(row_ptr) - 1
        rp, k1 = _ptr(row_ptr, np.int32)
        ci, k2 = _ptr(col_idx, np.int32)
        cv, k3 = _ptr(comp_vals, np.int64)
        al, k4 = _ptr(np.asarray(alphas, dtype=np.int32), np.int32)
        h = C.c_void_p()
        _check(lib().igm_upload_split(self.dev.h, self.n, self.nnz, rp, ci, self.ncomp, cv, al, C.byref(h)))
        self.h = h
        self.alphas = [int(a) for a in alphas]

    @property
    def depth(self) -> int:
        return self.ncomp - 1

    def __del__(self):
        try:
            lib().igm_split_free(self.h)
        except Exception:
            pass


class CsrMatrixF:
    """Device-resident FP64 CSR matrix (csr.hpp:10-18)."""

    def __init__(self, row_ptr, col_idx, vals, device: Optional[Device] = None):
        self.dev = _dev(device)
        self.n = len(row_ptr) - 1
        rp, k1 = _ptr(row_ptr, np.int32)
        ci, k2 = _ptr(col_idx, np.int32)
        v, k3 = _ptr(vals, np.float64)
        h = C.c_void_p()
        _check(lib().igm_upload_csrf(self.dev.h, self.n, rp, ci, v, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().igm_csrf_free(self.h)
        except Exception:
            pass


class IluFactors:
    """Device-resident integer ILU factors + wavefront schedule (ilu.hpp:27-32)."""

    def __init__(self, lower, upper, device: Optional[Device] = None):
        """lower/upper: (row_ptr, col_idx, vals, diag_pos) tuples."""
        self.dev = _dev(device)
        self.n = len(lower[0]) - 1
        keep = []
        ptrs = []
        for arrs in (lower, upper):
            for a, dt in zip(arrs, (np.int32, np.int32, np.int64, np.int32)):
                p, k = _ptr(a, dt)
                ptrs.append(p)
                keep.append(k)
        h = C.c_void_p()
        _check(lib().igm_upload_ilu(self.dev.h, self.n, *ptrs, C.byref(h)))
        self.h = h

    def levels(self, backward: bool = False) -> int:
        return int(lib().igm_ilu_levels(self.h, 1 if backward else 0))

    def pencil_bricks(self, backward: bool = False) -> int:
        """Bricks of the pencil wavefront used for this substitution (0: generic wavefront)."""
        return int(lib().igm_ilu_pencil(self.h, 1 if backward else 0))

    def schedule_info(self, backward: bool = False) -> dict:
        out = (C.c_int32 * 8)()
        lib().igm_ilu_schedule_info(self.h, 1 if backward else 0, out)
        b = out[7]
        return {"tiles": out[0], "segments": out[1], "levels": out[2], "max_deps": out[3],
                "grid": (out[4], out[5], out[6]), "brick": (b // 1000000, (b // 1000) % 1000, b % 1000)}

    def __del__(self):
        try:
            lib().igm_ilu_free(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------- config
@dataclass
class ShiftPlan:
    dot_b1: int = 0
    dot_b2: int = 0
    axpy_b1: int = 0
    norm_b1: int = 0
    div_b1: int = 0
    div_b2: int = 0
    givens_b2: int = 0
    rot_b: int = 0

    @staticmethod
    def default_unpreconditioned(f: int = 30) -> "ShiftPlan":  # fxp.cpp:129-141
        return ShiftPlan(16, 0, 16, 16, 16, f - 16, 16, 0)

    @staticmethod
    def default_preconditioned(f: int = 30) -> "ShiftPlan":  # fxp.cpp:143-148
        return ShiftPlan(div_b1=f)

    def c(self) -> _capi.Shifts:
        return _capi.Shifts(self.dot_b1, self.dot_b2, self.axpy_b1, self.norm_b1, self.div_b1,
                            self.div_b2, self.givens_b2, self.rot_b)

    def astuple(self) -> tuple:
        return (self.dot_b1, self.dot_b2, self.axpy_b1, self.norm_b1, self.div_b1, self.div_b2,
                self.givens_b2, self.rot_b)


class FxTrace:
    """FxTrace (fxp.hpp:51-103) backed by an igm_trace."""

    max_events = 1024

    def __init__(self, checked: bool = True, record_shifts: bool = False, shift_cap: int = 1 << 20):
        self._ev = (C.c_int32 * (4 * self.max_events))()
        self._sh = (C.c_int32 * (3 * (shift_cap if record_shifts else 1)))()
        self.c = _capi.Trace(checked=1 if checked else 0, record_shifts=1 if record_shifts else 0,
                             kernel=0, restart=0, step=0, total=0, n_events=0,
                             cap_events=self.max_events, events=C.cast(self._ev, _capi.i32p),
                             n_shifts=0, cap_shifts=shift_cap if record_shifts else 0,
                             shifts=C.cast(self._sh, _capi.i32p), exact=1)

    def set_kernel(self, name: str):
        self.c.kernel = KERNEL_NAMES.index(name) if name in KERNEL_NAMES else 0

    def set_location(self, restart: int, step: int):
        self.c.restart, self.c.step = restart, step

    @property
    def checked(self) -> bool:
        return bool(self.c.checked)

    @property
    def exact(self) -> bool:
        return bool(self.c.exact)

    def total_overflows(self) -> int:
        return int(self.c.total)

    @property
    def events(self):
        out = []
        for i in range(self.c.n_events):
            k, op, r, s = (self._ev[4 * i + q] for q in range(4))
            out.append((KERNEL_NAMES[k] if 0 <= k < len(KERNEL_NAMES) else "?", OP_NAMES[op], r, s))
        return out

    @property
    def shifts(self):
        n = min(self.c.n_shifts, self.c.cap_shifts)
        return [(KERNEL_NAMES[self._sh[3 * i]], self._sh[3 * i + 1], self._sh[3 * i + 2]) for i in range(n)]

    def ptr(self):
        return C.byref(self.c)


def _tptr(t: Optional[FxTrace]):
    return t.ptr() if t is not None else None


# ---------------------------------------------------------------- primitives
def spmv(m: SplitMatrix, s: int, v, trace: Optional[FxTrace] = None):
    out = _out_like(v, m.n, np.int64)
    pv, k1 = _ptr(v, np.int64)
    po, k2 = _ptr(out, np.int64)
    _check(lib().igm_spmv(m.dev.h, m.h, s, pv, po, _tptr(trace)))
    return out


def apply_inverse(f: IluFactors, y, trace: Optional[FxTrace] = None):
    out = _out_like(y, f.n, np.int64)
    py, k1 = _ptr(y, np.int64)
    po, k2 = _ptr(out, np.int64)
    _check(lib().igm_apply_inverse(f.dev.h, f.h, py, po, _tptr(trace)))
    return out


def apply_inverse_fp(f: IluFactors, y):
    out = _out_like(y, f.n, np.float64)
    py, k1 = _ptr(y, np.float64)
    po, k2 = _ptr(out, np.float64)
    _check(lib().igm_apply_inverse_fp(f.dev.h, f.h, py, po))
    return out


def fx_dot(v, w, f: int, b1: int, b2: int, trace: Optional[FxTrace] = None,
           device: Optional[Device] = None) -> int:
    d = _dev(device)
    pv, k1 = _ptr(v, np.int64)
    pw, k2 = _ptr(w, np.int64)
    out = C.c_int64()
    _check(lib().igm_fx_dot(d.h, len(v), pv, pw, f, b1, b2, C.byref(out), _tptr(trace)))
    return out.value


def fx_norm(v, f: int, b1: int, trace: Optional[FxTrace] = None, device: Optional[Device] = None) -> int:
    d = _dev(device)
    pv, k1 = _ptr(v, np.int64)
    out = C.c_int64()
    _check(lib().igm_fx_norm(d.h, len(v), pv, f, b1, C.byref(out), _tptr(trace)))
    return out.value


def fx_axpy_sub(w, h: int, v, f: int, b1: int, trace: Optional[FxTrace] = None,
                device: Optional[Device] = None):
    """In place on w (numpy int64 array or torch tensor), like fxp.cpp:88-104."""
    d = _dev(device)
    if not _is_torch(w) and (not isinstance(w, np.ndarray) or w.dtype != np.int64 or not w.flags.c_contiguous):
        raise ValueError("w must be a C-contiguous int64 numpy array or a CUDA tensor")
    pw = C.c_void_p(w.data_ptr() if _is_torch(w) else w.ctypes.data)
    pv, k1 = _ptr(v, np.int64)
    _check(lib().igm_fx_axpy_sub(d.h, len(w), pw, int(h), pv, f, b1, _tptr(trace)))
    return w


def spmv_fp(a: CsrMatrixF, x):
    out = _out_like(x, a.n, np.float64)
    px, k1 = _ptr(x, np.float64)
    po, k2 = _ptr(out, np.float64)
    _check(lib().igm_spmv_fp(a.dev.h, a.h, px, po))
    return out


def spmv_fp_split(m: SplitMatrix, s: int, x):
    out = _out_like(x, m.n, np.float64)
    px, k1 = _ptr(x, np.float64)
    po, k2 = _ptr(out, np.float64)
    _check(lib().igm_spmv_fp_split(m.dev.h, m.h, s, px, po))
    return out


def residual_fp(a: CsrMatrixF, x, b):
    out = _out_like(x, a.n, np.float64)
    px, k1 = _ptr(x, np.float64)
    pb, k2 = _ptr(b, np.float64)
    po, k3 = _ptr(out, np.float64)
    rel = C.c_double()
    _check(lib().igm_residual_fp(a.dev.h, a.h, px, pb, po, C.byref(rel)))
    return out, rel.value


def norm2(v, device: Optional[Device] = None) -> float:
    d = _dev(device)
    pv, k1 = _ptr(v, np.float64)
    out = C.c_double()
    _check(lib().igm_norm2(d.h, len(v), pv, C.byref(out)))
    return out.value


def gamma_scale(r, device: Optional[Device] = None):
    d = _dev(device)
    out = _out_like(r, len(r), np.float64)
    pr, k1 = _ptr(r, np.float64)
    po, k2 = _ptr(out, np.float64)
    g = C.c_double()
    _check(lib().igm_gamma_scale(d.h, len(r), pr, C.byref(g), po))
    return g.value, out


# ---------------------------------------------------------------- cycle / solve
@dataclass
class CycleConfig:
    m: int = 30
    frac_bits: int = 30
    shifts: ShiftPlan = field(default_factory=ShiftPlan)
    s: int = 0
    precond: Optional[IluFactors] = None
    collect_basis_norms: bool = False


@dataclass
class CycleResult:
    x: np.ndarray
    dim: int
    r0_norm: float
    g_abs: np.ndarray
    cos: np.ndarray
    sin: np.ndarray
    basis_norms: np.ndarray
    basis: Optional[np.ndarray]  # (n_basis, n) int64
    hess: np.ndarray             # (m+1)*m column-major
    g: np.ndarray
    cos_raw: np.ndarray
    sin_raw: np.ndarray


def run_cycle(m: SplitMatrix, cfg: CycleConfig, b, x0=None, trace: Optional[FxTrace] = None,
              state: bool = True) -> CycleResult:
    M, n = cfg.m, m.n
    cc = _capi.CycleCfg(M, cfg.frac_bits, cfg.s, cfg.shifts.c(),
                        cfg.precond.h if cfg.precond is not None else None,
                        1 if cfg.collect_basis_norms else 0)
    Mp = max(M, 1)
    gabs = np.zeros(Mp); cd = np.zeros(Mp); sd = np.zeros(Mp); bn = np.zeros(Mp + 1)
    basis = np.zeros(((Mp + 1), n), dtype=np.int64) if state else None
    hess = np.zeros((Mp + 1) * Mp, dtype=np.int64)
    g = np.zeros(Mp + 1, dtype=np.int64)
    cr = np.zeros(Mp, dtype=np.int64); sr = np.zeros(Mp, dtype=np.int64)
    co = _capi.CycleOut()
    co.g_abs = gabs.ctypes.data_as(_capi.f64p)
    co.cos_d = cd.ctypes.data_as(_capi.f64p)
    co.sin_d = sd.ctypes.data_as(_capi.f64p)
    co.basis_norms = bn.ctypes.data_as(_capi.f64p)
    co.basis = basis.ctypes.data_as(_capi.i64p) if state else None
    co.hess = hess.ctypes.data_as(_capi.i64p)
    co.g = g.ctypes.data_as(_capi.i64p)
    co.cos_raw = cr.ctypes.data_as(_capi.i64p)
    co.sin_raw = sr.ctypes.data_as(_capi.i64p)
    x = _out_like(b, n, np.float64)
    pb, k1 = _ptr(b, np.float64)
    px0, k2 = _ptr(x0, np.float64)
    px, k3 = _ptr(x, np.float64)
    _check(lib().igm_run_cycle(m.dev.h, m.h, C.byref(cc), pb, px0, px, C.byref(co), _tptr(trace)))
    d = co.dim
    return CycleResult(x=x, dim=d, r0_norm=co.r0_norm, g_abs=gabs[:d].copy(), cos=cd[:d].copy(),
                       sin=sd[:d].copy(), basis_norms=bn[:co.n_basis_norms].copy(),
                       basis=basis[:co.n_basis].copy() if state else None, hess=hess, g=g,
                       cos_raw=cr, sin_raw=sr)


@dataclass
class RefineConfig:
    tol: float = 1e-8
    max_refinements: int = 1000
    m: int = 30
    frac_bits: int = 30
    shifts: ShiftPlan = field(default_factory=ShiftPlan)
    s: int = 0
    checked: bool = True
    s_schedule: Optional[Callable[[int], int]] = None
    engine: int = 0  # 0 fixed_point, 1 floating_point (refine.hpp:22; refsolve.cpp)


@dataclass
class SolveReport:
    converged: bool
    refinements: int
    total_inner_iterations: int
    inner_dims: list
    relres_history: list
    gamma_history: list
    overflow_per_restart: list
    overflow_total: int
    wall_time_sec: float
    overflow_exact: bool


def solve(m: SplitMatrix, a_fp: CsrMatrixF, b, cfg: RefineConfig, precond: Optional[IluFactors] = None,
          trace: Optional[FxTrace] = None, x_out=None):
    R = max(cfg.max_refinements, 0)
    dims = np.zeros(R + 1, dtype=np.int32)
    rel = np.zeros(R + 2)
    gam = np.zeros(R + 1)
    ovf = np.zeros(R + 1, dtype=np.uint64)
    rep = _capi.Report()
    rep.inner_dims = dims.ctypes.data_as(_capi.i32p)
    rep.relres_history = rel.ctypes.data_as(_capi.f64p)
    rep.gamma_history = gam.ctypes.data_as(_capi.f64p)
    rep.overflow_per_restart = ovf.ctypes.data_as(_capi.u64p)
    rc = _capi.RefineCfg(cfg.tol, cfg.max_refinements, cfg.m, cfg.frac_bits, cfg.s,
                         1 if cfg.checked else 0, cfg.shifts.c(), None, _capi.SCHED_FN(), None, cfg.engine)
    cb = None
    if cfg.s_schedule is not None:
        fn = cfg.s_schedule
        cb = _capi.SCHED_FN(lambda user, k: int(fn(k)))
        rc.s_schedule_fn = cb
    x = x_out if x_out is not None else _out_like(b, m.n, np.float64)
    pb, k1 = _ptr(b, np.float64)
    px, k2 = _ptr(x, np.float64)
    _check(lib().igm_solve(m.dev.h, m.h, a_fp.h, pb, C.byref(rc), precond.h if precond is not None else None,
                           px, C.byref(rep), _tptr(trace)))
    k = rep.refinements
    report = SolveReport(
        converged=bool(rep.converged), refinements=k, total_inner_iterations=int(rep.total_inner_iterations),
        inner_dims=[int(v) for v in dims[:k]], relres_history=[float(v) for v in rel[:rep.n_relres]],
        gamma_history=[float(v) for v in gam[:k]], overflow_per_restart=[int(v) for v in ovf[:k]],
        overflow_total=int(rep.overflow_total), wall_time_sec=rep.wall_time_sec,
        overflow_exact=bool(rep.overflow_exact))
    return x, report


# ------------------------------------------------- config 3's WL = 32 variant
class SplitMatrix32:
    """A SplitMatrix's components narrowed to int32 words (igm_split32_from_split).
    WL = 32 has no reference implementation (fxp.hpp:22): parity is against
    oracle/igm_oracle32.c only (unpinned)."""

    def __init__(self, m: SplitMatrix):
        self.dev, self.n, self.ncomp, self.alphas = m.dev, m.n, m.ncomp, m.alphas
        self._src = m  # the CSR pattern is shared
        h = C.c_void_p()
        _check(lib().igm_split32_from_split(self.dev.h, m.h, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().igm_split32_free(self.h)
        except Exception:
            pass


def shifts32_plan(n: int, alpha_a: int, frac_bits: int) -> "ShiftPlan":
    """The builder's WL = 32 shift plan (igm_shifts32_plan)."""
    sh = _capi.Shifts()
    _check(lib().igm_shifts32_plan(int(n), alpha_a, frac_bits, C.byref(sh)))
    return ShiftPlan(sh.dot_b1, sh.dot_b2, sh.axpy_b1, sh.norm_b1, sh.div_b1, sh.div_b2, sh.givens_b2, sh.rot_b)


def run_cycle32(m: SplitMatrix32, m_steps: int, frac_bits: int, s: int, shifts: "ShiftPlan", b, checked=True):
    n = m.n
    cfg = _capi.Cycle32Cfg(m_steps, frac_bits, s, 1 if checked else 0, shifts.c())
    x = np.zeros(n)
    basis = np.zeros((m_steps + 1) * n, dtype=np.int32)
    hess = np.zeros((m_steps + 1) * m_steps, dtype=np.int32)
    g = np.zeros(m_steps + 1, dtype=np.int32)
    cs = np.zeros(m_steps, dtype=np.int32)
    sn = np.zeros(m_steps, dtype=np.int32)
    dim, nb, r0, ov = C.c_int(), C.c_int(), C.c_double(), C.c_uint64()
    pb, k1 = _ptr(b, np.float64)
    p = lambda a: C.c_void_p(a.ctypes.data)
    _check(lib().igm_run_cycle32(m.dev.h, m.h, C.byref(cfg), pb, p(x), C.byref(dim), C.byref(r0), p(basis),
                                 C.byref(nb), p(hess), p(g), p(cs), p(sn), C.byref(ov)))
    return dict(dim=dim.value, r0_norm=r0.value, basis=basis[:nb.value * n].copy(), n_basis=nb.value, hess=hess,
                g=g, cos_raw=cs, sin_raw=sn, x=x, overflows=int(ov.value))


def solve32(m: SplitMatrix32, a_fp: "CsrMatrixF", b, tol: float, max_refinements: int, m_steps: int, frac_bits: int,
            s: int, shifts: "ShiftPlan", checked=True, x_out=None):
    """The refinement loop around the WL = 32 cycle (igm_solve32)."""
    R = max(max_refinements, 0)
    dims = np.zeros(R + 1, dtype=np.int32)
    rel = np.zeros(R + 2)
    gam = np.zeros(R + 1)
    ovf = np.zeros(R + 1, dtype=np.uint64)
    rep = _capi.Report()
    rep.inner_dims = dims.ctypes.data_as(_capi.i32p)
    rep.relres_history = rel.ctypes.data_as(_capi.f64p)
    rep.gamma_history = gam.ctypes.data_as(_capi.f64p)
    rep.overflow_per_restart = ovf.ctypes.data_as(_capi.u64p)
    cfg = _capi.Cycle32Cfg(m_steps, frac_bits, s, 1 if checked else 0, shifts.c())
    x = x_out if x_out is not None else _out_like(b, m.n, np.float64)
    pb, k1 = _ptr(b, np.float64)
    px, k2 = _ptr(x, np.float64)
    _check(lib().igm_solve32(m.dev.h, m.h, a_fp.h, pb, C.c_double(tol), max_refinements, C.byref(cfg), px,
                             C.byref(rep)))
    k = rep.refinements
    return x, SolveReport(
        converged=bool(rep.converged), refinements=k, total_inner_iterations=int(rep.total_inner_iterations),
        inner_dims=[int(v) for v in dims[:k]], relres_history=[float(v) for v in rel[:rep.n_relres]],
        gamma_history=[float(v) for v in gam[:k]], overflow_per_restart=[int(v) for v in ovf[:k]],
        overflow_total=int(rep.overflow_total), wall_time_sec=rep.wall_time_sec,
        overflow_exact=bool(rep.overflow_exact))


def spmv_mgs(m: SplitMatrix, s: int, v_in, basis, k: int, f: int, dot_b1: int, dot_b2: int,
             axpy_b1: int, w):
    """Config-5 kernel call on device tensors: w = A v_in, then MGS against k basis vectors."""
    h = np.zeros(k, dtype=np.int64)
    for t in (v_in, basis, w):
        _ptr(t, np.int64)  # orders torch's stream before the call
    _check(lib().igm_spmv_mgs(m.dev.h, m.h, s, C.c_void_p(v_in.data_ptr()), C.c_void_p(basis.data_ptr()),
                              k, f, dot_b1, dot_b2, axpy_b1, C.c_void_p(w.data_ptr()),
                              h.ctypes.data_as(_capi.i64p)))
    return h


def mgs_pass(dev: "Device", mode: int, w, vprev, vcur, hacc, acc_out, f: int, dot_b1: int, dot_b2: int,
             axpy_b1: int) -> None:
    """One fused MGS pass on device tensors, enqueued on dev's stream (no sync):
    mode 0 dot, 1 axpy(vprev, h from hacc) + dot, 3 axpy only (igm_mgs_pass)."""
    p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    _check(lib().igm_mgs_pass(dev.h, int(w.numel()), mode, p(w), p(vprev), p(vcur), p(hacc), p(acc_out), f,
                              dot_b1, dot_b2, axpy_b1))


# ---------------------------------------------------------------- host setup
def row_scale(row_ptr, col_idx, vals, alpha_a: int):
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n = len(row_ptr) - 1
    out = np.empty_like(vals)
    scale = np.empty(n)
    _check(lib().igm_row_scale(n, C.c_void_p(row_ptr.ctypes.data), None, C.c_void_p(vals.ctypes.data),
                               alpha_a, C.c_void_p(out.ctypes.data), C.c_void_p(scale.ctypes.data)))
    return out, scale


def build_split(vals, alpha_a: int, max_components: int):
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    nnz = len(vals)
    comp = np.zeros((max(max_components, 1), nnz), dtype=np.int64)
    alphas = np.zeros(max(max_components, 1), dtype=np.int32)
    nc = C.c_int()
    ex = C.c_int()
    _check(lib().igm_build_split(0, nnz, C.c_void_p(vals.ctypes.data), alpha_a, max_components,
                                 C.c_void_p(comp.ctypes.data), C.c_void_p(alphas.ctypes.data),
                                 C.byref(nc), C.byref(ex)))
    return comp[:nc.value].copy(), [int(a) for a in alphas[:nc.value]], bool(ex.value)


def factorize_split_cast(row_ptr, col_idx, vals, return_lu: bool = False):
    """split_cast(factorize_ilu0(A)) -> (lower, upper) tuples of (row_ptr, col_idx, vals, diag_pos);
    return_lu: also the merged L, U values on A's pattern (ilu.cpp:29-49)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    n = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    lrp = np.zeros(n + 1, np.int32); urp = np.zeros(n + 1, np.int32)
    lci = np.zeros(nnz, np.int32); uci = np.zeros(nnz, np.int32)
    lv = np.zeros(nnz, np.int64); uv = np.zeros(nnz, np.int64)
    ldp = np.zeros(n, np.int32); udp = np.zeros(n, np.int32)
    p = lambda a: C.c_void_p(a.ctypes.data)
    lu = np.zeros(nnz, np.float64) if return_lu else None
    _check(lib().igm_factorize_split_cast_lu(n, p(row_ptr), p(col_idx), p(vals), p(lrp), p(lci), p(lv), p(ldp),
                                             p(urp), p(uci), p(uv), p(udp), p(lu) if return_lu else None))
    nl, nu = int(lrp[-1]), int(urp[-1])
    out = (lrp, lci[:nl].copy(), lv[:nl].copy(), ldp), (urp, uci[:nu].copy(), uv[:nu].copy(), udp)
    return out + (lu,) if return_lu else out


# ---------------------------------------------------------------- device setup
# row_scale / build_split / split_cast(factorize_ilu0)
# on the GPU (igm_*_dev), bit-identical to the host versions above.  numpy
# inputs give numpy outputs; torch CUDA tensors stay on the device.
def _alloc_like(t, n, dtype):
    if _is_torch(t) and t.is_cuda:
        import torch
        tdt = {np.int64: torch.int64, np.float64: torch.float64, np.int32: torch.int32}[dtype]
        return torch.empty(n, dtype=tdt, device=t.device)
    return np.empty(n, dtype=dtype)


def _vp(a, dtype):
    return _ptr(a, dtype)


def row_scale_device(row_ptr, col_idx, vals, alpha_a: int, device: Optional[Device] = None):
    dev = _dev(device)
    n = (row_ptr.numel() if _is_torch(row_ptr) else len(row_ptr)) - 1
    nnz = vals.numel() if _is_torch(vals) else len(vals)
    rp, k1 = _vp(row_ptr, np.int32)
    v, k2 = _vp(vals, np.float64)
    out, scale = _alloc_like(vals, nnz, np.float64), _alloc_like(vals, n, np.float64)
    po, k3 = _vp(out, np.float64)
    ps, k4 = _vp(scale, np.float64)
    _check(lib().igm_row_scale_dev(dev.h, n, rp, v, alpha_a, po, ps))
    return out, scale


def build_split_device(vals, alpha_a: int, max_components: int, device: Optional[Device] = None):
    dev = _dev(device)
    nnz = vals.numel() if _is_torch(vals) else len(vals)
    mc = max(max_components, 1)
    comp = _alloc_like(vals, mc * nnz, np.int64)
    v, k1 = _vp(vals, np.float64)
    pc, k2 = _vp(comp, np.int64)
    alphas = np.zeros(mc, dtype=np.int32)
    nc, ex = C.c_int(), C.c_int()
    _check(lib().igm_build_split_dev(dev.h, nnz, v, alpha_a, max_components, pc,
                                     C.c_void_p(alphas.ctypes.data), C.byref(nc), C.byref(ex)))
    k = nc.value
    return comp[:k * nnz].reshape(k, nnz), [int(a) for a in alphas[:k]], bool(ex.value)


def factorize_split_cast_device(row_ptr, col_idx, vals, device: Optional[Device] = None, return_lu: bool = False):
    """split_cast(factorize_ilu0(A)) on the device -> (lower, upper) tuples of
    (row_ptr, col_idx, vals, diag_pos), trimmed to the factors' sizes;
    return_lu: also the merged L, U values on A's pattern."""
    dev = _dev(device)
    n = (row_ptr.numel() if _is_torch(row_ptr) else len(row_ptr)) - 1
    nnz = col_idx.numel() if _is_torch(col_idx) else len(col_idx)
    bufs = [_alloc_like(vals, n + 1, np.int32), _alloc_like(vals, nnz, np.int32), _alloc_like(vals, nnz, np.int64),
            _alloc_like(vals, n, np.int32), _alloc_like(vals, n + 1, np.int32), _alloc_like(vals, nnz, np.int32),
            _alloc_like(vals, nnz, np.int64), _alloc_like(vals, n, np.int32)]
    ptrs = [_vp(b, b.dtype.type if isinstance(b, np.ndarray) else None)[0] if isinstance(b, np.ndarray)
            else C.c_void_p(b.data_ptr()) for b in bufs]
    rp, k1 = _vp(row_ptr, np.int32)
    ci, k2 = _vp(col_idx, np.int32)
    v, k3 = _vp(vals, np.float64)
    lu = _alloc_like(vals, nnz, np.float64) if return_lu else None
    plu = None if lu is None else (C.c_void_p(lu.ctypes.data) if isinstance(lu, np.ndarray)
                                   else C.c_void_p(lu.data_ptr()))
    _check(lib().igm_factorize_split_cast_dev_lu(dev.h, n, rp, ci, v, *ptrs, plu))
    lrp, lci, lv, ldp, urp, uci, uv, udp = bufs
    nl, nu = int(lrp[-1]), int(urp[-1])
    out = (lrp, lci[:nl], lv[:nl], ldp), (urp, uci[:nu], uv[:nu], udp)
    return out + (lu,) if return_lu else out
