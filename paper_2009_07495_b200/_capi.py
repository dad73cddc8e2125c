"""ctypes declarations of the C ABI in include/igm.h (libigm_b200.so).

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``).
Loading fails loudly when it is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libigm_b200.so"

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)

IGM_OK = 0
STATUS_NAMES = {
    0: "ok",
    1: "invalid_argument",
    2: "domain_error",
    3: "overflow_error",
    4: "runtime_error",
    5: "logic_error",
    6: "cuda_error",
    7: "nccl_error",
}

KERNEL_NAMES = ["", "spmv", "precond", "dot", "axpy", "norm", "vec_div", "givens",
                "givens_norm", "givens_div", "rot"]
OP_NAMES = ["", "add", "sub", "mul", "shl", "div"]
KCLASS_NAMES = ["spmv_int", "ilu_int", "ilu_fp", "mgs", "vec_div", "step_scalar", "norm2_serial",
                "residual_fp", "x_update", "encode", "other"]


class Shifts(C.Structure):
    _fields_ = [(n, C.c_int) for n in
                ("dot_b1", "dot_b2", "axpy_b1", "norm_b1", "div_b1", "div_b2", "givens_b2", "rot_b")]


class Trace(C.Structure):
    _fields_ = [
        ("checked", C.c_int), ("record_shifts", C.c_int),
        ("kernel", C.c_int), ("restart", C.c_int), ("step", C.c_int),
        ("total", C.c_uint64),
        ("n_events", C.c_int), ("cap_events", C.c_int), ("events", i32p),
        ("n_shifts", C.c_int64), ("cap_shifts", C.c_int), ("shifts", i32p),
        ("exact", C.c_int),
    ]


class CycleCfg(C.Structure):
    _fields_ = [("m", C.c_int), ("frac_bits", C.c_int), ("s", C.c_int), ("shifts", Shifts),
                ("precond", C.c_void_p), ("collect_basis_norms", C.c_int)]


class CycleOut(C.Structure):
    _fields_ = [
        ("dim", C.c_int), ("r0_norm", C.c_double),
        ("g_abs", f64p), ("cos_d", f64p), ("sin_d", f64p), ("basis_norms", f64p),
        ("n_basis_norms", C.c_int),
        ("basis", i64p), ("n_basis", C.c_int),
        ("hess", i64p), ("g", i64p), ("cos_raw", i64p), ("sin_raw", i64p),
    ]


class Cycle32Cfg(C.Structure):
    _fields_ = [("m", C.c_int), ("frac_bits", C.c_int), ("s", C.c_int), ("checked", C.c_int), ("shifts", Shifts)]


class DcInfo(C.Structure):
    _fields_ = [("dim", C.c_int), ("stop", C.c_int), ("nbasis", C.c_int), ("add_inexact", C.c_int),
                ("r0_norm", C.c_double), ("relnorm", C.c_double), ("nb", C.c_double), ("nr", C.c_double),
                ("gamma", C.c_double), ("overflows", C.c_uint64)]


IGM_DS_RED, IGM_DS_LCNT, IGM_DS_VCNT, IGM_DS_RMAX, IGM_DS_CHAIN = range(5)
K_COUNT, OP_COUNT = 11, 6

SCHED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int)


class RefineCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_refinements", C.c_int), ("m", C.c_int),
                ("frac_bits", C.c_int), ("s", C.c_int), ("checked", C.c_int),
                ("shifts", Shifts), ("s_schedule", i32p), ("s_schedule_fn", SCHED_FN),
                ("s_schedule_user", C.c_void_p), ("engine", C.c_int)]


class Report(C.Structure):
    _fields_ = [
        ("converged", C.c_int), ("refinements", C.c_int),
        ("total_inner_iterations", C.c_int64),
        ("inner_dims", i32p), ("relres_history", f64p), ("n_relres", C.c_int),
        ("gamma_history", f64p), ("overflow_per_restart", u64p),
        ("overflow_total", C.c_uint64), ("wall_time_sec", C.c_double),
        ("overflow_exact", C.c_int),
    ]


# (name, restype, argtypes) for every entry point declared in include/igm.h
SIGNATURES = [
    ("igm_ctx_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("igm_ctx_destroy", None, [C.c_void_p]),
    ("igm_ctx_synchronize", C.c_int, [C.c_void_p]),
    ("igm_ctx_stream", C.c_void_p, [C.c_void_p]),
    ("igm_ctx_launch_count", C.c_uint64, [C.c_void_p]),
    ("igm_set_exact_overflow_counts", C.c_int, [C.c_void_p, C.c_int]),
    ("igm_last_error", C.c_char_p, []),
    ("igm_version", C.c_char_p, []),
    ("igm_profile_enable", None, [C.c_int]),
    ("igm_profile_collect", C.c_int, [f64p, u64p]),
    ("igm_upload_split", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                   C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("igm_split_free", None, [C.c_void_p]),
    ("igm_upload_csrf", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
    ("igm_csrf_free", None, [C.c_void_p]),
    ("igm_upload_ilu", C.c_int, [C.c_void_p, C.c_int] + [C.c_void_p] * 8 + [C.POINTER(C.c_void_p)]),
    ("igm_ilu_free", None, [C.c_void_p]),
    ("igm_ilu_levels", C.c_int, [C.c_void_p, C.c_int]),
    ("igm_ilu_schedule_info", None, [C.c_void_p, C.c_int, i32p]),
    ("igm_ilu_pencil", C.c_int, [C.c_void_p, C.c_int]),
    ("igm_debug_pencil_stream", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                          C.c_int, C.c_int, C.c_int, i32p]),
    ("igm_debug_pencil27_stream", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                            C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong)]),
    ("igm_debug_tri_trace", None, [C.c_int, C.c_void_p]),
    ("igm_debug_arn_ts", C.c_int, [C.c_int, C.c_void_p, C.c_int]),
    ("igm_debug_fx_selftest", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("igm_debug_tri_schedule", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_int, i32p]),
    ("igm_spmv", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(Trace)]),
    ("igm_apply_inverse", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Trace)]),
    ("igm_apply_inverse_fp", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("igm_fx_dot", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                             i64p, C.POINTER(Trace)]),
    ("igm_fx_norm", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int, i64p,
                              C.POINTER(Trace)]),
    ("igm_fx_axpy_sub", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int,
                                  C.c_int, C.POINTER(Trace)]),
    ("igm_spmv_fp", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("igm_residual_fp", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, f64p]),
    ("igm_spmv_fp_split", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    ("igm_norm2", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, f64p]),
    ("igm_gamma_scale", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, f64p, C.c_void_p]),
    ("igm_run_cycle", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(CycleCfg), C.c_void_p, C.c_void_p,
                                C.c_void_p, C.POINTER(CycleOut), C.POINTER(Trace)]),
    ("igm_solve", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(RefineCfg),
                            C.c_void_p, C.c_void_p, C.POINTER(Report), C.POINTER(Trace)]),
    ("igm_spmv_mgs", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                               C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, i64p]),
    ("igm_fp_cycle", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_void_p]),
    ("igm_mgs_pass", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    # row-block partition building blocks (dist.solve_sharded); device pointers, asynchronous
    ("igm_dstate_create", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    ("igm_dstate_free", None, [C.c_void_p]),
    ("igm_dstate_buffer", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    ("igm_dc_reset", C.c_int, [C.c_void_p, C.c_void_p]),
    ("igm_dc_residual", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("igm_dc_norm2", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("igm_dc_begin", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("igm_dc_scale", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("igm_dc_tri_fp", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    ("igm_dc_tri", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                             C.c_int]),
    ("igm_dc_tri_piped", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                   C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_uint64]),
    ("igm_dev_alloc", C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_void_p)]),
    ("igm_dev_free", None, [C.c_void_p]),
    ("igm_ipc_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("igm_ipc_open", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("igm_ipc_close", None, [C.c_void_p]),
    # one-shot P2P mailbox reductions
    ("igm_mbox_create", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("igm_mbox_free", None, [C.c_void_p]),
    ("igm_mbox_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("igm_mbox_connect_ipc", C.c_int, [C.c_void_p, C.c_void_p]),
    ("igm_mbox_connect_local", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("igm_mbox_publish", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("igm_mbox_collect", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("igm_mbox_allreduce", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("igm_mbox_status", C.c_int, [C.c_void_p, C.c_void_p]),
    ("igm_dc_encode", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]),
    ("igm_dc_spmv", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                              C.c_int]),
    ("igm_dc_mgs_pass", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_int, C.POINTER(Shifts), C.c_int]),
    ("igm_dc_step", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(Shifts), C.c_void_p,
                              C.c_int]),
    ("igm_dc_vec_div", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                 C.POINTER(Shifts), C.c_int]),
    ("igm_dc_finish", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]),
    ("igm_dc_fetch", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    # config 3's WL = 32 variant
    ("igm_split32_from_split", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("igm_split32_free", None, [C.c_void_p]),
    ("igm_shifts32_plan", C.c_int, [C.c_longlong, C.c_int, C.c_int, C.POINTER(Shifts)]),
    ("igm_run_cycle32", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Cycle32Cfg), C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int),
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    ("igm_solve32", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                              C.POINTER(Cycle32Cfg), C.c_void_p, C.POINTER(Report)]),
    ("igm_row_scale_dev", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                    C.c_void_p]),
    ("igm_build_split_dev", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                      C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("igm_factorize_split_cast_dev", C.c_int, [C.c_void_p, C.c_int] + [C.c_void_p] * 11),
    ("igm_row_scale", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                C.c_void_p]),
    ("igm_build_split", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                  C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("igm_factorize_split_cast", C.c_int, [C.c_int] + [C.c_void_p] * 11),
    ("igm_factorize_split_cast_lu", C.c_int, [C.c_int] + [C.c_void_p] * 12),
    ("igm_factorize_split_cast_dev_lu", C.c_int, [C.c_void_p, C.c_int] + [C.c_void_p] * 12),
]

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load libigm_b200.so (no fallback: raises if it has not been built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(f"{p} is missing: build it with `make` or __graft_entry__.build(); "
                           "the int-GMRES path has no CPU fallback")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
