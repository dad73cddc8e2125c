"""Config 3's WL = 32 variant (BASELINE.json configs[2]: "WL=32 fixed point").

The reference hard-wires WL = 64 (fxp.hpp:22; SPEC.md:149 non-goal), so this
path has NO reference implementation: PARITY IS UNPINNED.  What pins it:
  * the CPU restatement oracle/igm_oracle32.c reproduces the reference-pinned
    WL = 64 restatement (oracle/igm_oracle.c) word for word on inputs where no
    32-bit word overflows (test_oracle32_matches_wl64_without_overflow), so its
    control flow and shift semantics are the reference's;
  * the CUDA path (csrc/wl32.cu, igm_run_cycle32 / igm_solve32) is compared
    word for word with that restatement, including wrapping runs.
"""
import hashlib

import numpy as np
import pytest

from workloads import gen


def _h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _setup(O, rp, ci, v, alpha):
    A = O.csrf(rp, ci, v)
    vals, scale = O.row_scale(A, alpha)
    comp, al, _ = O.build_split(vals, alpha, 1)
    return vals, scale, comp, al


def test_oracle32_matches_wl64_without_overflow(oracle):
    from oracle.ffi import Oracle32, Shifts
    O32 = Oracle32()
    rp, ci, v = gen.upwind_2d(8)
    n = len(rp) - 1
    for alpha, f, sh in [(4, 14, (8, 2, 6, 8, 5, 5, 6, 0)), (5, 14, (9, 3, 7, 9, 4, 6, 7, 0))]:
        vals, scale, comp, al = _setup(oracle, rp, ci, v, alpha)
        b = gen.uniform(5, n) / scale
        c32 = O32.run_cycle(rp, ci, comp.astype(np.int32), al, 10, f, 0, Shifts(*sh), b)
        c64 = oracle.run_cycle(oracle.split(rp, ci, comp, al), 10, f, 0, Shifts(*sh), b, np.zeros(n))
        assert c32["overflows"] == 0
        assert c32["dim"] == c64["dim"] and c32["n_basis"] == c64["n_basis"]
        assert np.array_equal(c32["basis"].astype(np.int64), np.asarray(c64["basis"]).ravel()[:c32["basis"].size])
        assert np.array_equal(c32["hess"].astype(np.int64), c64["hess"])
        assert np.array_equal(c32["g"].astype(np.int64), c64["g"])
        assert np.array_equal(c32["x"], c64["x"])


def test_shifts32_plan_rule(igm):
    # the builder's plan (igm_shifts32_plan): every product and n-term sum of
    # the cycle inside 31 bits for O(1) basis words, |A| <= 2^alpha
    p = igm.shifts32_plan(1_000_000, 8, 18)
    assert (p.dot_b1, p.dot_b2, p.axpy_b1, p.norm_b1, p.div_b1, p.div_b2, p.givens_b2, p.rot_b) == \
        (17, 9, 15, 13, 3, 11, 16, 3)
    for n in (64, 3000, 10 ** 6):
        for f in (14, 16, 18, 20):
            q = igm.shifts32_plan(n, 8, f)
            assert q.rot_b == max(0, f - 15) and 2 * (f - q.norm_b1) <= 30
            assert 0 <= q.div_b1 <= f and q.div_b1 + q.div_b2 <= f


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["band3000", "upwind2d", "band3000_wrap"])
def test_run_cycle32_bit_exact(igm, oracle, case):
    from oracle.ffi import Oracle32, Shifts
    O32 = Oracle32()
    if case.startswith("band"):
        n = 3000
        rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
        alpha, f, m = 8, 20, 50
    else:
        rp, ci, v = gen.upwind_2d(8)
        n = len(rp) - 1
        alpha, f, m = 6, 16, 20
    vals, scale, comp, al = _setup(oracle, rp, ci, v, alpha)
    b = gen.uniform(gen.SEED_BASE ^ 103, n) / scale
    sh = igm.shifts32_plan(n, alpha, f)
    if case.endswith("wrap"):  # no guard shifts: products and sums wrap mod 2^32
        sh = igm.ShiftPlan(0, 0, 0, f - 15, 0, 0, 0, f - 15)
    S = igm.SplitMatrix(rp, ci, comp, al)
    S32 = igm.SplitMatrix32(S)
    try:
        ref = O32.run_cycle(rp, ci, comp.astype(np.int32), al, m, f, 0, Shifts(*sh.astuple()), b)
    except RuntimeError as e:
        # the wrapping plan ends in a domain error (a wrapped norm accumulator or
        # a zero divisor) in the restatement: the CUDA path must raise as well
        with pytest.raises((ArithmeticError, RuntimeError, ValueError)):
            igm.run_cycle32(S32, m, f, 0, sh, b)
        return
    got = igm.run_cycle32(S32, m, f, 0, sh, b)
    assert got["dim"] == ref["dim"] and got["n_basis"] == ref["n_basis"]
    assert got["r0_norm"] == ref["r0_norm"]
    assert np.array_equal(got["basis"], ref["basis"])
    for k in ("hess", "g", "cos_raw", "sin_raw"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["x"], ref["x"])
    if not case.endswith("wrap"):
        assert got["overflows"] == ref["overflows"] == 0


@pytest.mark.gpu
def test_solve32_bit_exact(igm, oracle):
    from oracle.ffi import Oracle32, Shifts
    O32 = Oracle32()
    n = 30000
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    alpha, f = 8, 18
    vals, scale, comp, al = _setup(oracle, rp, ci, v, alpha)
    b = gen.uniform(gen.SEED_BASE ^ 103, n) / scale
    sh = igm.shifts32_plan(n, alpha, f)
    xr, rr = O32.solve(rp, ci, comp.astype(np.int32), al, vals, b, 1e-10, 30, 50, f, 0, Shifts(*sh.astuple()))
    S32 = igm.SplitMatrix32(igm.SplitMatrix(rp, ci, comp, al))
    A = igm.CsrMatrixF(rp, ci, vals)
    x, rep = igm.solve32(S32, A, b, 1e-10, 30, 50, f, 0, sh)
    assert rr["converged"] and rep.converged
    assert rep.relres_history == rr["relres_history"]
    assert rep.gamma_history == rr["gamma_history"]
    assert rep.inner_dims == rr["inner_dims"]
    assert rep.overflow_total == rr["overflow_total"] == 0
    assert _h(x) == _h(xr)
