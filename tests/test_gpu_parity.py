"""Parity of the B200 path (C ABI -> sm_100a kernels) with the CPU oracle and
with golden outputs of the reference library.  Bit-exact on every integer
word (basis, Hessenberg, g, rotations, SpMV / ILU outputs) and on the FP64
bookends (x, residual history) -- the FP kernels reproduce the reference's
operation order with no contraction."""
import hashlib
import os
import re

import numpy as np
import pytest

from oracle.ffi import PyTrace, Shifts
from tests.cases import CASES, build_case

pytestmark = pytest.mark.gpu
I64_MIN, I64_MAX = np.iinfo(np.int64).min, np.iinfo(np.int64).max


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gpu(igm):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return igm


def product_case(igm, oracle, name):
    c = build_case(name, oracle)
    c["S"] = igm.SplitMatrix(c["rp"], c["ci"], c["comp"], c["alphas"])
    c["A"] = igm.CsrMatrixF(c["rp"], c["ci"], c["vals"])
    if c.get("ilu"):
        c["F"] = igm.IluFactors(c["lower"], c["upper"])
    c["plan"] = igm.ShiftPlan(*c["shifts"])
    return c


@pytest.mark.parametrize("name", sorted(CASES))
def test_spmv_bit_exact(gpu, oracle, goldens, name):
    c = product_case(gpu, oracle, name)
    rng = np.random.default_rng(1)
    for s in range(c["ncomp"]):
        for v in (c["v_full"], rng.integers(-(1 << 31), 1 << 31, c["n"], dtype=np.int64)):
            t1, t2 = gpu.FxTrace(), PyTrace()
            out = gpu.spmv(c["S"], s, v, t1)
            assert np.array_equal(out, oracle.spmv(c["sp"], s, v, t2))
            assert t1.total_overflows() == t2.total  # per-row sequential: exact
            assert t1.events == t2.events  # split.cpp:141-153 order (trace_order.cu)
        if "spmv" in goldens["cases"][name]:
            assert h(gpu.spmv(c["S"], s, c["v_full"])) == goldens["cases"][name]["spmv"][str(s)]


@pytest.mark.parametrize("kind", ["27pt_18", "band_6000", "7pt_17"])
def test_spmv_layout_variants_bit_exact(gpu, oracle, kind, monkeypatch):
    """The integer SpMV kernels that re-lay the matrix or its loads out --
    k_spmv_int_sell (sliced ELL: rows of 9..32 entries), k_spmv_int_r8
    (register-batched: short rows), k_spmv_int_staged (IGM_SPMV_SELL=0 on long
    rows) -- against the oracle's split.cpp:137-157 on matrices of n >= 4096:
    every output word, the checked-mode event totals and the ordered event
    lists, on full-range vectors (products and running sums wrap) and on
    small ones."""
    from workloads import gen
    if kind == "27pt_18":
        rp, ci, v = gen.stencil27(18, 3)
    elif kind == "band_6000":
        rp, ci, v = gen.random_band_fast(6000, 9)
    else:
        rp, ci, v = gen.upwind_3d(17, 20.0)
    n = len(rp) - 1
    vals, _ = oracle.row_scale(oracle.csrf(rp, ci, v), 32)
    comp, al, _ = oracle.build_split(vals, 32, 1)
    sp = oracle.split(rp, ci, comp, al)
    rng = np.random.default_rng(5)
    vecs = (rng.integers(-(1 << 63), (1 << 63) - 1, n, dtype=np.int64),
            rng.integers(-(1 << 28), 1 << 28, n, dtype=np.int64))
    for env in ({}, {"IGM_SPMV_SELL": "0"}):
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        S = gpu.SplitMatrix(rp, ci, comp, al)  # (the sliced copy is decided at upload)
        for vec in vecs:
            t1, t2 = gpu.FxTrace(), PyTrace()
            out = gpu.spmv(S, 0, vec, t1)
            assert np.array_equal(out, oracle.spmv(sp, 0, vec, t2)), (kind, env)
            assert t1.total_overflows() == t2.total
            assert t1.events == t2.events
            assert np.array_equal(gpu.spmv(S, 0, vec), out)  # unchecked path
        for k in env:
            monkeypatch.delenv(k)


@pytest.mark.parametrize("name", ["cfg2_16", "cfg4_12", "ilu_random"])
def test_ilu_apply_bit_exact(gpu, oracle, goldens, name):
    c = product_case(gpu, oracle, name)
    g = goldens["cases"][name]
    assert h(gpu.apply_inverse(c["F"], c["y_int"])) == g["apply_inverse"]
    assert h(gpu.apply_inverse_fp(c["F"], c["y_fp"])) == g["apply_inverse_fp"]
    for y in (c["v_full"], c["y_int"]):
        t1, t2 = gpu.FxTrace(), PyTrace()
        assert np.array_equal(gpu.apply_inverse(c["F"], y, t1), oracle.apply_inverse(c["il"], y, t2))
        assert t1.total_overflows() == t2.total
        assert t1.events == t2.events
    for _ in range(3):  # repeated launches: the spin-wait protocol is re-armed every call
        assert h(gpu.apply_inverse(c["F"], c["y_int"])) == g["apply_inverse"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_run_cycle_state_bit_exact(gpu, oracle, goldens, name):
    c = product_case(gpu, oracle, name)
    cfg = gpu.CycleConfig(m=c["m"], frac_bits=30, shifts=c["plan"], s=c["s"], precond=c.get("F"))
    r = gpu.run_cycle(c["S"], cfg, c["b"], np.zeros(c["n"]))
    g = goldens["cases"][name]["cycle"]
    assert r.dim == g["dim"] and r.r0_norm == g["r0_norm"] and len(r.basis) == g["n_basis"]
    assert h(r.basis) == g["basis"]
    assert h(r.hess) == g["hess"] and h(r.g) == g["g"]
    assert h(r.cos_raw) == g["cos_raw"] and h(r.sin_raw) == g["sin_raw"]
    assert h(r.x) == g["x"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_solve_bit_exact(gpu, oracle, goldens, name):
    c = product_case(gpu, oracle, name)
    cfg = gpu.RefineConfig(tol=c["tol"], max_refinements=c["max_ref"], m=c["m"], frac_bits=30,
                           shifts=c["plan"], s=c["s"], checked=True)
    x, rep = gpu.solve(c["S"], c["A"], c["b"], cfg, precond=c.get("F"))
    g = goldens["cases"][name]["solve"]
    assert h(x) == g["x"]
    want = g["report"]
    assert rep.converged == want["converged"] and rep.refinements == want["refinements"]
    assert rep.total_inner_iterations == want["total_inner_iterations"]
    assert rep.inner_dims == want["inner_dims"]
    assert rep.relres_history == want["relres_history"]
    assert rep.gamma_history == want["gamma_history"]
    assert rep.overflow_per_restart == want["overflow_per_restart"]
    assert rep.overflow_total == want["overflow_total"] and rep.overflow_exact


def test_vector_kernels_random(gpu, oracle):
    rng = np.random.default_rng(99)
    for n in (1, 2, 31, 64, 1000, 4097, 100003):
        v = rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64)
        w = rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64)
        b1, b2 = int(rng.integers(0, 30)), int(rng.integers(0, 30))
        assert gpu.fx_dot(v, w, 30, b1, b2) == oracle.fx_dot(v, w, 30, b1, b2)
        hh = int(rng.integers(I64_MIN, I64_MAX))
        t1, t2 = gpu.FxTrace(), PyTrace()
        ww = w.copy()
        gpu.fx_axpy_sub(ww, hh, v, 30, b1, t1)
        assert np.array_equal(ww, oracle.fx_axpy_sub(w, hh, v, 30, b1, t2))
        assert t1.total_overflows() == t2.total
        assert t1.events == t2.events
        t1, t2 = gpu.FxTrace(), PyTrace()
        assert gpu.fx_dot(v, w, 30, b1, b2, t1) == oracle.fx_dot(v, w, 30, b1, b2, t2)
        assert t1.events == t2.events  # mul / running-sum add per element (fxp.cpp:57-61), then the shl
        lim = (1 << 40) if n < 10000 else (1 << 33)  # keep sum of squares < 2^63
        u = rng.integers(-lim, lim, n, dtype=np.int64)
        t1, t2 = gpu.FxTrace(), PyTrace()
        assert gpu.fx_norm(u, 30, 16, t1) == oracle.fx_norm(u, 30, 16, t2)
        assert t1.total_overflows() == t2.total  # square wraps are exact
        assert t1.events == t2.events
        x = rng.uniform(-1, 1, n)
        assert gpu.norm2(x) == oracle.norm2(x)


def test_norm_wrap_raises(gpu):
    with pytest.raises(ArithmeticError, match="wrapped negative"):
        gpu.fx_norm(np.array([3 << 30], dtype=np.int64), 30, 0)  # test_fxp.cpp:144-149


def test_fp_bookends_bit_exact(gpu, oracle):
    c = product_case(gpu, oracle, "cfg1")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, c["n"])
    r1, rel1 = gpu.residual_fp(c["A"], x, c["b"])
    r2, rel2 = oracle.residual_fp(c["af"], x, c["b"])
    assert np.array_equal(r1, r2) and rel1 == rel2
    assert np.array_equal(gpu.spmv_fp_split(c["S"], 0, x), oracle.spmv_fp_split(c["sp"], 0, x))
    g, bk = gpu.gamma_scale(r1)
    assert g == np.abs(r2).max() and np.array_equal(bk, r2 / g)
    with pytest.raises(ValueError, match="zero residual"):
        gpu.gamma_scale(np.zeros(4))


def test_run_cycle_nonzero_x0(gpu, oracle):
    c = product_case(gpu, oracle, "split_s3")
    x0 = np.random.default_rng(5).uniform(-1, 1, c["n"])
    cfg = gpu.CycleConfig(m=c["m"], frac_bits=30, shifts=c["plan"], s=c["s"])
    r = gpu.run_cycle(c["S"], cfg, c["b"], x0)
    o = oracle.run_cycle(c["sp"], c["m"], 30, c["s"], Shifts(*c["shifts"]), c["b"], x0)
    assert r.dim == o["dim"] and np.array_equal(r.x, o["x"]) and np.array_equal(r.basis, o["basis"])


def test_cycle_edge_cases(gpu, oracle):
    from workloads import gen
    # zero right-hand side: x unchanged, dim 0 (test_gmres_cycle.cpp:192-204)
    rp, ci, v = gen.laplacian2d(3)
    comp, al, _ = gpu.build_split(v, 16, 4)
    S = gpu.SplitMatrix(rp, ci, comp, al)
    cfg = gpu.CycleConfig(m=5, frac_bits=30, shifts=gpu.ShiftPlan.default_unpreconditioned(30))
    r = gpu.run_cycle(S, cfg, np.zeros(9), np.zeros(9))
    assert r.dim == 0 and r.r0_norm == 0.0 and not r.x.any()
    # cyclic permutation: exact happy breakdown at step n (test_gmres_cycle.cpp:167-190)
    n = 8
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.array([(i - 1) % n for i in range(n)], dtype=np.int32)
    comp, al, _ = gpu.build_split(np.ones(n), 16, 2)
    S = gpu.SplitMatrix(rp, ci, comp, al)
    b = np.zeros(n)
    b[0] = 1.0
    r = gpu.run_cycle(S, gpu.CycleConfig(m=n + 4, frac_bits=30, shifts=gpu.ShiftPlan.default_unpreconditioned(30)),
                      b, np.zeros(n))
    assert r.dim == n and len(r.basis) == n
    # argument validation (test_gmres_cycle.cpp:206-221)
    with pytest.raises(ValueError, match="m must be"):
        gpu.run_cycle(S, gpu.CycleConfig(m=0, shifts=gpu.ShiftPlan.default_unpreconditioned(30)), b, np.zeros(n))
    with pytest.raises(ValueError, match="splitting depth"):
        gpu.run_cycle(S, gpu.CycleConfig(m=5, s=5, shifts=gpu.ShiftPlan.default_unpreconditioned(30)), b,
                      np.zeros(n))


def test_solve_edge_cases(gpu, oracle):
    c = product_case(gpu, oracle, "cfg1")
    plan = c["plan"]
    # zero rhs converges with no refinement (test_refine.cpp:372-380)
    x, rep = gpu.solve(c["S"], c["A"], np.zeros(c["n"]), gpu.RefineConfig(m=5, shifts=plan))
    assert rep.converged and rep.refinements == 0 and rep.relres_history == [0.0] and not x.any()
    # max_refinements = 0 reports the initial state (test_refine.cpp:382-390)
    x, rep = gpu.solve(c["S"], c["A"], c["b"], gpu.RefineConfig(m=5, shifts=plan, max_refinements=0))
    assert not rep.converged and rep.refinements == 0 and rep.relres_history == [1.0]
    with pytest.raises(ValueError, match="max_refinements"):
        gpu.solve(c["S"], c["A"], c["b"], gpu.RefineConfig(m=5, shifts=plan, max_refinements=-1))


def test_s_schedule_consulted_once_per_refinement(gpu, oracle):
    c = product_case(gpu, oracle, "split_s3")
    asked = []
    full = c["ncomp"] - 1

    def sched(k):
        asked.append(k)
        return min(k, full)
    cfg = gpu.RefineConfig(tol=1e-10, max_refinements=100, m=c["m"], shifts=c["plan"], s_schedule=sched)
    x, rep = gpu.solve(c["S"], c["A"], c["b"], cfg)
    assert asked == list(range(rep.refinements))
    xo, ro = oracle.solve(c["sp"], c["af"], c["b"], 1e-10, 100, c["m"], 30, 0, Shifts(*c["shifts"]),
                          s_schedule=[min(k, full) for k in range(100)])
    assert np.array_equal(x, xo) and rep.relres_history == ro["relres_history"]


def test_overflow_counts_and_traces(gpu, oracle):
    """Removing the dot guard shift wraps products (test_refine.cpp:392-426):
    the device counts events exactly and surfaces the same failure."""
    from workloads import gen
    rp, ci, v = gen.laplacian2d(8)
    vals, scale = gpu.row_scale(rp, ci, v, 16)
    comp, al, _ = gpu.build_split(vals, 16, 10)
    S = gpu.SplitMatrix(rp, ci, comp, al)
    A = gpu.CsrMatrixF(rp, ci, vals)
    b = np.ones(len(rp) - 1) / scale
    plan = gpu.ShiftPlan(0, 0, 16, 16, 16, 14, 16, 0)
    t = gpu.FxTrace(checked=True)
    try:
        gpu.solve(S, A, b, gpu.RefineConfig(tol=1e-8, max_refinements=3, m=6, shifts=plan, s=len(al) - 1), trace=t)
        threw = None
    except (ArithmeticError, ValueError, OverflowError, RuntimeError) as e:
        threw = type(e)
    sp = oracle.split(rp, ci, comp, al)
    to = PyTrace()
    from oracle.ffi import CheckerError
    try:
        oracle.solve(sp, oracle.csrf(rp, ci, vals), b, 1e-8, 3, 6, 30, len(al) - 1, Shifts(0, 0, 16, 16, 16, 14, 16, 0),
                     trace=to)
        othrew = None
    except CheckerError as e:
        othrew = e.code
    assert t.total_overflows() > 0 and to.total > 0
    assert (threw is None) == (othrew is None)
    assert t.events[0][2] == 0  # first events belong to restart 0
    if t.exact:
        assert t.total_overflows() == to.total


def test_spmv_mgs_microbench_parity(gpu, oracle):
    """Config-5 call (SpMV + MGS against k basis vectors, unchecked) at small n."""
    import torch
    from workloads import gen
    rp, ci, v = gen.upwind_3d(20, 20.0)
    vals, _ = gpu.row_scale(rp, ci, v, 16)
    comp, al, _ = gpu.build_split(vals, 16, 1)
    S = gpu.SplitMatrix(rp, ci, comp, al)
    n, k = len(rp) - 1, 7
    basis = gen.uniform_int(5, k * n, -(1 << 40), 1 << 40).reshape(k, n)
    vin = gen.uniform_int(6, n, -(1 << 40), 1 << 40)
    w = torch.empty(n, dtype=torch.int64, device="cuda")
    hs = gpu.spmv_mgs(S, 0, torch.from_numpy(vin).cuda(), torch.from_numpy(basis).cuda(), k, 30, 16, 0, 16, w)
    sp = oracle.split(rp, ci, comp, al)
    wo = oracle.spmv(sp, 0, vin)
    for i in range(k):
        hi = oracle.fx_dot(wo, basis[i], 30, 16, 0)
        assert hi == hs[i]
        wo = oracle.fx_axpy_sub(wo, hi, basis[i], 30, 16)
    assert np.array_equal(w.cpu().numpy(), wo)


def test_device_resident_inputs(gpu, oracle):
    """torch CUDA tensors are used in place (no staging) and give the same bits."""
    import torch
    c = product_case(gpu, oracle, "cfg2_16")
    cfg = gpu.RefineConfig(tol=c["tol"], max_refinements=c["max_ref"], m=c["m"], shifts=c["plan"])
    xh, _ = gpu.solve(c["S"], c["A"], c["b"], cfg, precond=c["F"])
    xd = torch.empty(c["n"], dtype=torch.float64, device="cuda")
    gpu.solve(c["S"], c["A"], torch.from_numpy(c["b"]).cuda(), cfg, precond=c["F"], x_out=xd)
    assert np.array_equal(xh, xd.cpu().numpy())
    yd = gpu.apply_inverse(c["F"], torch.from_numpy(c["y_int"]).cuda())
    assert np.array_equal(yd.cpu().numpy(), gpu.apply_inverse(c["F"], c["y_int"]))


def _norm2_cases():
    rng = np.random.default_rng(2024)
    cases = [np.zeros(0), np.zeros(5), np.array([3.0, 4.0]), rng.uniform(-1, 1, 1),
             rng.uniform(-1, 1, 8191), rng.uniform(-1, 1, 8192), rng.uniform(-1, 1, 8193),
             rng.uniform(-1, 1, 300000)]
    # exact powers of two: every term exact, many binade crossings
    cases.append(np.ldexp(1.0, rng.integers(-40, 40, 50000)))
    # ties: running sum in [2,4) has ulp 2^-51; (2^-26)^2 = 2^-52 is exactly half an ulp
    t = np.full(40000, 2.0 ** -26)
    t[0] = 1.5
    t[1000::997] = 2.0 ** -25.5 if False else 1.0
    cases.append(t)
    t2 = np.full(30000, 2.0 ** -26)
    t2[0] = np.sqrt(2.5)
    cases.append(t2)
    # subnormal squares and huge dynamic range
    cases.append(np.concatenate([np.full(5000, 1e-160), rng.uniform(-1, 1, 5000) * 1e-155]))
    cases.append(rng.uniform(-1, 1, 60000) * np.ldexp(1.0, rng.integers(-500, 500, 60000)))
    # overflow to inf, then nan
    cases.append(np.array([1e200, 1e200, 1.0]))
    cases.append(np.array([1.0, np.nan, 2.0]))
    return cases


def test_norm2_exact_parallel_chain(gpu, oracle):
    """The parallel norm2 (binade automaton scan) is bit-identical to the
    sequential FP64 chain of split.cpp:45-49 on adversarial data."""
    for x in _norm2_cases():
        a = gpu.norm2(x)
        b = oracle.norm2(x)
        assert np.float64(a).tobytes() == np.float64(b).tobytes(), (len(x), a, b)


@pytest.mark.parametrize("g,k", [(96, 30), (256, 8)])
def test_spmv_mgs_large_vs_torch(gpu, g, k):
    """Config-5 call at scale (n = g^3, vectors far beyond L2) against an
    independent torch int64 implementation: wrapping products, arithmetic
    shifts (floor), wrapping sums -- the same mod-2^64 algebra."""
    import torch
    from workloads import gen
    rp, ci, v = gen.upwind_3d_lean(g, 20.0)
    vals, _ = gpu.row_scale(rp, ci, v, 16)
    comp, al, _ = gpu.build_split(vals, 16, 1)
    S = gpu.SplitMatrix(rp, ci, comp, al)
    n = len(rp) - 1
    basis = torch.stack([gen.device_uniform_int40(n, 99, (i + 1) * n) for i in range(k)])
    vin = gen.device_uniform_int40(n, 99, 0)
    w = torch.empty(n, dtype=torch.int64, device="cuda")
    hs = gpu.spmv_mgs(S, 0, vin, basis, k, 30, 16, 0, 16, w)
    # torch reference
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.from_numpy(np.diff(rp).astype(np.int64)).cuda())
    prod = torch.from_numpy(comp[0]).cuda() * vin[torch.from_numpy(ci.astype(np.int64)).cuda()]
    wr = torch.zeros(n, dtype=torch.int64, device="cuda").index_add_(0, rows, prod)
    for i in range(k):
        acc = int(((wr >> 16) * basis[i]).sum().item())
        h = acc >> 14  # fx_dot finalisation: e = f - b1 - b2 = 14
        assert h == hs[i]
        wr = wr - (((h >> 16) * basis[i]) >> 14)
    assert torch.equal(wr, w)


def _grid_factors(gpu, dims, offs, seed):
    from workloads import gen
    rng = np.random.default_rng(seed)
    coef = {k: rng.uniform(-1.4, -0.6) for k in range(len(offs))}
    centre = offs.index((0, 0, 0))
    coef[centre] = 2.0 * len(offs)
    rp, ci, v = gen._stencil_csr(dims, offs, lambda o, r: np.full(r.shape, coef[o]))
    vals, _ = gpu.row_scale(rp, ci, v, 32)
    return gpu.factorize_split_cast(rp, ci, vals)


_SEVEN = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
_TWENTY7 = [(a, b, c) for c in (-1, 0, 1) for b in (-1, 0, 1) for a in (-1, 0, 1)]


@pytest.mark.parametrize("dims,offs", [((64, 64, 80), _SEVEN), ((128, 48, 70), _SEVEN), ((40, 40, 40), _TWENTY7)],
                         ids=["7pt-64x64x80", "7pt-128x48x70", "27pt-40cube"])
def test_ilu_apply_multi_tile(gpu, oracle, dims, offs):
    """Bit-exact ILU apply on grids of many bricks / z-layers and > 148*8*256
    rows (every launch path of the wavefront: cross-tile words, capped grids),
    integer, FP and checked, over repeated launches."""
    lo, up = _grid_factors(gpu, dims, offs, seed=sum(dims))
    F = gpu.IluFactors(lo, up)
    assert F.schedule_info(False)["tiles"] > 1
    il = oracle.ilu(lo, up)
    n = len(lo[0]) - 1
    from workloads import gen
    y = gen.uniform_int(11, n, -(1 << 45), 1 << 45)
    want = oracle.apply_inverse(il, y)
    for _ in range(3):
        assert np.array_equal(gpu.apply_inverse(F, y), want)
    yf = gen.uniform(12, n)
    assert np.array_equal(gpu.apply_inverse_fp(F, yf), oracle.apply_inverse_fp(il, yf))
    t1, t2 = gpu.FxTrace(), PyTrace()
    yw = gen.uniform_int(13, n, -(1 << 62), 1 << 62)
    assert np.array_equal(gpu.apply_inverse(F, yw, t1), oracle.apply_inverse(il, yw, t2))
    assert t1.total_overflows() == t2.total


def test_ilu_apply_unstructured_many_tiles(gpu, oracle):
    """Contiguous-block tiling (no grid detected) with long cross-tile lists."""
    from workloads import gen
    rp, ci, v = gen.random_dominant(4000, 0.002, 1.3, gen.SEED_BASE ^ 91)
    vals, _ = gpu.row_scale(rp, ci, v, 32)
    lo, up = gpu.factorize_split_cast(rp, ci, vals)
    F = gpu.IluFactors(lo, up)
    assert F.schedule_info(False)["tiles"] > 1
    il = oracle.ilu(lo, up)
    y = gen.uniform_int(14, len(rp) - 1, -(1 << 45), 1 << 45)
    want = oracle.apply_inverse(il, y)
    for _ in range(2):
        assert np.array_equal(gpu.apply_inverse(F, y), want)


@pytest.mark.parametrize("precond,g", [(False, 18), (True, 40)], ids=["plain", "ilu"])
def test_run_cycle_large_vs_oracle(gpu, oracle, precond, g):
    """A full cycle on grids whose rows do not divide evenly over the SMs
    (18^3 unpreconditioned, 40^3 with ILU; n % 4 == 0 selects the persistent
    path): the persistent Arnoldi-step
    kernel against the oracle, checked (trace totals) and unchecked, every
    basis word and Hessenberg entry; error behaviour must match too."""
    from workloads import gen
    from oracle.ffi import CheckerError
    from tests.cases import PRE, UNPRE
    rp, ci, v = gen.upwind_3d(g, 20.0)
    n = len(rp) - 1
    A = oracle.csrf(rp, ci, v)
    vals, scale = oracle.row_scale(A, 32)
    comp, alphas, _ = oracle.build_split(vals, 32, 1)
    sp = oracle.split(rp, ci, comp, alphas)
    S = gpu.SplitMatrix(rp, ci, comp, alphas)
    b = gen.uniform(78, n)
    plan = PRE if precond else UNPRE
    F = il = None
    if precond:
        lo, up = oracle.factorize_split_cast(oracle.csrf(rp, ci, vals))
        il = oracle.ilu(lo, up)
        F = gpu.IluFactors(lo, up)
    for checked in (False, True):
        t1, t2 = (gpu.FxTrace(), PyTrace()) if checked else (None, None)
        cfg = gpu.CycleConfig(m=12, frac_bits=30, shifts=gpu.ShiftPlan(*plan), s=0, precond=F)
        try:
            o = oracle.run_cycle(sp, 12, 30, 0, Shifts(*plan), b, np.zeros(n), precond=il, trace=t2)
        except CheckerError as e:
            with pytest.raises(ArithmeticError, match=re.escape(e.msg.split(":")[0])):
                gpu.run_cycle(S, cfg, b, np.zeros(n), t1)
            continue
        r = gpu.run_cycle(S, cfg, b, np.zeros(n), t1)
        assert r.dim == o["dim"] and r.dim > 3
        assert np.array_equal(r.basis, o["basis"])
        assert np.array_equal(r.hess, o["hess"]) and np.array_equal(r.g, o["g"])
        assert np.array_equal(r.x, o["x"])
        if checked:
            assert t1.total_overflows() == t2.total


def test_sharded_driver_cuda_backend(gpu, oracle):
    """dist.spmv_mgs_sharded through the CUDA slab backend (igm_spmv on the
    extended local CSR + igm_mgs_pass) == the oracle's reference sequence.
    Multi-rank partition / halo / allreduce logic: tests/test_dist.py (gloo)."""
    import torch
    import torch.distributed as tdist
    from paper_2009_07495_b200 import dist as D
    from workloads import gen
    g, k = 20, 6
    sl = D.make_slab(g, g * g, 0, 1)
    rp, ci, v, h0, own0, own1 = gen.upwind_3d_slab(g, 20.0, sl.z0, sl.z1)
    vals, _ = gpu.row_scale(rp, ci, v, 16)
    comp, al, _ = gpu.build_split(vals, 16, 2)
    dev = gpu.Device.default()
    be = D.CudaSlabBackend(gpu, dev)
    S = be.upload(rp, ci, comp, al)
    n = g ** 3
    rng = np.random.default_rng(9)
    vfull = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
    bfull = rng.integers(-(1 << 40), 1 << 40, (k, n), dtype=np.int64)
    work = dict(vext=torch.zeros(sl.next_, dtype=torch.int64, device="cuda"),
                wext=torch.zeros(sl.next_, dtype=torch.int64, device="cuda"),
                acc=torch.zeros(k, dtype=torch.int64, device="cuda"))
    w, acc = D.spmv_mgs_sharded(be, sl, S, 1, torch.from_numpy(vfull).cuda(), torch.from_numpy(bfull).cuda(), k,
                                30, 16, 0, 16, tdist, work)
    torch.cuda.synchronize()
    rpg, cig, vg = gen.upwind_3d(g, 20.0)
    valsg, _ = gpu.row_scale(rpg, cig, vg, 16)
    compg, alg, _ = oracle.build_split(valsg, 16, 2)
    sp = oracle.split(rpg, cig, compg, alg)
    wo = oracle.spmv(sp, 1, vfull)
    accs = acc.cpu().numpy()
    for i in range(k):
        h = oracle.fx_dot(wo, bfull[i], 30, 16, 0)
        assert h == D.fx_dot_finalize(int(accs[i]), 30, 16, 0)
        wo = oracle.fx_axpy_sub(wo, h, bfull[i], 30, 16)
    assert np.array_equal(w.cpu().numpy(), wo)


def test_cpp_dropin_solve(gpu, oracle, tmp_path):
    """A C++ program written against the reference's API (intgmres::solve,
    row_scale, build_split, factorize_ilu0 / split_cast; tests/cpp) and linked
    to libigm_b200.so: its x and report match the oracle bit for bit."""
    import subprocess
    from tests.test_capi import build_cpp_dropin
    from workloads import gen
    from tests.cases import PRE, UNPRE
    exe = build_cpp_dropin(tmp_path)
    out = subprocess.run([str(exe), "32"], check=True, capture_output=True, text=True, timeout=300).stdout
    got = {}
    for line in out.splitlines():
        tag, key, *vals = line.split()
        got.setdefault(tag, {})[key] = vals
    rp, ci, v = gen.upwind_2d(32)
    n = len(rp) - 1
    xs = (np.arange(n) % 7) * 0.25 - 0.75
    bh = gen.spmv_np(rp, ci, v, xs)
    for tag, alpha, plan, pre in (("plain", 16, UNPRE, False), ("ilu", 32, PRE, True)):
        A = oracle.csrf(rp, ci, v)
        vals, scale = oracle.row_scale(A, alpha)
        af = oracle.csrf(rp, ci, vals)
        comp, al, _ = oracle.build_split(vals, alpha, 1)
        sp = oracle.split(rp, ci, comp, al)
        il = None
        if pre:
            lo, up = oracle.factorize_split_cast(af)
            il = oracle.ilu(lo, up)
        x, rep = oracle.solve(sp, af, bh / scale, 1e-10, 60, 30, 30, 0, Shifts(*plan), checked=True, precond=il)
        g = got[tag]
        assert int(g["refinements"][0]) == rep["refinements"] and int(g["refinements"][2]) == rep["total_inner_iterations"]
        assert int(g["refinements"][4]) == rep["overflow_total"] and int(g["refinements"][6]) == int(rep["converged"])
        assert [float.fromhex(t) for t in g["relres"]] == rep["relres_history"]
        assert np.array_equal(np.array([float.fromhex(t) for t in g["x"]]), x)


def test_cpp_dropin_operator_cache(gpu, tmp_path):
    """The C++ drop-in's verified operator cache (shim.cpp): a repeated
    intgmres::solve on unchanged containers reuses the upload and returns the
    same bits; operators overwritten IN PLACE (same addresses and sizes) are
    detected by the content fingerprint, which is checked on host threads
    while the GPU already solves on the cached copy, and the solve is repeated
    on a fresh upload -- its result equals the one from separate containers."""
    import subprocess
    from tests.test_capi import build_cpp_dropin
    exe = build_cpp_dropin(tmp_path)
    out = subprocess.run([str(exe), "24", "cache"], check=True, capture_output=True, text=True, timeout=300).stdout
    line = [ln for ln in out.splitlines() if ln.startswith("cache ")]
    assert line, out
    assert line[0].split() == ["cache", "repeat_same", "1", "inplace", "1", "mutated_detected", "1",
                               "differs_from_first", "1"], out


@pytest.mark.parametrize("name", ["cfg1", "cfg2_16"])
def test_fp64_engine_vs_reference(gpu, oracle, reference, name):
    """Engine::floating_point (refsolve.cpp via refine.cpp:74-82) on the
    device vs the reference library's own FP engine.  The SpMV, ILU, norms,
    scalings and x updates follow the reference's order bit for bit; the MGS
    dots are tree reductions, so the comparison is by convergence and
    iteration counts and by x to solver accuracy."""
    c = product_case(gpu, oracle, name)
    rc = build_case(name, reference)
    cfg = gpu.RefineConfig(tol=c["tol"], max_refinements=c["max_ref"], m=c["m"], frac_bits=30, shifts=c["plan"],
                           s=c["s"], checked=True, engine=1)
    x, rep = gpu.solve(c["S"], c["A"], c["b"], cfg, precond=c.get("F"))
    xr, rr = reference.solve(rc["sp"], rc["af"], rc["b"], c["tol"], c["max_ref"], c["m"], 30, c["s"],
                             Shifts(*c["shifts"]), checked=True, precond=rc.get("il"), engine=1)
    assert rep.converged and rr["converged"]
    assert abs(rep.refinements - rr["refinements"]) <= 1
    assert abs(rep.total_inner_iterations - rr["total_inner_iterations"]) <= max(2, rr["total_inner_iterations"] // 10)
    assert rep.relres_history[0] == rr["relres_history"][0]  # same residual kernel, same x = 0
    assert np.linalg.norm(x - xr) <= 1e-6 * np.linalg.norm(xr)
    assert rep.overflow_total == 0


def test_cpp_refsolve(gpu, reference, tmp_path):
    """fp_cycle / solve_fp of the drop-in API (device FP64 GMRES) against the
    reference library's own: Krylov dimensions, r0 norm (bit-exact: same
    residual, preconditioner and norm order), restarts within one and x to
    solver accuracy (the MGS dots are tree reductions)."""
    import ctypes as C
    import subprocess
    from pathlib import Path
    from workloads import gen
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2009_07495_b200"
    exe = tmp_path / "refsolve_run"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{root / 'include'}", str(root / "tests/cpp/refsolve_run.cpp"),
                    f"-L{lib}", "-ligm_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True,
                   capture_output=True, text=True)
    out = subprocess.run([str(exe), "24"], check=True, capture_output=True, text=True, timeout=300).stdout
    got = {}
    for line in out.splitlines():
        tok = line.split()
        d = {}
        k = 1
        while k < len(tok):
            if tok[k] == "x":
                d["x"] = np.array([float.fromhex(v) for v in tok[k + 1:]])
                break
            d[tok[k]] = tok[k + 1]
            k += 2
        got[tok[0]] = d
    rp, ci, v = gen.upwind_2d(24)
    n = len(rp) - 1
    A = reference.csrf(rp, ci, v)
    xs = (np.arange(n) % 7) * 0.25 - 0.75
    b = gen.spmv_np(rp, ci, v, xs)
    x0 = (np.arange(n) % 5) * 0.125
    lib_r = reference.lib
    p = lambda a_: a_.ctypes.data_as(C.c_void_p)
    for pre in (0, 1):
        xr = np.zeros(n); dim = C.c_int(); r0 = C.c_double(); gab = np.zeros(20)
        assert lib_r.ref_fp_cycle(C.byref(A), 20, p(b), p(x0), pre, p(xr), C.byref(dim), C.byref(r0), p(gab)) == 0
        gc = got[f"cycle{pre}"]
        assert int(gc["dim"]) == dim.value
        assert float.fromhex(gc["r0"]) == r0.value
        assert np.linalg.norm(gc["x"] - xr) <= 1e-9 * np.linalg.norm(xr)
        xs_ = np.zeros(n); rs = C.c_int(); it = C.c_long(); cv = C.c_int()
        assert lib_r.ref_solve_fp(C.byref(A), p(b), 20, C.c_double(1e-10), 100000, pre, p(xs_), C.byref(rs),
                                  C.byref(it), C.byref(cv)) == 0
        gs = got[f"solve{pre}"]
        assert int(gs["conv"]) == 1 and cv.value == 1
        assert abs(int(gs["restarts"]) - rs.value) <= 1
        assert np.linalg.norm(gs["x"] - xs_) <= 1e-7 * np.linalg.norm(xs_)


def test_cpp_experiment(gpu, reference, tmp_path):
    """run_experiment of the drop-in API (Matrix Market in, CSV history and
    summary out) vs the reference library's run_experiment on the same file:
    byte-identical CSV and summary for the integer solver (bit-exact solve),
    the same restarts (within one) for the FP64 comparator."""
    import ctypes as C
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2009_07495_b200"
    exe = tmp_path / "experiment_run"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{root / 'include'}", str(root / "tests/cpp/experiment_run.cpp"),
                    f"-L{lib}", "-ligm_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True,
                   capture_output=True, text=True)
    mtx = tmp_path / "upwind24.mtx"
    out = subprocess.run([str(exe), str(mtx), "24"], check=True, capture_output=True, text=True, timeout=300).stdout
    blocks = {}
    for part in out.split("### ")[1:]:
        head, body = part.split("\n", 1)
        blocks[tuple(int(t) for t in head.split())] = body.rstrip("\n")
    for (solver, pre), body in blocks.items():
        csv = C.create_string_buffer(1 << 16)
        summ = C.create_string_buffer(1024)
        assert reference.lib.ref_run_experiment(str(mtx).encode(), solver, pre, 20, C.c_double(1e-10), 60, csv,
                                                len(csv), summ, len(summ)) == 0
        ref_text = csv.value.decode() + summ.value.decode()
        if solver == 0:
            assert body == ref_text
        else:
            ours = body.splitlines()
            refl = ref_text.splitlines()
            assert abs(len(ours) - len(refl)) <= 1 and ours[-1].split()[:4] == refl[-1].split()[:4]
            assert ours[-1].endswith("converged=yes") and refl[-1].endswith("converged=yes")


@pytest.mark.parametrize("kind,g,world,local", [("27pt_ilu", 12, 1, False), ("27pt_ilu", 12, 3, False),
                                                ("7pt_plain", 10, 2, False), ("7pt_ilu", 16, 2, False),
                                                ("27pt_ilu", 12, 3, True), ("7pt_ilu", 16, 2, True)])
def test_sharded_solve_cuda_backend(gpu, oracle, kind, g, world, local):
    """dist.solve_sharded through the product kernels (igm_dc_* entries: rank
    local SpMV / MGS passes / replicated scalar step / vec_div / pipelined
    global ILU / relayed norm2 / residual) on `world` ranks sharing this GPU
    as threads with their own contexts and streams (exchanges are host copies:
    no kernel waits on another rank) == the single-process oracle solve, bit
    for bit.  Multi-process gloo runs of the same driver: tests/test_dist.py.
    local: the ranks' inputs come from dist.setup_slab_local (own planes
    only; device row_scale / build_split, the ILU(0) plane relay through
    igm_factorize_split_cast_dev_lu)."""
    import torch
    from tests.test_dist import run_sharded_threads, check_sharded_vs_oracle
    from paper_2009_07495_b200 import dist as D
    devs = {}

    def make_backend(rank):
        devs[rank] = gpu.Device(0)
        return D.CudaSlabBackend(gpu, devs[rank])

    m, s = 10, (0 if kind.endswith("_ilu") else 1)
    x, reps, prob = run_sharded_threads(oracle, make_backend, kind, g, m, s, world, to_dev=lambda t: t.cuda(),
                                        local=local)
    check_sharded_vs_oracle(oracle, x, reps, prob, m, s)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_16", "cfg4_12", "cfg3_small", "split_s3", "ilu_random"])
def test_device_setup_bit_exact(gpu, oracle, name):
    """Device-side setup (igm_row_scale_dev / igm_build_split_dev /
    igm_factorize_split_cast_dev) == the oracle's
    restatement of row_scale, build_split and split_cast(factorize_ilu0),
    array for array (host numpy and device tensor arguments)."""
    import torch
    from tests.cases import CASES, build_case
    c = build_case(name, oracle)
    rp, ci, v = c["rp"], c["ci"], c["v"]
    vals, scale = gpu.row_scale_device(rp, ci, v, c["alpha"])
    assert np.array_equal(vals, c["vals"]) and np.array_equal(scale, c["scale"])
    comp, al, ex = gpu.build_split_device(vals, c["alpha"], CASES[name]["ncomp"])
    assert al == list(c["alphas"]) and np.array_equal(comp, np.atleast_2d(c["comp"]))
    co, alo, exo = oracle.build_split(vals, c["alpha"], CASES[name]["ncomp"])
    assert ex == exo
    # device-resident arguments (torch CUDA tensors in, out)
    td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    vd, sd = gpu.row_scale_device(td(rp.astype(np.int32)), td(ci.astype(np.int32)), td(v), c["alpha"])
    assert np.array_equal(vd.cpu().numpy(), c["vals"]) and np.array_equal(sd.cpu().numpy(), c["scale"])
    if c.get("ilu"):
        lo, up = gpu.factorize_split_cast_device(rp, ci, vals)
        for a, b in zip(lo + up, list(c["lower"]) + list(c["upper"])):
            assert np.array_equal(np.asarray(a), np.asarray(b))
        lod, upd = gpu.factorize_split_cast_device(td(rp.astype(np.int32)), td(ci.astype(np.int32)), td(vals))
        for a, b in zip(lod + upd, list(c["lower"]) + list(c["upper"])):
            assert np.array_equal(a.cpu().numpy(), np.asarray(b))


def test_device_setup_errors(gpu):
    """The reference's setup exceptions (type and text, first offending row)."""
    rp = np.array([0, 1, 1, 2], np.int32)  # row 1 empty
    with pytest.raises(RuntimeError, match=r"row_scale: row 1 has no nonzero entry"):
        gpu.row_scale_device(rp, np.array([0, 2], np.int32), np.array([1.0, 2.0]), 16)
    with pytest.raises(ValueError, match="build_split: need at least one component"):
        gpu.build_split_device(np.array([1.0]), 16, 0)
    # row 2 has no diagonal in its pattern
    rp = np.array([0, 1, 2, 3], np.int32)
    with pytest.raises(RuntimeError, match=r"factorize_ilu0: row 2 has no diagonal entry in the pattern"):
        gpu.factorize_split_cast_device(rp, np.array([0, 1, 0], np.int32), np.array([2.0, 2.0, 1.0]))
    # zero pivot in row 1 (a_11 - a_10 a_01 / a_00 = 1 - 1 = 0)
    rp = np.array([0, 2, 4], np.int32)
    with pytest.raises(RuntimeError, match=r"factorize_ilu0: zero pivot in row 1"):
        gpu.factorize_split_cast_device(rp, np.array([0, 1, 0, 1], np.int32), np.array([1.0, 1.0, 1.0, 1.0]))
    # sqrt|d| truncates to zero
    rp = np.array([0, 1, 2], np.int32)
    with pytest.raises(RuntimeError, match=r"split_cast: diagonal entry of row 0 truncates to zero"):
        gpu.factorize_split_cast_device(rp, np.array([0, 1], np.int32), np.array([0.5, 4.0]))


def test_exact_overflow_counts(gpu, oracle):
    """Exact running-sum overflow events: with
    igm_set_exact_overflow_counts on, fx_dot / fx_norm reductions whose sums
    wrap up and down many times (and whose products wrap too) report the
    reference's sequential event count, and the trace stays exact."""
    from oracle.ffi import CheckerError
    dev = gpu.Device.default()
    dev.set_exact_overflow_counts(True)
    try:
        rng = np.random.default_rng(3)
        n = 50_000
        mag = rng.integers(1 << 61, 1 << 62, n, dtype=np.int64)
        v = np.where(rng.random(n) < 0.55, mag, -mag).astype(np.int64)
        for w in (np.ones(n, np.int64), rng.integers(-5, 6, n, dtype=np.int64)):
            t, to = gpu.FxTrace(checked=True), PyTrace()
            assert gpu.fx_dot(v, w, 30, 0, 0, t) == oracle.fx_dot(v, w, 30, 0, 0, to)
            assert t.exact and t.total_overflows() == to.total > 100
        for seed in range(4):
            r2 = np.random.default_rng(10 + seed)
            vn = r2.integers(-(1 << 33), 1 << 33, 20_000 + seed, dtype=np.int64)
            t, to = gpu.FxTrace(checked=True), PyTrace()
            try:
                ro = oracle.fx_norm(vn, 31, 0, to)
            except CheckerError:
                ro = None
            if ro is None:
                with pytest.raises(ArithmeticError):
                    gpu.fx_norm(vn, 31, 0, t)
            else:
                assert gpu.fx_norm(vn, 31, 0, t) == ro
            assert t.exact and t.total_overflows() == to.total > 100
        # a whole solve whose dot products wrap (test_refine.cpp:392-426 setup)
        from workloads import gen
        rp, ci, vv = gen.laplacian2d(8)
        vals, scale = gpu.row_scale(rp, ci, vv, 16)
        comp, al, _ = gpu.build_split(vals, 16, 10)
        S, A = gpu.SplitMatrix(rp, ci, comp, al), gpu.CsrMatrixF(rp, ci, vals)
        b = np.ones(len(rp) - 1) / scale
        plan = gpu.ShiftPlan(0, 0, 16, 16, 16, 14, 16, 0)
        t, to = gpu.FxTrace(checked=True), PyTrace()
        try:
            gpu.solve(S, A, b, gpu.RefineConfig(tol=1e-8, max_refinements=3, m=6, shifts=plan, s=len(al) - 1),
                      trace=t)
            threw = False
        except (ArithmeticError, ValueError, OverflowError, RuntimeError):
            threw = True
        try:
            oracle.solve(oracle.split(rp, ci, comp, al), oracle.csrf(rp, ci, vals), b, 1e-8, 3, 6, 30, len(al) - 1,
                         Shifts(0, 0, 16, 16, 16, 14, 16, 0), trace=to)
            othrew = False
        except CheckerError:
            othrew = True
        assert threw == othrew
        assert t.exact and t.total_overflows() == to.total > 0
    finally:
        dev.set_exact_overflow_counts(False)


_PENCIL_SHAPES = [(12, 12, 12), (17, 35, 9), (16, 16, 40), (33, 9, 20), (5, 70, 3), (2, 2, 50), (64, 64, 1)]


@pytest.mark.parametrize("dims", _PENCIL_SHAPES, ids=["x".join(map(str, d)) for d in _PENCIL_SHAPES])
def test_ilu_pencil_wavefront(gpu, oracle, dims):
    """The structured 7-point pencil wavefront (csrc/tri_pencil.cuh) on ragged
    grids (partial bricks in x and y, short and single-plane z): bit-exact vs
    the oracle's sequential substitution (ilu.cpp:122-155), integer with and
    without wrapping, checked-mode event totals, repeated launches, and equal
    to the generic wavefront on the same factors."""
    offs = _SEVEN if dims[2] > 1 else [o for o in _SEVEN if o[2] == 0]
    lo, up = _grid_factors(gpu, dims, offs, seed=7 + sum(dims))
    F = gpu.IluFactors(lo, up)
    assert F.pencil_bricks(False) > 0 and F.pencil_bricks(True) > 0
    il = oracle.ilu(lo, up)
    n = len(lo[0]) - 1
    from workloads import gen
    for seed, mag in ((21, 45), (22, 62)):
        y = gen.uniform_int(seed, n, -(1 << mag), 1 << mag)
        t1, t2 = gpu.FxTrace(), PyTrace()
        want = oracle.apply_inverse(il, y, t2)
        for _ in range(2):
            assert np.array_equal(gpu.apply_inverse(F, y), want)
        assert np.array_equal(gpu.apply_inverse(F, y, t1), want)
        assert t1.total_overflows() == t2.total
    # FP64 substitution on the integer factors (apply_inverse_fp), with -0.0
    # and tiny right-hand sides: absent stencil entries must not be applied
    yf = gen.uniform(24, n)
    yf[::7] = -0.0
    yf[3::11] = 5e-324
    assert np.array_equal(gpu.apply_inverse_fp(F, yf).view(np.int64), oracle.apply_inverse_fp(il, yf).view(np.int64))
    os.environ["IGM_PENCIL"] = "0"
    try:
        G = gpu.IluFactors(lo, up)
    finally:
        del os.environ["IGM_PENCIL"]
    assert G.pencil_bricks(False) == 0
    y = gen.uniform_int(23, n, -(1 << 50), 1 << 50)
    assert np.array_equal(gpu.apply_inverse(G, y), gpu.apply_inverse(F, y))


_CERT_SCRIPT = r"""
import sys, json
import numpy as np
import paper_2009_07495_b200 as gpu
from workloads import gen
plan = tuple(json.loads(sys.argv[1]))
rp, ci, v = gen.laplacian2d(64)
n = len(rp) - 1
vals, scale = gpu.row_scale(rp, ci, v, 16)
comp, al, _ = gpu.build_split(vals, 16, 1)
S = gpu.SplitMatrix(rp, ci, comp, al)
b = gen.uniform(31, n) / scale
t = gpu.FxTrace(checked=True)
try:
    r = gpu.run_cycle(S, gpu.CycleConfig(m=8, shifts=gpu.ShiftPlan(*plan)), b, np.zeros(n), trace=t)
    st = [int(r.dim), int(np.bitwise_xor.reduce(r.basis.view(np.uint64))), int(np.bitwise_xor.reduce(r.hess.view(np.uint64)))]
except Exception as e:
    st = type(e).__name__
print(json.dumps({"state": st, "total": t.total_overflows(), "exact": t.exact, "events": sorted(map(list, t.events))}))
"""


@pytest.mark.parametrize("plan", [(16, 0, 16, 16, 16, 14, 16, 0), (0, 0, 16, 16, 16, 14, 16, 0), (0, 0, 0, 0, 0, 30, 0, 0)],
                         ids=["guarded", "dot-guard-removed", "no-shifts"])
def test_arnoldi_overflow_certificate(gpu, plan):
    """The persistent Arnoldi step skips per-element product / subtraction
    overflow tests for a pass only when the CTA's magnitude bounds prove none
    can occur (kernels.cu k_arnoldi certify).  On n = 4096 (the fused path),
    with plans that do and do not wrap, its checked-mode trace (events,
    total, exactness) and cycle state equal those of the separate pass
    kernels, which test every element (IGM_ARNOLDI=0)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"IGM_ARNOLDI": "0"}):
        r = subprocess.run([sys.executable, "-c", _CERT_SCRIPT, json.dumps(plan)], cwd=root, capture_output=True,
                           text=True, env={**os.environ, **env}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
    if plan[:2] == (0, 0) and plan[2] == 16:  # the wrapping plan: events on both paths
        assert outs[0]["total"] > 0


_SPMV_CERT_SCRIPT = r"""
import sys, json
import numpy as np
import paper_2009_07495_b200 as gpu
from workloads import gen
alpha, f = int(sys.argv[1]), int(sys.argv[2])
rp, ci, v = gen.upwind_3d(16, 20.0)
n = len(rp) - 1
vals, scale = gpu.row_scale(rp, ci, v, alpha)
comp, al, _ = gpu.build_split(vals, alpha, 1)
S = gpu.SplitMatrix(rp, ci, comp, al)
b = gen.uniform(31, n) / scale
t = gpu.FxTrace(checked=True)
try:
    r = gpu.run_cycle(S, gpu.CycleConfig(m=6, frac_bits=f, shifts=gpu.ShiftPlan(16, 0, 16, 16, 16, 14, 16, 0)), b,
                      np.zeros(n), trace=t)
    st = [int(r.dim), int(np.bitwise_xor.reduce(r.basis.view(np.uint64))), int(np.bitwise_xor.reduce(r.hess.view(np.uint64)))]
except Exception as e:
    st = type(e).__name__
ev = sorted(map(list, t.events))
print(json.dumps({"state": st, "total": t.total_overflows(), "exact": t.exact, "events": ev,
                  "spmv_events": sum(1 for e in ev if e[0] == "spmv")}))
"""


@pytest.mark.parametrize("alpha,f,wraps", [(16, 30, False), (40, 44, True)], ids=["configured", "products-wrap"])
def test_spmv_magnitude_certificate(gpu, alpha, f, wraps):
    """k_spmv_int_r8 (7-point rows, the persistent cycle of n = 4096) skips its
    per-product overflow tests only under the magnitude certificate
    8 * max|a| * max|v_j| < 2^63 (max|v_j| recorded by the Arnoldi kernel).
    Its checked-mode trace and cycle state equal those of the generic
    one-thread-per-row kernel that tests every product (IGM_SPMV_R8=0) and of
    the separate pass kernels, which pass no bound (IGM_ARNOLDI=0) -- on a
    configured run (no events) and with alpha_a = 40, Q19.44, where the
    products of split.cpp:137-157 wrap and the certificate must fail."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"IGM_SPMV_R8": "0"}, {"IGM_ARNOLDI": "0"}):
        r = subprocess.run([sys.executable, "-c", _SPMV_CERT_SCRIPT, str(alpha), str(f)], cwd=root,
                           capture_output=True, text=True, env={**os.environ, **env}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1] == outs[2]
    if wraps:
        assert outs[0]["spmv_events"] > 0 or outs[0]["total"] > 1024
    else:
        assert outs[0]["total"] == 0


_P27_SHAPES = [(12, 12, 12), (17, 35, 9), (33, 20, 7), (2, 2, 30), (40, 3, 5)]


@pytest.mark.parametrize("dims", _P27_SHAPES, ids=["x".join(map(str, d)) for d in _P27_SHAPES])
def test_ilu_pencil27_wavefront(gpu, oracle, dims):
    """The 27-point pencil wavefront (csrc/pencil27.cuh) on ragged grids:
    integer substitutions bit-exact vs the oracle's sequential ones
    (ilu.cpp:122-155), with and without wrapping, checked-mode event totals,
    repeated launches, and equal to the generic wavefront."""
    lo, up = _grid_factors(gpu, dims, _TWENTY7, seed=11 + sum(dims))
    F = gpu.IluFactors(lo, up)
    assert F.pencil_bricks(False) > 0 and F.pencil_bricks(True) > 0
    il = oracle.ilu(lo, up)
    n = len(lo[0]) - 1
    from workloads import gen
    for seed, mag in ((31, 45), (32, 62)):
        y = gen.uniform_int(seed, n, -(1 << mag), 1 << mag)
        t1, t2 = gpu.FxTrace(), PyTrace()
        want = oracle.apply_inverse(il, y, t2)
        for _ in range(2):
            assert np.array_equal(gpu.apply_inverse(F, y), want)
        assert np.array_equal(gpu.apply_inverse(F, y, t1), want)
        assert t1.total_overflows() == t2.total
    yf = gen.uniform(34, n)
    yf[::5] = -0.0
    assert np.array_equal(gpu.apply_inverse_fp(F, yf).view(np.int64), oracle.apply_inverse_fp(il, yf).view(np.int64))
    os.environ["IGM_PENCIL"] = "0"
    try:
        G = gpu.IluFactors(lo, up)
    finally:
        del os.environ["IGM_PENCIL"]
    assert G.pencil_bricks(False) == 0
    y = gen.uniform_int(33, n, -(1 << 50), 1 << 50)
    assert np.array_equal(gpu.apply_inverse(G, y), gpu.apply_inverse(F, y))


@pytest.mark.parametrize("kind,g,world", [("7pt", 16, 2), ("7pt", 24, 3), ("7pt", 40, 4), ("27pt", 12, 2),
                                          ("27pt", 20, 3), ("27pt", 33, 4)])
def test_piped_substitution_protocol(gpu, oracle, kind, g, world):
    """igm_dc_tri_piped, the word protocol of the pipelined slab
    substitutions (dist.ZPipe): rank r's forward wavefront stores its last
    own plane as tagged words into rank r+1's import buffer and rank r+1's
    wavefront reads its halo plane from there; backward the same from r+1 to
    r; both pencil wavefronts (7-point k_tri_pencil2, 27-point k_tri27:
    BASELINE config 4's factors).  Here the ranks share this GPU, so they run strictly one after the
    other (each launch completes before the next rank's starts: no kernel ever
    waits on another); the buffers are plain device pointers instead of IPC
    mappings.  Concatenated own rows == the global substitution pair of the
    oracle (ilu.cpp:122-180), bit for bit, over two calls (epochs 1, 2) with
    different right-hand sides -- a stale word of call 1 must not satisfy
    call 2."""
    import ctypes as C
    import torch
    from paper_2009_07495_b200 import dist as D
    from workloads import gen
    rp, ci, v = gen.upwind_3d(g, 20.0) if kind == "7pt" else gen.stencil27(g, 5)
    n = len(rp) - 1
    vals, _ = oracle.row_scale(oracle.csrf(rp, ci, v), 32)
    lower, upper = oracle.factorize_split_cast(oracle.csrf(rp, ci, vals))
    eye = (np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.ones(n, np.int64),
           np.arange(n, dtype=np.int32))
    fwd, bwd = oracle.ilu(lower, eye), oracle.ilu(eye, upper)
    ranks = []
    for r in range(world):
        sl = D.make_slab(g, g * g, r, world)
        be = D.CudaSlabBackend(gpu, gpu.Device(0))
        fac = be.upload_factors(D.slab_factor(lower, sl), D.slab_factor(upper, sl))
        assert be.pipe_capable(fac, sl), fac.schedule_info()
        st = be.state(1)
        with be.stream():
            be.reset(st)
        ranks.append(dict(sl=sl, be=be, fac=fac, st=st, kf=D.ZPipe.planes(sl),
                          imp_f=be.pipe_alloc(sl.plane) if r > 0 else None,
                          imp_b=be.pipe_alloc(sl.plane) if r < world - 1 else None))
    rng = np.random.default_rng(7)
    try:
        for epoch in (1, 2):
            y = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
            want = oracle.apply_inverse(bwd, oracle.apply_inverse(fwd, y))
            for R in ranks:
                sl = R["sl"]
                g0, g1 = sl.global_rows
                R["y"] = torch.zeros(sl.next_, dtype=torch.int64, device="cuda")
                R["y"][sl.own0:sl.own1] = torch.from_numpy(y[g0:g1]).cuda()
                R["mid"] = torch.full((sl.next_,), 7, dtype=torch.int64, device="cuda")
                R["out"] = torch.full((sl.next_,), 7, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            for r in range(world):  # forward: rank order
                R = ranks[r]
                nxt = ranks[r + 1]["imp_f"] if r < world - 1 else None
                R["be"].tri_piped(R["st"], R["fac"], False, R["y"], R["mid"], 0, True, R["imp_f"], nxt,
                                  R["kf"][0], epoch << 32)
                R["be"].sync()
            for r in reversed(range(world)):  # backward: reverse rank order
                R = ranks[r]
                prv = ranks[r - 1]["imp_b"] if r > 0 else None
                R["be"].tri_piped(R["st"], R["fac"], True, R["mid"], R["out"], 0, True, R["imp_b"], prv,
                                  R["kf"][1], epoch << 32)
                R["be"].sync()
            got = np.concatenate([R["out"][R["sl"].own0:R["sl"].own1].cpu().numpy() for R in ranks])
            assert np.array_equal(got, want), epoch
            for R in ranks:
                R["be"].fetch(R["st"])  # raises on a device error
                assert int(R["st"].view("lcnt", 0).sum()) == 0  # checked mode: no overflow event
    finally:
        for R in ranks:
            for k in ("imp_f", "imp_b"):
                if R[k] is not None:
                    gpu.lib().igm_dev_free(C.c_void_p(R[k]))


@pytest.mark.parametrize("world,nwords", [(2, 3), (3, 40), (8, 3), (5, 1200)])
def test_mailbox_allreduce_protocol(gpu, world, nwords):
    """igm_mbox_*: the one-shot P2P mailbox reduction of the partitioned
    solve's per-pass accumulators (fx_dot / fx_norm wrapping sums,
    fxp.cpp:49-86).  The ranks share this GPU (mailboxes
    connected as same-process peers), so each reduction is run as its two
    halves -- every rank publishes, then every rank collects -- and no kernel
    ever waits on another.  Result on every rank == the wrapping u64 sum /
    the signed int64 max over ranks, over several sequence numbers (a stale
    word of reduction k-2 in the same parity slot must not satisfy k) and
    through the chunked igm_mbox_allreduce of a single-rank world."""
    import ctypes as C
    import torch
    L = gpu.lib()
    devs = [gpu.Device(0) for _ in range(world)]
    max_words = 512
    boxes = []
    for r in range(world):
        mb = C.c_void_p()
        gpu._check(L.igm_mbox_create(devs[r].h, r, world, max_words, C.byref(mb)))
        boxes.append(mb)
    try:
        arr = (C.c_void_p * world)(*[b.value for b in boxes])
        for r in range(world):
            gpu._check(L.igm_mbox_connect_local(boxes[r], arr))
        rng = np.random.default_rng(world * 1000 + nwords)
        for it in range(5):
            op = it % 2  # SUM, MAX, SUM, ...
            host = rng.integers(-(1 << 63), (1 << 63) - 1, (world, nwords), dtype=np.int64, endpoint=True)
            if it == 3:
                host[:] = host[0]  # equal words from every rank (torn-word check must still pass)
            want = host.view(np.uint64).sum(axis=0, dtype=np.uint64).view(np.int64) if op == 0 else host.max(axis=0)
            t = [torch.from_numpy(host[r].copy()).cuda() for r in range(world)]
            torch.cuda.synchronize()
            for o in range(0, nwords, max_words):  # the chunks igm_mbox_allreduce would issue
                k = min(max_words, nwords - o)
                for r in range(world):
                    gpu._check(L.igm_mbox_publish(devs[r].h, boxes[r], C.c_void_p(t[r][o:].data_ptr()), k))
                for r in range(world):
                    devs[r].synchronize()
                for r in range(world):
                    gpu._check(L.igm_mbox_collect(devs[r].h, boxes[r], C.c_void_p(t[r][o:].data_ptr()), k, op))
            for r in range(world):
                gpu._check(L.igm_mbox_status(devs[r].h, boxes[r]))
                assert np.array_equal(t[r].cpu().numpy(), want), (it, r)
        # a world of one: allreduce is the identity, any n
        one = C.c_void_p()
        gpu._check(L.igm_mbox_create(devs[0].h, 0, 1, 4, C.byref(one)))
        x = torch.arange(10, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        gpu._check(L.igm_mbox_allreduce(devs[0].h, one, C.c_void_p(x.data_ptr()), 10, 0))
        gpu._check(L.igm_mbox_status(devs[0].h, one))
        assert x.cpu().tolist() == list(range(10))
        L.igm_mbox_free(one)
        # argument errors
        assert L.igm_mbox_publish(devs[0].h, boxes[0], C.c_void_p(t[0].data_ptr()), max_words + 1) == 1
        assert L.igm_mbox_collect(devs[0].h, boxes[0], C.c_void_p(t[0].data_ptr()), 1, 7) == 1
    finally:
        for b in boxes:
            L.igm_mbox_free(b)


def test_mailbox_timeout_reports(gpu, monkeypatch):
    """a collect whose peer never publishes gives up and igm_mbox_status
    reports IGM_CUDA_ERROR instead of hanging the stream"""
    import ctypes as C
    import torch
    monkeypatch.setenv("IGM_MBOX_TIMEOUT_MS", "50")
    L = gpu.lib()
    devs = [gpu.Device(0) for _ in range(2)]
    boxes = []
    for r in range(2):
        mb = C.c_void_p()
        gpu._check(L.igm_mbox_create(devs[r].h, r, 2, 8, C.byref(mb)))
        boxes.append(mb)
    try:
        arr = (C.c_void_p * 2)(*[b.value for b in boxes])
        for r in range(2):
            gpu._check(L.igm_mbox_connect_local(boxes[r], arr))
        t = torch.ones(3, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        gpu._check(L.igm_mbox_publish(devs[0].h, boxes[0], C.c_void_p(t.data_ptr()), 3))
        gpu._check(L.igm_mbox_collect(devs[0].h, boxes[0], C.c_void_p(t.data_ptr()), 3, 0))  # rank 1 silent
        assert L.igm_mbox_status(devs[0].h, boxes[0]) == 6  # IGM_CUDA_ERROR
        assert b"timed out" in L.igm_last_error()
    finally:
        for b in boxes:
            L.igm_mbox_free(b)


def test_fx_device_fast_paths(gpu):
    """The device fast paths of the scalar helpers (fx_core.cuh: FP64
    estimate + exact 128-bit remainder fix-ups) against exact integer
    arithmetic: floor sqrt (fxp.cpp:20-33), the round-up division magic,
    truncating int64 division (fxp.hpp:145-152), and 128/64 floor division --
    on edge values (0, 1, squares +-1, powers of two +-1, 2^63, 2^64 - 1) and
    random words of every magnitude."""
    import ctypes as C
    import math
    M = (1 << 64) - 1
    edge = {0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, (1 << 63) - 1, 1 << 63,
            (1 << 63) + 1, M, M - 1, ((1 << 32) - 1) ** 2, ((1 << 32) - 1) ** 2 - 1, ((1 << 32) - 1) ** 2 + 1}
    for k in range(1, 64):
        edge |= {(1 << k) - 1, 1 << k, ((1 << k) + 1) & M}
    for r in (3, 1000, 65535, 65536, 94906265, 94906266, 3037000499, 3037000500, 4294967295):
        edge |= {r * r - 1, r * r, r * r + 1}
    edge = sorted(e & M for e in edge)
    rng = np.random.default_rng(11)
    rand = [int(x) >> int(s) for x, s in zip(rng.integers(0, 1 << 63, 4000, dtype=np.uint64).astype(object) * 2 +
                                             rng.integers(0, 2, 4000).astype(object),
                                             rng.integers(0, 64, 4000))]
    a = [x for x in edge for _ in range(3)] + rand + rand[::-1]
    b = [edge[(i * 7 + 3) % len(edge)] for i in range(len(edge) * 3)] + rand[::-1] + [max(1, x >> 40) for x in rand]
    n = len(a)
    A = np.array(a, dtype=np.uint64)
    B = np.array(b, dtype=np.uint64)
    out = np.zeros(4 * n, dtype=np.uint64)
    assert gpu.lib().igm_debug_fx_selftest(n, A.ctypes.data_as(C.c_void_p), B.ctypes.data_as(C.c_void_p),
                                           out.ctypes.data_as(C.c_void_p)) == 0
    out = out.reshape(n, 4)
    sgn = lambda v: v - (1 << 64) if v >= 1 << 63 else v
    for i in range(n):
        x, y = a[i], b[i] if b[i] else 1
        want_sqrt = math.isqrt(x)
        l = 0 if y == 1 else (y - 1).bit_length()
        want_m = ((((1 << l) - y) << 64) // y + 1) & M
        sx, sy = sgn(x), sgn(y)
        if sx == -(1 << 63) and sy == -1:
            want_q = 0
        else:
            q = abs(sx) // abs(sy)
            want_q = (-q if (sx < 0) != (sy < 0) else q) & M
        want_u = ((((x % y) << 64) | ((~x ^ y) & M)) // y) & M
        got = [int(v) for v in out[i]]
        assert got == [want_sqrt, want_m, want_q, want_u], (x, y, got, [want_sqrt, want_m, want_q, want_u])


# (grid kind, size, row-scale alpha, split depth, plan, ILU): plans that wrap
# (found with the restatement; event totals per kernel in the comments)
_ORDER_CASES = {
    "dot-guard-removed": ("lap", 8, 16, 10, (0, 0, 16, 16, 16, 14, 16, 0), False),  # dot mul/add
    "ilu-spmv-precond": ("up", 12, 36, 1, (0, 0, 0, 0, 28, 0, 0, 0), True),  # spmv mul/add, precond sub
    "ilu-capped": ("up", 12, 40, 1, (4, 4, 0, 0, 20, 0, 8, 0), True),  # > 1024 events: the list is capped
    "mgs-vecdiv-error": ("lap", 8, 33, 1, (4, 4, 0, 0, 20, 0, 8, 0), False),  # dot/axpy/norm/vec_div/givens/rot,
}                                                                             # then a domain_error


def _order_case(gpu, oracle, name):
    from workloads import gen
    kind, g, alpha, depth, plan, ilu = _ORDER_CASES[name]
    rp, ci, v = gen.upwind_2d(g) if kind == "up" else gen.laplacian2d(g)
    n = len(rp) - 1
    f = 30
    vals, scale = gpu.row_scale(rp, ci, v, alpha)
    comp, al, _ = gpu.build_split(vals, alpha, depth)
    pre = opre = None
    if ilu:
        lo, up = gpu.factorize_split_cast(rp, ci, vals)
        pre, opre = gpu.IluFactors(lo, up), oracle.ilu(lo, up)
    b = gen.uniform(31, n) / scale
    return rp, ci, vals, comp, al, plan, pre, opre, b, f


@pytest.mark.parametrize("name", list(_ORDER_CASES))
def test_overflow_event_order(gpu, oracle, name):
    """FxTrace::events in the reference's sequential order (fxp.hpp:51-103,
    refine.cpp:100): plans that wrap products and running sums in spmv,
    the ILU substitutions, the MGS dots / axpys, the norm, vec_div and the
    scalar Givens work; the device counts are grouped per (step, kernel, op),
    the list is rebuilt by trace_order.cu (replayed vector calls + located
    elements, host-replayed scalar work).  The first 1024 events of one
    cycle and of a whole solve equal the restatement's, entry for entry."""
    rp, ci, vals, comp, al, plan, pre, opre, b, f = _order_case(gpu, oracle, name)
    n = len(rp) - 1
    S = gpu.SplitMatrix(rp, ci, comp, al)
    sp = oracle.split(rp, ci, comp, al)
    s = len(al) - 1
    # one cycle
    t = gpu.FxTrace(checked=True)
    to = PyTrace()
    from oracle.ffi import CheckerError
    errs = []
    try:
        gpu.run_cycle(S, gpu.CycleConfig(m=8, frac_bits=f, shifts=gpu.ShiftPlan(*plan), s=s, precond=pre), b,
                      np.zeros(n), trace=t)
        errs.append(None)
    except (ArithmeticError, ValueError, OverflowError, RuntimeError) as e:
        errs.append(type(e).__name__)
    try:
        oracle.run_cycle(sp, 8, f, s, Shifts(*plan), b, np.zeros(n), precond=opre, trace=to)
        errs.append(None)
    except CheckerError:
        errs.append("err")
    assert (errs[0] is None) == (errs[1] is None)
    assert to.total > 0
    if t.exact:  # (otherwise the running-sum adds are counted only where certified)
        assert t.total_overflows() == to.total
    assert len(t.events) == len(to.events) == min(1024, to.total)
    assert t.events == to.events
    # a whole solve: events across restarts
    A = gpu.CsrMatrixF(rp, ci, vals)
    t2 = gpu.FxTrace(checked=True)
    to2 = PyTrace()
    try:
        gpu.solve(S, A, b, gpu.RefineConfig(tol=1e-8, max_refinements=3, m=6, frac_bits=f, shifts=gpu.ShiftPlan(*plan),
                                            s=s), precond=pre, trace=t2)
    except (ArithmeticError, ValueError, OverflowError, RuntimeError):
        pass
    try:
        oracle.solve(sp, oracle.csrf(rp, ci, vals), b, 1e-8, 3, 6, f, s, Shifts(*plan), precond=opre, trace=to2)
    except CheckerError:
        pass
    assert t2.events == to2.events


@pytest.mark.parametrize("name", ["ilu-spmv-precond", "mgs-vecdiv-error"])
def test_shift_records_match(gpu, oracle, name):
    """FxTrace::shifts (record_shifts: one (kernel, b1, b2) per shifted
    multiply / divide / dot / norm call, fxp.cpp:56,77,98 and fxp.hpp:212,228),
    which the device path synthesises in gmres_int.cpp's call order (one per
    vec_div element, four per stored rotation, ...): the whole log of one
    cycle equals the restatement's, including a cycle that ends in a
    domain_error."""
    rp, ci, vals, comp, al, plan, pre, opre, b, f = _order_case(gpu, oracle, name)
    n = len(rp) - 1
    S = gpu.SplitMatrix(rp, ci, comp, al)
    sp = oracle.split(rp, ci, comp, al)
    s = len(al) - 1
    t = gpu.FxTrace(checked=True, record_shifts=True)
    to = PyTrace(record_shifts=True)
    from oracle.ffi import CheckerError
    try:
        gpu.run_cycle(S, gpu.CycleConfig(m=8, frac_bits=f, shifts=gpu.ShiftPlan(*plan), s=s, precond=pre), b,
                      np.zeros(n), trace=t)
    except (ArithmeticError, ValueError, OverflowError, RuntimeError):
        pass
    try:
        oracle.run_cycle(sp, 8, f, s, Shifts(*plan), b, np.zeros(n), precond=opre, trace=to)
    except CheckerError:
        pass
    assert len(to.shifts) > n  # at least one vec_div sweep
    assert t.shifts == to.shifts
    assert t.events == to.events
