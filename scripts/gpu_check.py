"""Quick GPU-vs-oracle parity sweep (developer tool; the pytest suite is tests/)."""
import sys, time, traceback
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import paper_2009_07495_b200 as igm
from oracle.ffi import Oracle, Shifts, PyTrace
from workloads import gen

O = Oracle()
ok_all = True
def check(name, cond):
    global ok_all
    print(("PASS " if cond else "FAIL ") + name, flush=True)
    ok_all &= bool(cond)

def prob(rp, ci, v, alpha, ncomp, seed):
    vals, scale = igm.row_scale(rp, ci, v, alpha)
    comp, al, ex = igm.build_split(vals, alpha, ncomp)
    xs = gen.uniform(seed, len(rp) - 1)
    b = gen.spmv_np(rp, ci, v, xs) / scale
    return vals, comp, al, b

try:
    t0 = time.time()
    rp, ci, v = gen.upwind_2d(64)
    vals, comp, al, b = prob(rp, ci, v, 16, 3, 11)
    S = igm.SplitMatrix(rp, ci, comp, al)
    So = O.split(rp, ci, comp, al)
    n = len(rp) - 1
    rng = np.random.default_rng(1)
    for s in range(len(al)):
        vv = rng.integers(-(1 << 31), 1 << 31, n, dtype=np.int64)
        check(f"spmv s={s}", np.array_equal(igm.spmv(S, s, vv), O.spmv(So, s, vv)))
    vv = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, n, dtype=np.int64)
    t1, t2 = igm.FxTrace(), PyTrace()
    check("spmv fullrange", np.array_equal(igm.spmv(S, 0, vv, t1), O.spmv(So, 0, vv, t2)))
    check(f"spmv overflow count {t1.total_overflows()} vs {t2.total}", t1.total_overflows() == t2.total)
    w = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
    check("fx_dot", igm.fx_dot(vv, w, 30, 16, 0) == O.fx_dot(vv, w, 30, 16, 0))
    check("fx_norm", igm.fx_norm(w, 30, 16) == O.fx_norm(w, 30, 16))
    ww = w.copy(); igm.fx_axpy_sub(ww, 123456789, vv, 30, 16)
    check("fx_axpy", np.array_equal(ww, O.fx_axpy_sub(w, 123456789, vv, 30, 16)))
    xx = rng.uniform(-1, 1, n)
    A = igm.CsrMatrixF(rp, ci, vals); Ao = O.csrf(rp, ci, vals)
    r1, rel1 = igm.residual_fp(A, xx, b); r2, rel2 = O.residual_fp(Ao, xx, b)
    check("residual_fp", np.array_equal(r1, r2) and rel1 == rel2)
    check("norm2", igm.norm2(xx) == O.norm2(xx))
    # run_cycle unpreconditioned
    sh = igm.ShiftPlan.default_unpreconditioned(30)
    cfg = igm.CycleConfig(m=30, frac_bits=30, shifts=sh, s=0)
    c1 = igm.run_cycle(S, cfg, b, np.zeros(n))
    c2 = O.run_cycle(So, 30, 30, 0, Shifts(16, 0, 16, 16, 16, 14, 16, 0), b, np.zeros(n))
    check(f"cycle dim {c1.dim} {c2['dim']}", c1.dim == c2["dim"])
    check("cycle hess", np.array_equal(c1.hess, c2["hess"]))
    check("cycle g", np.array_equal(c1.g, c2["g"]))
    check("cycle basis", np.array_equal(c1.basis, c2["basis"]))
    check("cycle x", np.array_equal(c1.x, c2["x"]))
    # solve cfg1
    comp1, al1, _ = igm.build_split(vals, 16, 1)
    S1 = igm.SplitMatrix(rp, ci, comp1, al1); S1o = O.split(rp, ci, comp1, al1)
    rc = igm.RefineConfig(tol=1e-10, max_refinements=1000, m=30, frac_bits=30, shifts=sh, s=0)
    t0s = time.time(); x1, rep1 = igm.solve(S1, A, b, rc); ts = time.time() - t0s
    x2, rep2 = O.solve(S1o, Ao, b, 1e-10, 1000, 30, 30, 0, Shifts(16, 0, 16, 16, 16, 14, 16, 0))
    print("gpu solve", ts, rep1.refinements, rep1.total_inner_iterations, rep1.relres_history[-1])
    check("solve x", np.array_equal(x1, x2))
    check("solve relres", rep1.relres_history == rep2["relres_history"])
    check("solve dims", rep1.inner_dims == rep2["inner_dims"])
    # ILU path on a small 3D problem
    rp3, ci3, v3 = gen.upwind_3d(16)
    vals3, comp3, al3, b3 = prob(rp3, ci3, v3, 32, 1, 22)
    lo, up = igm.factorize_split_cast(rp3, ci3, vals3)
    A3o = O.csrf(rp3, ci3, vals3)
    lo2, up2 = O.factorize_split_cast(A3o)
    check("ilu setup", all(np.array_equal(a, c) for a, c in zip(lo + up, lo2 + up2)))
    F = igm.IluFactors(lo, up); Fo = O.ilu(lo, up)
    n3 = len(rp3) - 1
    print("levels", F.levels(False), F.levels(True))
    y = rng.integers(-(1 << 45), 1 << 45, n3, dtype=np.int64)
    check("apply_inverse", np.array_equal(igm.apply_inverse(F, y), O.apply_inverse(Fo, y)))
    yf = rng.uniform(-1, 1, n3)
    check("apply_inverse_fp", np.array_equal(igm.apply_inverse_fp(F, yf), O.apply_inverse_fp(Fo, yf)))
    S3 = igm.SplitMatrix(rp3, ci3, comp3, al3); S3o = O.split(rp3, ci3, comp3, al3)
    A3 = igm.CsrMatrixF(rp3, ci3, vals3)
    shp = igm.ShiftPlan.default_preconditioned(30)
    rc3 = igm.RefineConfig(tol=1e-10, max_refinements=100, m=30, frac_bits=30, shifts=shp, s=0)
    x3, rep3 = igm.solve(S3, A3, b3, rc3, precond=F)
    x4, rep4 = O.solve(S3o, A3o, b3, 1e-10, 100, 30, 30, 0, Shifts(0, 0, 0, 0, 30, 0, 0, 0), precond=Fo)
    print("ilu solve", rep3.refinements, rep3.total_inner_iterations, rep3.relres_history[-1], rep4["relres_history"][-1])
    check("ilu solve x", np.array_equal(x3, x4))
    check("ilu solve relres", rep3.relres_history == rep4["relres_history"])
    print("elapsed", time.time() - t0)
except Exception:
    traceback.print_exc()
    ok_all = False
print("ALL OK" if ok_all else "SOME FAILED")
sys.exit(0 if ok_all else 1)
