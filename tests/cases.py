"""Parity cases shared by the oracle tests, the GPU tests and the golden generator.

Each case builds its inputs with workloads.gen (seeded) and runs the host setup
(row scaling, splitting, ILU(0) + cast) with the given checker backend, so the
oracle, the reference and the B200 product all see identical arrays.
"""
import numpy as np

from workloads import gen

UNPRE = (16, 0, 16, 16, 16, 14, 16, 0)   # ShiftPlan::default_unpreconditioned(Q.30)
PRE = (0, 0, 0, 0, 30, 0, 0, 0)          # ShiftPlan::default_preconditioned(Q.30)

CASES = {
    # config 1 of BASELINE.json (2D upwind CD 64x64, alpha 16, GMRES(30), tol 1e-10)
    "cfg1": dict(kind="upwind2d", g=64, alpha=16, ncomp=1, s=0, m=30, tol=1e-10, max_ref=1000,
                 shifts=UNPRE, ilu=False, solve=True, cycle=True, spmv=True, setup=True, seed=1),
    # config 2 family at 16^3 (ILU(0), alpha 32, preconditioned preset)
    "cfg2_16": dict(kind="upwind3d", g=16, alpha=32, ncomp=1, s=0, m=30, tol=1e-10, max_ref=100,
                    shifts=PRE, ilu=True, solve=True, cycle=True, ilu_apply=True, setup=True, seed=2),
    # config 4 family (27-point) at 12^3 with ILU(0)
    "cfg4_12": dict(kind="stencil27", g=12, alpha=32, ncomp=1, s=0, m=30, tol=1e-10, max_ref=100,
                    shifts=PRE, ilu=True, solve=True, cycle=True, ilu_apply=True, setup=True, seed=4),
    # config 3 family (random band + 10 random columns), small n, GMRES(50)
    "cfg3_small": dict(kind="random_band", n=3000, alpha=16, ncomp=1, s=0, m=50, tol=1e-10, max_ref=100,
                       shifts=UNPRE, ilu=False, solve=True, cycle=True, spmv=True, setup=True, seed=3),
    # multi-component split (s = depth) on a random dominant matrix
    "split_s3": dict(kind="random_dominant", n=200, alpha=16, ncomp=4, s=3, m=20, tol=1e-10, max_ref=200,
                     shifts=UNPRE, ilu=False, solve=True, cycle=True, spmv=True, setup=True, seed=5),
    # ILU on a random dominant (unstructured: contiguous tiles)
    "ilu_random": dict(kind="random_dominant", n=400, alpha=32, ncomp=1, s=0, m=20, tol=1e-10, max_ref=100,
                       shifts=PRE, ilu=True, solve=True, cycle=True, ilu_apply=True, setup=True, seed=6),
}


def matrix(c):
    k = c["kind"]
    if k == "upwind2d":
        return gen.upwind_2d(c["g"])
    if k == "upwind3d":
        return gen.upwind_3d(c["g"], 20.0)
    if k == "stencil27":
        return gen.stencil27(c["g"], gen.SEED_BASE ^ 4)
    if k == "random_band":
        return gen.random_band(c["n"], gen.SEED_BASE ^ 3)
    if k == "random_dominant":
        return gen.random_dominant(c["n"], 0.05, 1.3, gen.SEED_BASE ^ c["seed"])
    raise KeyError(k)


def build_case(name, B):
    """Inputs + checker-side handles for backend B (Oracle or Reference)."""
    c = dict(CASES[name])
    rp, ci, v = matrix(c)
    n = len(rp) - 1
    c.update(rp=rp, ci=ci, v=v, n=n)
    A = B.csrf(rp, ci, v)
    vals, scale = B.row_scale(A, c["alpha"])
    af = B.csrf(rp, ci, vals)
    if B.prefix == "ref_":
        comp, alphas, _ = B.build_split(af, c["alpha"], c["ncomp"])
    else:
        comp, alphas, _ = B.build_split(vals, c["alpha"], c["ncomp"])
    c["ncomp"] = len(alphas)
    c["s"] = min(c["s"], len(alphas) - 1)
    xs = gen.uniform(gen.SEED_BASE ^ (100 + c["seed"]), n)
    bh = gen.spmv_np(rp, ci, v, xs)
    c.update(vals=vals, scale=scale, comp=comp, alphas=alphas, b=bh / scale, af=af,
             sp=B.split(rp, ci, comp, alphas))
    if c.get("ilu"):
        lo, up = B.factorize_split_cast(af)
        c["ilu_arrays"] = list(lo) + list(up)
        c["lower"], c["upper"] = lo, up
        c["il"] = B.ilu(lo, up)
    c["v_full"] = gen.uniform_int(gen.SEED_BASE ^ 77, n, -(1 << 62), (1 << 62) - 1) * 2 + 1
    c["y_int"] = gen.uniform_int(gen.SEED_BASE ^ 78, n, -(1 << 45), 1 << 45)
    c["y_fp"] = gen.uniform(gen.SEED_BASE ^ 79, n)
    return c
