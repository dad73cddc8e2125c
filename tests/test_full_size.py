"""Full-size parity at the BASELINE.json sizes, against golden outputs of the
REFERENCE library (tests/golden/full_goldens.json, made by
tests/golden/make_full_goldens.py from oracle/_ref in the build container).

  cfg2  128^3 7-pt + ILU(0), GMRES(30): device setup arrays and the whole
        solve (every x word, relres / gamma histories, dims, overflow counts)
  cfg3  n = 1M random band, WL64, GMRES(50): device setup and the whole solve
  cfg4  256^3 27-point + ILU(0): device setup, SpMV, one ILU apply, the first
        cycle's state (basis, H, g, cos, sin, x) and the whole solve
  cfg5  400^3 kernel call: w = spmv(A, 0, v_30) + MGS against 30 vectors

Inputs are regenerated from workloads/gen.py (seeded SplitMix64); the input
hashes are checked first so a generator change cannot pass silently.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from workloads import gen

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_goldens.json")
UNPRE = (16, 0, 16, 16, 16, 14, 16, 0)
PRE = (0, 0, 0, 0, 30, 0, 0, 0)


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def h(a) -> str:
    a = _np(a)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def full():
    with open(GOLD) as f:
        return json.load(f)


def device_setup(igm, rp, ci, v, alpha, ilu):
    vals, scale = igm.row_scale_device(rp, ci, v, alpha)
    comp, al, _ = igm.build_split_device(vals, alpha, 1)
    out = dict(vals=vals, scale=scale, comp=comp, al=al)
    if ilu:
        out["fac"] = igm.factorize_split_cast_device(rp, ci, vals)
    return out


def check_setup(P, g):
    assert h(P["vals"]) == g["scaled"] and h(P["scale"]) == g["scale"]
    assert h(P["comp"]) == g["comp"] and list(P["al"]) == g["alphas"]
    if "ilu" in g:
        arrs = list(P["fac"][0]) + list(P["fac"][1])
        dts = [np.int32, np.int32, np.int64, np.int32] * 2
        got = [h(np.ascontiguousarray(a.cpu().numpy() if hasattr(a, "cpu") else a, dt)) for a, dt in zip(arrs, dts)]
        assert got == g["ilu"], "device ILU(0) + split_cast differs from the reference"


def check_solve(igm, S, A, F, b, m, shifts, g):
    cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=m, frac_bits=30, shifts=igm.ShiftPlan(*shifts),
                           checked=True)
    tr = igm.FxTrace()
    x, rep = igm.solve(S, A, b, cfg, precond=F, trace=tr)
    r = g["report"]
    assert rep.inner_dims == r["inner_dims"]
    assert rep.relres_history == r["relres_history"]
    assert rep.gamma_history == r["gamma_history"]
    assert rep.converged == r["converged"] and rep.refinements == r["refinements"]
    assert rep.total_inner_iterations == r["total_inner_iterations"]
    assert rep.overflow_per_restart == r["overflow_per_restart"] and rep.overflow_total == r["overflow_total"]
    assert tr.total_overflows() == g["trace_total"]
    assert h(x) == g["x"], "x differs from the reference solve"


def test_cfg2_full_solve(full):
    import paper_2009_07495_b200 as igm
    g = full["cfg2"]
    rp, ci, v = gen.upwind_3d(128, 20.0)
    n = len(rp) - 1
    assert n == g["n"] and h(v) == g["inputs"]["matrix"]
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 2, n))
    P = device_setup(igm, rp, ci, v, 32, True)
    check_setup(P, g["setup"])
    b = bh / _np(P["scale"])
    assert h(b) == g["inputs"]["b"]
    S = igm.SplitMatrix(rp, ci, P["comp"], P["al"])
    A = igm.CsrMatrixF(rp, ci, P["vals"])
    F = igm.IluFactors(*P["fac"])
    check_solve(igm, S, A, F, b, 30, PRE, g["solve"])


def test_cfg3_full_solve(full):
    import paper_2009_07495_b200 as igm
    g = full["cfg3"]
    n = g["n"]
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    assert h(ci) == g["inputs"]["cols"] and h(v) == g["inputs"]["matrix"]
    bh = gen.uniform(gen.SEED_BASE ^ 103, n)
    P = device_setup(igm, rp, ci, v, 16, False)
    check_setup(P, g["setup"])
    b = bh / _np(P["scale"])
    assert h(b) == g["inputs"]["b"]
    S = igm.SplitMatrix(rp, ci, P["comp"], P["al"])
    A = igm.CsrMatrixF(rp, ci, P["vals"])
    check_solve(igm, S, A, None, b, 50, UNPRE, g["solve"])


@pytest.fixture(scope="module")
def cfg4(full):
    import paper_2009_07495_b200 as igm
    if "cfg4" not in full:
        pytest.skip("config-4 reference golden not generated (tests/golden/make_full_goldens.py --configs 4)")
    g = full["cfg4"]
    rp, ci, v = gen.stencil27_lean(g["g"], gen.SEED_BASE ^ 4)
    n = len(rp) - 1
    assert n == g["n"] and h(v) == g["inputs"]["matrix"]
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 104, n))
    P = device_setup(igm, rp, ci, v, 32, True)
    del v
    b = bh / _np(P["scale"])
    S = igm.SplitMatrix(rp, ci, P["comp"], P["al"])
    A = igm.CsrMatrixF(rp, ci, P["vals"])
    F = igm.IluFactors(*P["fac"])
    yield dict(g=g, P=P, b=b, S=S, A=A, F=F, n=n)


def test_cfg4_setup_spmv_ilu(cfg4):
    import paper_2009_07495_b200 as igm
    g, n = cfg4["g"], cfg4["n"]
    check_setup(cfg4["P"], g["setup"])
    assert h(cfg4["b"]) == g["inputs"]["b"]
    assert cfg4["F"].pencil_bricks(False) > 0, "27-point pencil wavefront not selected"
    vin = gen.uniform_int(gen.SEED_BASE ^ 77, n, -(1 << 40), 1 << 40)
    assert h(igm.spmv(cfg4["S"], 0, vin)) == g["spmv"]
    y = gen.uniform_int(gen.SEED_BASE ^ 78, n, -(1 << 45), 1 << 45)
    assert h(igm.apply_inverse(cfg4["F"], y)) == g["apply_inverse"]


def test_cfg4_first_cycle(cfg4):
    import paper_2009_07495_b200 as igm
    g, n = cfg4["g"]["cycle"], cfg4["n"]
    cyc = igm.run_cycle(cfg4["S"], igm.CycleConfig(m=30, shifts=igm.ShiftPlan(*PRE), precond=cfg4["F"]),
                        cfg4["b"], np.zeros(n))
    assert cyc.dim == g["dim"] and cyc.r0_norm == g["r0_norm"]
    assert len(cyc.basis) == g["n_basis"] and h(cyc.basis) == g["basis"]
    for k in ("hess", "g", "cos_raw", "sin_raw", "x"):
        assert h(getattr(cyc, k)) == g[k], k


def test_cfg4_full_solve(cfg4):
    import paper_2009_07495_b200 as igm
    if "solve" not in cfg4["g"]:
        pytest.skip("reference whole-solve golden not generated")
    check_solve(igm, cfg4["S"], cfg4["A"], cfg4["F"], cfg4["b"], 30, PRE, cfg4["g"]["solve"])


def test_cfg5_kernel_call(full):
    import torch
    import paper_2009_07495_b200 as igm
    g = full["cfg5"]
    rp, ci, v = gen.upwind_3d_lean(g["g"], 20.0)
    n = len(rp) - 1
    vals, _ = igm.row_scale_device(rp, ci, v, 16)
    del v
    comp, al, _ = igm.build_split_device(vals, 16, 1)
    del vals
    assert h(comp) == g["comp"]
    S = igm.SplitMatrix(rp, ci, comp, al)
    del comp
    seed = gen.SEED_BASE ^ 5
    k = g["k"]
    basis = torch.empty((k, n), dtype=torch.int64, device="cuda")
    for i in range(k):
        basis[i] = gen.device_uniform_int40(n, seed, (i + 1) * n, "cuda")
    vin = gen.device_uniform_int40(n, seed, 0, "cuda")
    w = torch.empty(n, dtype=torch.int64, device="cuda")
    hs = igm.spmv_mgs(S, 0, vin, basis, k, 30, 16, 0, 16, w)
    torch.cuda.synchronize()
    assert [int(x) for x in hs] == g["h"]
    assert h(w) == g["w"]
    del S, basis, vin, w
    torch.cuda.empty_cache()
