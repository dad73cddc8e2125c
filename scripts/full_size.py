"""Full-size runs of BASELINE configs 2, 3 and 4 on one B200 with parity
against the CPU oracle (test infrastructure: the oracle is the checker).

  cfg2  128^3 7-pt upwind CD, ILU(0), GMRES(30): the whole solve bit-exact
        vs the oracle (every x word, relres / gamma history, inner dims).
  cfg3  n = 1M random band + 10 random columns, WL64, GMRES(50), b ~ U[-1,1):
        the whole solve bit-exact vs the oracle.
  cfg4  256^3 27-point, ILU(0), GMRES(30): SpMV, one ILU apply and the first
        2-step cycle bit-exact vs the oracle (its full solve would take hours
        on one core); the full GPU solve checked by properties (converged,
        relres < tol, an independent FP64 residual of x).

Writes one JSON object per config to the path given by --out."""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2009_07495_b200 as igm  # noqa: E402
from oracle.ffi import Oracle, Shifts  # noqa: E402
from workloads import gen  # noqa: E402

UNPRE = (16, 0, 16, 16, 16, 14, 16, 0)
PRE = (0, 0, 0, 0, 30, 0, 0, 0)


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def setup(rp, ci, v, bh, alpha, ncomp, ilu):
    t = time.time()
    vals, scale = igm.row_scale(rp, ci, v, alpha)
    comp, al, _ = igm.build_split(vals, alpha, ncomp)
    fac = igm.factorize_split_cast(rp, ci, vals) if ilu else None
    return dict(vals=vals, scale=scale, comp=comp, al=al, fac=fac, b=bh / scale, setup_s=time.time() - t)


def dev_setup(rp, ci, v, P, alpha, ncomp, ilu):
    """device-side setup (8(f) row 1) from device-resident inputs: timing and
    array-for-array equality with the host setup P"""
    import torch
    td = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    rpd, cid, vd = td(rp), td(ci), td(v)
    torch.cuda.synchronize()
    t = time.time()
    vals, scale = igm.row_scale_device(rpd, cid, vd, alpha)
    comp, al, _ = igm.build_split_device(vals, alpha, ncomp)
    fac = igm.factorize_split_cast_device(rpd, cid, vals) if ilu else None
    torch.cuda.synchronize()
    dt = time.time() - t
    same = (np.array_equal(vals.cpu().numpy(), P["vals"]) and np.array_equal(scale.cpu().numpy(), P["scale"])
            and al == list(P["al"]) and np.array_equal(comp.cpu().numpy(), np.atleast_2d(P["comp"])))
    if ilu:
        for a, b in zip(fac[0] + fac[1], list(P["fac"][0]) + list(P["fac"][1])):
            same = same and np.array_equal(a.cpu().numpy(), np.asarray(b))
    return dict(device_setup_s=dt, device_setup_bit_exact=bool(same))


def gpu_solve(rp, ci, P, m, shifts, tol=1e-10, reps=2):
    S = igm.SplitMatrix(rp, ci, P["comp"], P["al"])
    A = igm.CsrMatrixF(rp, ci, P["vals"])
    F = igm.IluFactors(*P["fac"]) if P["fac"] is not None else None
    cfg = igm.RefineConfig(tol=tol, max_refinements=100, m=m, frac_bits=30, shifts=igm.ShiftPlan(*shifts),
                           checked=True)
    import torch
    bd = torch.from_numpy(P["b"]).cuda()
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.time()
        x, rep = igm.solve(S, A, bd, cfg, precond=F)
        torch.cuda.synchronize()
        dt = time.time() - t
        best = dt if best is None else min(best, dt)
    return S, A, F, x.cpu().numpy() if hasattr(x, "cpu") else x, rep, best


def class_times(S, A, F, P, m, shifts):
    """per-kernel-class device time of one more solve (CUDA events, igm_profile_*)"""
    import torch
    from paper_2009_07495_b200._capi import KCLASS_NAMES
    cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=m, frac_bits=30, shifts=igm.ShiftPlan(*shifts),
                           checked=True)
    bd = torch.from_numpy(P["b"]).cuda()
    igm.lib().igm_profile_enable(1)
    igm.solve(S, A, bd, cfg, precond=F)
    igm.lib().igm_profile_enable(0)
    kms = np.zeros(len(KCLASS_NAMES))
    kcnt = np.zeros(len(KCLASS_NAMES), np.uint64)
    igm.lib().igm_profile_collect(kms.ctypes.data_as(igm._capi.f64p), kcnt.ctypes.data_as(igm._capi.u64p))
    return {nm: [round(float(kms[i]), 3), int(kcnt[i])] for i, nm in enumerate(KCLASS_NAMES) if kcnt[i]}


def report(rep):
    return dict(converged=rep.converged, refinements=rep.refinements,
                iterations=rep.total_inner_iterations, relres=rep.relres_history[-1],
                overflows=rep.overflow_total)


def oracle_solve(O, rp, ci, P, m, shifts):
    sp, af = O.split(rp, ci, P["comp"], P["al"]), O.csrf(rp, ci, P["vals"])
    il = O.ilu(*P["fac"]) if P["fac"] is not None else None
    t = time.time()
    xo, ro = O.solve(sp, af, P["b"], 1e-10, 100, m, 30, 0, Shifts(*shifts), precond=il)
    return xo, ro, time.time() - t


def full_parity(out, name, rp, ci, P, m, shifts, O):
    S, A, F, x, rep, dt = gpu_solve(rp, ci, P, m, shifts)
    xo, ro, to = oracle_solve(O, rp, ci, P, m, shifts)
    same = (np.array_equal(x, xo) and rep.relres_history == ro["relres_history"]
            and rep.inner_dims == ro["inner_dims"] and rep.gamma_history == ro["gamma_history"])
    out.update(gpu=report(rep), gpu_solve_s=dt, gpu_iters_per_s=rep.total_inner_iterations / dt,
               oracle_solve_s=to, oracle_iters_per_s=ro["total_inner_iterations"] / to,
               x_hash=h(x), bit_exact_solve=bool(same))
    assert same, f"{name}: solve differs from the oracle"


def cfg2(O):
    g = 128
    rp, ci, v = gen.upwind_3d(g, 20.0)
    n = len(rp) - 1
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 2, n))
    P = setup(rp, ci, v, bh, 32, 1, True)
    out = dict(config="cfg2", n=n, nnz=int(rp[-1]), setup_s=P["setup_s"])
    out.update(dev_setup(rp, ci, v, P, 32, 1, True))
    full_parity(out, "cfg2", rp, ci, P, 30, PRE, O)
    return out


def cfg3(O):
    n = 1_000_000
    t = time.time()
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    bh = gen.uniform(gen.SEED_BASE ^ 103, n)
    gen_s = time.time() - t
    P = setup(rp, ci, v, bh, 16, 1, False)
    out = dict(config="cfg3 (WL64)", n=n, nnz=int(rp[-1]), gen_s=gen_s, setup_s=P["setup_s"])
    full_parity(out, "cfg3", rp, ci, P, 50, UNPRE, O)
    return out


def cfg4(O, g=256):
    t = time.time()
    rp, ci, v = gen.stencil27_lean(g, gen.SEED_BASE ^ 4)
    n = len(rp) - 1
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 104, n))
    gen_s = time.time() - t
    P = setup(rp, ci, v, bh, 32, 1, True)
    out = dict(config=f"cfg4 ({g}^3 27-pt)", n=n, nnz=int(rp[-1]), nnz_l=int(P["fac"][0][0][-1]),
               gen_s=gen_s, setup_s=P["setup_s"])
    out.update(dev_setup(rp, ci, v, P, 32, 1, True))
    t = time.time()
    S, A, F, x, rep, dt = gpu_solve(rp, ci, P, 30, PRE, reps=1)
    out["upload_and_solve_s"] = time.time() - t
    out.update(gpu=report(rep), gpu_solve_s=dt, gpu_iters_per_s=rep.total_inner_iterations / dt,
               levels=[F.levels(False), F.levels(True)], schedule=[F.schedule_info(False), F.schedule_info(True)])
    out["breakdown_ms"] = class_times(S, A, F, P, 30, PRE)
    # property: independent FP64 residual of the GPU's x on the scaled system
    r = P["b"] - gen.spmv_np(rp, ci, P["vals"], x)
    out["indep_relres"] = float(np.linalg.norm(r) / np.linalg.norm(P["b"]))
    assert rep.converged and out["indep_relres"] < 1e-9
    # bit-exact pieces vs the oracle at full size
    sp, il = O.split(rp, ci, P["comp"], P["al"]), O.ilu(*P["fac"])
    vin = gen.uniform_int(gen.SEED_BASE ^ 77, n, -(1 << 40), 1 << 40)
    t = time.time()
    ok_spmv = np.array_equal(igm.spmv(S, 0, vin), O.spmv(sp, 0, vin))
    y = gen.uniform_int(gen.SEED_BASE ^ 78, n, -(1 << 45), 1 << 45)
    ok_ilu = np.array_equal(igm.apply_inverse(F, y), O.apply_inverse(il, y))
    cyc = igm.run_cycle(S, igm.CycleConfig(m=2, shifts=igm.ShiftPlan(*PRE), precond=F), P["b"], np.zeros(n))
    ro = O.run_cycle(sp, 2, 30, 0, Shifts(*PRE), P["b"], np.zeros(n), precond=il)
    ok_cyc = (cyc.dim == ro["dim"] and np.array_equal(cyc.basis, ro["basis"])
              and np.array_equal(cyc.hess, ro["hess"]) and np.array_equal(cyc.x, ro["x"]))
    out.update(bit_exact_spmv=bool(ok_spmv), bit_exact_ilu_apply=bool(ok_ilu), bit_exact_cycle_m2=bool(ok_cyc),
               oracle_pieces_s=time.time() - t)
    assert ok_spmv and ok_ilu and ok_cyc
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,2,4")
    ap.add_argument("--out", default="gpurun_out/full_size.jsonl")
    ap.add_argument("--g4", type=int, default=256)
    a = ap.parse_args()
    O = Oracle()
    for c in a.configs.split(","):
        t = time.time()
        res = {"2": cfg2, "3": cfg3, "4": lambda O: cfg4(O, a.g4)}[c](O)
        res["wall_s"] = time.time() - t
        print(json.dumps(res), flush=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(res) + "\n")
