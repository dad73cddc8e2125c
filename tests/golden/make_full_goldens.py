"""Generate tests/golden/full_goldens.json: FULL-SIZE reference outputs for the
BASELINE.json configs, computed by the REFERENCE library itself
(oracle/_ref/libintgmres_ref.so, compiled from /root/reference/proj/core).

TEST INFRASTRUCTURE.  Runs only in the build container (the reference does not
travel); the committed JSON (hashes + reports, a few KB) pins the CUDA path at
the sizes BASELINE.json names, in the driver-run `-m gpu` suite
(tests/test_full_size.py) and in bench.py's self-check.

  cfg2  128^3 7-pt upwind CD + ILU(0), GMRES(30), tol 1e-10: setup arrays and
        the whole solve (x, report)                       (refine.cpp:21-106)
  cfg3  n = 1M random band + 10 random columns, WL64, GMRES(50): whole solve
  cfg4  256^3 27-point + ILU(0), GMRES(30): setup arrays, SpMV of a full-range
        vector, one integer ILU apply, the first cycle's state and the whole
        solve                                        (gmres_int.cpp:42-196)
  cfg5  400^3 7-pt (alpha 16, A_0): w = spmv(A, 0, v_30), then for i < 30
        h_i = fx_dot(w, v_i, 16, 0); fx_axpy_sub(w, h_i, v_i, 16)
        (bench_kernels.cpp's call, split.cpp:137-157, fxp.cpp:49-104)

Each config runs in its own process (memory):
    python tests/golden/make_full_goldens.py --configs 2,3,5,4
"""
import argparse
import hashlib
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from workloads import gen  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full_goldens.json")
UNPRE = (16, 0, 16, 16, 16, 14, 16, 0)
PRE = (0, 0, 0, 0, 30, 0, 0, 0)


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_setup(R, rp, ci, v, alpha, ilu):
    A = R.csrf(rp, ci, v)
    vals, scale = R.row_scale(A, alpha)
    As = R.csrf(rp, ci, vals)
    comp, al, _ = R.build_split(As, alpha, 1)
    out = dict(vals=vals, scale=scale, comp=comp, al=al, As=As, sp=R.split(rp, ci, comp, al))
    if ilu:
        lo, up = R.factorize_split_cast(As)
        out.update(lo=lo, up=up, il=R.ilu(lo, up))
    return out


def setup_rec(P):
    rec = {"scaled": h(P["vals"]), "scale": h(P["scale"]), "comp": h(P["comp"]), "alphas": P["al"]}
    if "lo" in P:
        rec["ilu"] = [h(a) for a in list(P["lo"]) + list(P["up"])]
        rec["nnz_l"], rec["nnz_u"] = int(P["lo"][0][-1]), int(P["up"][0][-1])
    return rec


def solve_rec(R, P, b, m, shifts):
    from oracle.ffi import PyTrace, Shifts
    tr = PyTrace()
    t = time.time()
    x, rep = R.solve(P["sp"], P["As"], b, 1e-10, 100, m, 30, 0, Shifts(*shifts), checked=True,
                     precond=P.get("il"), trace=tr)
    wall = rep.pop("wall_time_sec")
    return {"x": h(x), "report": rep, "trace_total": tr.total, "ref_wall_s": round(wall, 2),
            "ref_solve_s": round(time.time() - t, 2)}


def cycle_rec(R, P, b, m, shifts):
    from oracle.ffi import Shifts
    n = len(b)
    cy = R.run_cycle(P["sp"], m, 30, 0, Shifts(*shifts), b, np.zeros(n), precond=P.get("il"))
    return {"dim": cy["dim"], "r0_norm": cy["r0_norm"], "n_basis": cy["n_basis"], "basis": h(cy["basis"]),
            "hess": h(cy["hess"]), "g": h(cy["g"]), "cos_raw": h(cy["cos_raw"]), "sin_raw": h(cy["sin_raw"]),
            "x": h(cy["x"])}


def cfg2(R):
    rp, ci, v = gen.upwind_3d(128, 20.0)
    n = len(rp) - 1
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 2, n))
    P = ref_setup(R, rp, ci, v, 32, True)
    b = bh / P["scale"]
    return {"n": n, "nnz": int(rp[-1]), "inputs": {"matrix": h(v), "b": h(b)}, "setup": setup_rec(P),
            "solve": solve_rec(R, P, b, 30, PRE)}


def cfg3(R):
    n = 1_000_000
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    bh = gen.uniform(gen.SEED_BASE ^ 103, n)
    P = ref_setup(R, rp, ci, v, 16, False)
    b = bh / P["scale"]
    return {"n": n, "nnz": int(rp[-1]), "inputs": {"cols": h(ci), "matrix": h(v), "b": h(b)},
            "setup": setup_rec(P), "solve": solve_rec(R, P, b, 50, UNPRE)}


def cfg4(R, g=256, whole=True):
    rp, ci, v = gen.stencil27_lean(g, gen.SEED_BASE ^ 4)
    n = len(rp) - 1
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 104, n))
    mh = h(v)
    P = ref_setup(R, rp, ci, v, 32, True)
    del v
    b = bh / P["scale"]
    out = {"g": g, "n": n, "nnz": int(rp[-1]), "inputs": {"matrix": mh, "b": h(b)}, "setup": setup_rec(P)}
    vin = gen.uniform_int(gen.SEED_BASE ^ 77, n, -(1 << 40), 1 << 40)
    out["spmv"] = h(R.spmv(P["sp"], 0, vin))
    y = gen.uniform_int(gen.SEED_BASE ^ 78, n, -(1 << 45), 1 << 45)
    out["apply_inverse"] = h(R.apply_inverse(P["il"], y))
    del vin, y
    t = time.time()
    out["cycle"] = cycle_rec(R, P, b, 30, PRE)
    out["cycle"]["ref_s"] = round(time.time() - t, 1)
    if whole:
        out["solve"] = solve_rec(R, P, b, 30, PRE)
    return out


def uniform_int40(n, seed, offset):
    """numpy twin of gen.device_uniform_int40: integers uniform in [-2^40, 2^40)"""
    z = gen.splitmix64(seed, n, offset)
    return ((z >> np.uint64(23)) & np.uint64((1 << 41) - 1)).astype(np.int64) - (1 << 40)


def cfg5(R, g=400, k=30):
    rp, ci, v = gen.upwind_3d_lean(g, 20.0)
    n = len(rp) - 1
    A = R.csrf(rp, ci, v)
    vals, _ = R.row_scale(A, 16)
    del v
    As = R.csrf(rp, ci, vals)
    comp, al, _ = R.build_split(As, 16, 1)
    sp = R.split(rp, ci, comp, al)
    seed = gen.SEED_BASE ^ 5
    t = time.time()
    w = R.spmv(sp, 0, uniform_int40(n, seed, 0))
    hs = []
    for i in range(k):
        vi = uniform_int40(n, seed, (i + 1) * n)
        hi = R.fx_dot(w, vi, 30, 16, 0)
        w = R.fx_axpy_sub(w, hi, vi, 30, 16)
        hs.append(int(hi))
    return {"g": g, "n": n, "nnz": int(rp[-1]), "k": k, "comp": h(comp), "w": h(w), "h": hs,
            "ref_s": round(time.time() - t, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5,4")
    ap.add_argument("--one", default=None, help="internal: run one config in this process")
    ap.add_argument("--g4", type=int, default=256)
    ap.add_argument("--no-whole4", action="store_true")
    a = ap.parse_args()
    if a.one is not None:
        from oracle.ffi import Reference
        R = Reference()
        t = time.time()
        rec = {"2": cfg2, "3": cfg3, "5": cfg5,
               "4": lambda R: cfg4(R, a.g4, not a.no_whole4)}[a.one](R)
        rec["gen_wall_s"] = round(time.time() - t, 1)
        print("@@" + json.dumps(rec), flush=True)
        return
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data["_source"] = ("reference library (oracle/_ref, built from /root/reference/proj/core) at the "
                       "BASELINE.json sizes; inputs from workloads/gen.py; regenerate with "
                       "tests/golden/make_full_goldens.py")
    for c in a.configs.split(","):
        cmd = [sys.executable, __file__, "--one", c, "--g4", str(a.g4)] + (["--no-whole4"] if a.no_whole4 else [])
        p = subprocess.run(cmd, capture_output=True, text=True)
        line = [ln for ln in p.stdout.splitlines() if ln.startswith("@@")]
        if p.returncode != 0 or not line:
            print(f"cfg{c} FAILED rc={p.returncode}\n{p.stderr[-3000:]}", flush=True)
            continue
        data[f"cfg{c}"] = json.loads(line[0][2:])
        print(f"cfg{c} done ({data[f'cfg{c}']['gen_wall_s']} s)", flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
