"""Config 3 (n = 1M random band + 10 random columns, GMRES(50), refinement to
1e-10) at WL = 64 (alpha 16, Q33.30, the reference's unpreconditioned preset)
and at WL = 32 (alpha 8, Q13.18, the builder's plan igm_shifts32_plan):
iterations/s and time to solution on one B200.  WL = 32 is checked against the
CPU restatement oracle/igm_oracle32.c at full size when --check is given
(~80 s of CPU), WL = 64 against the reference golden."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2009_07495_b200 as igm
    from workloads import gen
    dev = igm.Device(0)
    igm.Device._default = dev
    n = a.n
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    bh = gen.uniform(gen.SEED_BASE ^ 103, n)
    out = {"n": n, "nnz": int(rp[-1])}
    for wl, alpha, f in ((64, 16, 30), (32, 8, 18)):
        vals, scale = igm.row_scale_device(rp, ci, v, alpha)
        comp, al, _ = igm.build_split_device(vals, alpha, 1)
        b = bh / np.asarray(scale)
        S = igm.SplitMatrix(rp, ci, comp, al)
        A = igm.CsrMatrixF(rp, ci, vals)
        db = torch.from_numpy(b).cuda()
        dx = torch.empty(n, dtype=torch.float64, device="cuda")
        if wl == 64:
            cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=50, frac_bits=f,
                                   shifts=igm.ShiftPlan.default_unpreconditioned(f), checked=True)
            run = lambda: igm.solve(S, A, db, cfg, x_out=dx)
        else:
            S32 = igm.SplitMatrix32(S)
            sh = igm.shifts32_plan(n, alpha, f)
            run = lambda: igm.solve32(S32, A, db, 1e-10, 100, 50, f, 0, sh, x_out=dx)
        _, rep = run()  # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(a.reps):
            _, rep = run()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / a.reps
        rec = {"alpha": alpha, "frac_bits": f, "iters": rep.total_inner_iterations, "refinements": rep.refinements,
               "converged": rep.converged, "final_relres": rep.relres_history[-1], "overflows": rep.overflow_total,
               "s_per_solve": round(dt, 4), "iters_per_s": round(rep.total_inner_iterations / dt, 1)}
        if wl == 32:
            rec["shifts"] = list(sh.astuple())
            if a.check:
                from oracle.ffi import Oracle, Oracle32, Shifts
                O = Oracle()
                Ah = O.csrf(rp, ci, v)
                hv, hs = O.row_scale(Ah, alpha)
                hc, hal, _ = O.build_split(hv, alpha, 1)
                xr, rr = Oracle32().solve(rp, ci, hc.astype(np.int32), hal, hv, bh / hs, 1e-10, 100, 50, f, 0,
                                          Shifts(*sh.astuple()))
                rec["parity_vs_oracle32"] = bool(np.array_equal(dx.cpu().numpy(), xr) and
                                                 rep.relres_history == rr["relres_history"])
        out[f"wl{wl}"] = rec
        print(json.dumps({f"wl{wl}": rec}), flush=True)
    print("@@" + json.dumps(out))


if __name__ == "__main__":
    main()
