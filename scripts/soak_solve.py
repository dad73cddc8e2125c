"""Soak: N whole config-2 solves (and M config-1-size solves with a wrapping
plan) back to back, every x hashed against the first one / the reference
golden -- a race in the persistent Arnoldi kernel's streaming refill, the
pair recount or the SpMV certificate would show up as a differing word.

    python scripts/soak_solve.py [n_solves] [2|3]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2009_07495_b200 as igm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
which = sys.argv[2] if len(sys.argv) > 2 else "2"
with open(os.path.join(bench.ROOT, "tests", "golden", "full_goldens.json")) as f:
    golds = json.load(f)
if which == "3":  # n = 1M random band, GMRES(50): sliced-ELL SpMV + persistent Arnoldi step
    from workloads import gen
    n = golds["cfg3"]["n"]
    rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
    vals, scale = igm.row_scale_device(rp, ci, v, 16)
    comp, al, _ = igm.build_split_device(vals, 16, 1)
    b = gen.uniform(gen.SEED_BASE ^ 103, n) / np.asarray(scale)
    S, A, F = igm.SplitMatrix(rp, ci, comp, al), igm.CsrMatrixF(rp, ci, vals), None
    cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=50, frac_bits=30,
                           shifts=igm.ShiftPlan.default_unpreconditioned(30), checked=True)
    gold, its = golds["cfg3"]["solve"]["x"], golds["cfg3"]["solve"]["report"]["total_inner_iterations"]
else:
    rp, ci, v, bh = bench.config2(128)
    S, A, F, b, lower, upper, _ = bench.setup_b200(rp, ci, v, bh)
    cfg = bench.solve_cfg(igm)
    gold, its = golds["cfg2"]["solve"]["x"], 150
t0 = time.time()
bad = 0
for i in range(N):
    x, rep = igm.solve(S, A, b, cfg, precond=F)
    h = hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()
    if h != gold or rep.total_inner_iterations != its:
        bad += 1
        print(f"solve {i}: x differs from the reference golden ({h[:16]}), {rep.total_inner_iterations} iterations")
print(f"{N} config-{which} solves in {time.time() - t0:.1f} s, {bad} differing from the reference golden")
sys.exit(1 if bad else 0)
