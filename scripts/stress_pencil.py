"""Repeat pencil-wavefront applies on several grids and compare every result
with the first (and the oracle once): catches intermittent handoff races."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07495_b200 as igm
from oracle.ffi import Oracle
from workloads import gen

O = Oracle()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
offs7 = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
offs27 = [(a, b, c) for c in (-1, 0, 1) for b in (-1, 0, 1) for a in (-1, 0, 1)]
bad = 0
cases = [(d, offs7) for d in [(128, 128, 128), (64, 96, 33), (17, 35, 9), (200, 24, 10)]]
cases += [(d, offs27) for d in [(96, 96, 48), (33, 47, 21), (12, 12, 12)]]
for dims, offs in cases:
    rng = np.random.default_rng(sum(dims))
    coef = {q: rng.uniform(-1.4, -0.6) for q in range(len(offs))}
    coef[offs.index((0, 0, 0))] = 2.0 * len(offs)
    rp, ci, v = gen._stencil_csr(dims, offs, lambda o, r: np.full(r.shape, coef[o]))
    vals, _ = igm.row_scale(rp, ci, v, 32)
    lo, up = igm.factorize_split_cast(rp, ci, vals)
    F = igm.IluFactors(lo, up)
    n = len(rp) - 1
    y = gen.uniform_int(5, n, -(1 << 45), 1 << 45)
    yf = gen.uniform(6, n)
    want = O.apply_inverse(O.ilu(lo, up), y) if n <= 300000 else None
    first = igm.apply_inverse(F, y)
    firstf = igm.apply_inverse_fp(F, yf)
    if want is not None and not np.array_equal(first, want):
        bad += 1
        print("oracle mismatch", dims)
    for r in range(reps):
        if not np.array_equal(igm.apply_inverse(F, y), first):
            bad += 1
            print("int mismatch", dims, r)
        if not np.array_equal(igm.apply_inverse_fp(F, yf).view(np.int64), firstf.view(np.int64)):
            bad += 1
            print("fp mismatch", dims, r)
    print(dims, len(offs), "pt, pencil bricks", F.pencil_bricks(False), "reps", reps, "bad so far", bad, flush=True)
print("TOTAL BAD", bad)
