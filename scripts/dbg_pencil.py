"""Debug: one triangular solve at a time through the C ABI (the other factor
the identity), pencil path vs a sequential Python substitution."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07495_b200 as igm
from workloads import gen

g = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rp, ci, v = gen.upwind_3d(g, 20.0)
n = len(rp) - 1
vals, scale = igm.row_scale(rp, ci, v, 32)
lo, up = igm.factorize_split_cast(rp, ci, vals)

def ident():
    return (np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.ones(n, np.int64), np.arange(n, dtype=np.int32))

def solve(f, y, upper):
    frp, fci, fv, fdp = f
    z = [0] * n
    order = range(n - 1, -1, -1) if upper else range(n)
    for r in order:
        acc = int(y[r])
        for q in range(frp[r], frp[r + 1]):
            if q == fdp[r]:
                continue
            acc = (acc - int(fv[q]) * z[fci[q]]) & ((1 << 64) - 1)
            if acc >= 1 << 63: acc -= 1 << 64
        d = int(fv[fdp[r]])
        qq = abs(acc) // abs(d)
        z[r] = qq if (acc < 0) == (d < 0) else -qq
        z[r] = ((z[r] + (1 << 63)) % (1 << 64)) - (1 << 63)
    return np.array(z, dtype=np.int64)

rng = np.random.default_rng(3)
y = rng.integers(-(1 << 45), 1 << 45, n, dtype=np.int64)
print("lower nnz", lo[0][-1], "upper nnz", up[0][-1], "maxabs", np.abs(lo[2][:lo[0][-1]]).max(), np.abs(up[2][:up[0][-1]]).max())
for name, L, U, upper in (("lower", lo, ident(), False), ("upper", ident(), up, True)):
    F = igm.IluFactors(L, U)
    info = F.schedule_info(backward=upper)
    got = igm.apply_inverse(F, y)
    ref = solve(U if upper else L, y, upper)
    bad = np.nonzero(got != ref)[0]
    print(name, info, "mismatches", len(bad))
    for r in bad[:8]:
        rs = n - 1 - r if upper else r
        print("   row", r, "solve-order (i,j,k)", (rs % g, (rs // g) % g, rs // (g * g)), "got", got[r], "ref", ref[r])
    if len(bad):
        rs = (n - 1 - bad) if upper else bad
        for nm, arr in (("i", rs % g), ("j", (rs // g) % g), ("k", rs // (g * g))):
            print("   bad rows by", nm, np.bincount(arr, minlength=g).tolist())
        # first failing row in solve order and its inputs
        r = bad[np.argmin(rs)]
        print("   first bad (solve order)", rs.min(), "got", got[r], "ref", ref[r])
