"""Debug: structured multi-brick ILU apply vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2009_07495_b200 import _capi
if os.environ.get("LIBNAME"):
    _capi.LIB_PATH = _capi._HERE / os.environ["LIBNAME"]
import paper_2009_07495_b200 as igm
from workloads import gen
from oracle.ffi import Oracle
dims = tuple(int(x) for x in os.environ.get("DIMS", "16,16,128").split(","))
offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
coef = {0: -1.3, 1: -1.2, 2: -1.1, 3: 8.0, 4: -0.9, 5: -0.8, 6: -0.7}
rp, ci, v = gen._stencil_csr(dims, offs, lambda o, r: np.full(r.shape, coef[o]))
vals, _ = igm.row_scale(rp, ci, v, 32)
lo, up = igm.factorize_split_cast(rp, ci, vals)
n = len(rp) - 1
ident = (np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.ones(n, np.int64),
         np.arange(n, dtype=np.int32))
which = os.environ.get("WHICH", "both")
if which == "lower":
    up = ident
elif which == "upper":
    lo = ident
elif which == "ident":
    lo, up = ident, ident
F = igm.IluFactors(lo, up)
print("lower", F.schedule_info(False), flush=True)
n = len(rp) - 1
y = gen.uniform_int(7, n, -(1 << 45), 1 << 45)
orc = Oracle()
il = orc.ilu(lo, up)
want = orc.apply_inverse(il, y)
for rep in range(3):
    got = igm.apply_inverse(F, y)
    bad = np.nonzero(got != want)[0]
    print("rep", rep, "mismatches", len(bad), "first", bad[:10], flush=True)
    if len(bad) and os.environ.get("SHOW"):
        for r in bad[:4]:
            print("   row", r, "got", int(got[r]), "want", int(want[r]), "diff", int(got[r]) - int(want[r]))
