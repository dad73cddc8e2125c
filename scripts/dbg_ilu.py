"""Debug: multi-tile ILU apply vs the oracle (row-level mismatch report)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2009_07495_b200 import _capi
if os.environ.get("LIBNAME"):
    _capi.LIB_PATH = _capi._HERE / os.environ["LIBNAME"]
import paper_2009_07495_b200 as igm
from tests.cases import build_case
from oracle.ffi import Oracle
orc = Oracle()
c = build_case(os.environ.get("CASE", "ilu_random"), orc)
F = igm.IluFactors(c["lower"], c["upper"])
print("lower", F.schedule_info(False), "upper", F.schedule_info(True))
y = c["y_int"]
want = orc.apply_inverse(c["il"], y)
for rep in range(3):
    got = igm.apply_inverse(F, y)
    bad = np.nonzero(got != want)[0]
    print("rep", rep, "mismatches", len(bad), "first", bad[:20])
