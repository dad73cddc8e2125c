"""Run the cfg2 integer ILU apply a few times (ncu target)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2009_07495_b200 as igm
from workloads import gen
g = int(os.environ.get("GRID", "128"))
rp, ci, v = gen.upwind_3d(g, 20.0)
vals, scale = igm.row_scale(rp, ci, v, 32)
lo, up = igm.factorize_split_cast(rp, ci, vals)
F = igm.IluFactors(lo, up)
n = len(rp) - 1
import torch
y = torch.from_numpy(gen.uniform_int(7, n, -(1 << 45), 1 << 45)).cuda()
reps = int(os.environ.get("REPS", "3"))
for _ in range(reps):
    z = igm.apply_inverse(F, y)
torch.cuda.synchronize()
t0 = time.time()
for _ in range(reps):
    z = igm.apply_inverse(F, y)
torch.cuda.synchronize()
print("apply_inverse ms", (time.time() - t0) / reps * 1e3, "levels", F.levels(False))
