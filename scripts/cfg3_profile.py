import sys, os, json
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2009_07495_b200 as igm
from paper_2009_07495_b200._capi import KCLASS_NAMES
from workloads import gen
dev = igm.Device(0); igm.Device._default = dev
n = 1_000_000
rp, ci, v = gen.random_band_fast(n, gen.SEED_BASE ^ 3)
bh = gen.uniform(gen.SEED_BASE ^ 103, n)
vals, scale = igm.row_scale_device(rp, ci, v, 16)
comp, al, _ = igm.build_split_device(vals, 16, 1)
b = bh / np.asarray(scale)
S = igm.SplitMatrix(rp, ci, comp, al); A = igm.CsrMatrixF(rp, ci, vals)
db = torch.from_numpy(b).cuda(); dx = torch.empty(n, dtype=torch.float64, device="cuda")
cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=50, frac_bits=30, shifts=igm.ShiftPlan.default_unpreconditioned(30), checked=True)
igm.solve(S, A, db, cfg, x_out=dx)
igm.lib().igm_profile_enable(1)
_, rep = igm.solve(S, A, db, cfg, x_out=dx)
igm.lib().igm_profile_enable(0)
kms = np.zeros(11); kcnt = np.zeros(11, dtype=np.uint64)
igm.lib().igm_profile_collect(kms.ctypes.data_as(igm._capi.f64p), kcnt.ctypes.data_as(igm._capi.u64p))
print("iters", rep.total_inner_iterations, "nnz", int(rp[-1]), "maxrow", int(np.diff(rp).max()))
print({KCLASS_NAMES[i]: (round(float(kms[i]),3), int(kcnt[i])) for i in range(11) if kcnt[i]})
