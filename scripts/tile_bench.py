"""Per-level cost of the ILU wavefront in ONE tile (16x16x64 brick, 94 levels)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07495_b200 import _capi
if os.environ.get("SKEL"):
    _capi.LIB_PATH = _capi._HERE / "libigm_skel.so"
if os.environ.get("LIBNAME"):
    _capi.LIB_PATH = _capi._HERE / os.environ["LIBNAME"]
import numpy as np, torch
import paper_2009_07495_b200 as igm
from workloads import gen
dims = tuple(int(x) for x in os.environ.get("DIMS", "16,16,64").split(","))
h = 1.0 / 129
offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
coef = {0: -1 / h**2 - 20 / h, 1: -1 / h**2 - 20 / h, 2: -1 / h**2 - 20 / h, 3: 6 / h**2 + 60 / h,
        4: -1 / h**2, 5: -1 / h**2, 6: -1 / h**2}
if os.environ.get("KIND") == "27":
    assert dims[0] == dims[1] == dims[2]
    rp, ci, v = gen.stencil27_lean(dims[0], 5)
else:
    rp, ci, v = gen._stencil_csr(dims, offs, lambda o, r: np.full(r.shape, coef[o]))
vals, _ = igm.row_scale(rp, ci, v, 32)
lo, up = igm.factorize_split_cast(rp, ci, vals)
F = igm.IluFactors(lo, up)
n = len(rp) - 1
y = torch.from_numpy(gen.uniform_int(7, n, -(1 << 45), 1 << 45)).cuda()
z = torch.empty(n, dtype=torch.int64, device="cuda")
dev = igm.Device.default()
lib = igm.lib()
import ctypes as C
def run():
    lib.igm_apply_inverse(dev.h, F.h, C.c_void_p(y.data_ptr()), C.c_void_p(z.data_ptr()), None)
for _ in range(5): run()
torch.cuda.synchronize()
R = 200
t0 = time.time()
for _ in range(R): run()
torch.cuda.synchronize()
dt = (time.time() - t0) / R
info = F.schedule_info(False)
L = info["levels"]
print(f"kind {os.environ.get('KIND','7')} brick {info['brick']} dims {dims} tiles {info['tiles']} levels {L}: apply {dt*1e6:.1f} us -> {dt*1e6/(2*L):.3f} us/level (fwd+bwd, incl. launch)")
