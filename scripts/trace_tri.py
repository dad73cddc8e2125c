import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2009_07495_b200 import _capi
if os.environ.get('LIBNAME'):
    _capi.LIB_PATH = _capi._HERE / os.environ['LIBNAME']
import paper_2009_07495_b200 as igm
from workloads import gen
dims = tuple(int(x) for x in os.environ.get("DIMS", "128,128,128").split(","))
if len(set(dims)) == 1:
    rp, ci, v = gen.upwind_3d(dims[0], 20.0)
else:
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    coef = {0: -1.3, 1: -1.2, 2: -1.1, 3: 8.0, 4: -0.9, 5: -0.8, 6: -0.7}
    rp, ci, v = gen._stencil_csr(dims, offs, lambda o, r: np.full(r.shape, coef[o]))
vals, scale = igm.row_scale(rp, ci, v, 32)
lo, up = igm.factorize_split_cast(rp, ci, vals)
F = igm.IluFactors(lo, up)
n = len(rp) - 1
print("fwd", F.schedule_info(False))
y = torch.from_numpy(gen.uniform_int(7, n, -(1 << 45), 1 << 45)).cuda()
z = igm.apply_inverse(F, y)
buf = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
lib = igm.lib()
names = ["poll0", "poll1", "c_presync", "c_postsync", "c_done", "pub_sync", "pub_done"]
tiles = [int(x) for x in os.environ.get("TILES", "0,1,9,63,127").split(",")]
for tile in tiles:
    buf.zero_()
    lib.igm_debug_tri_trace(tile, C.c_void_p(buf.data_ptr()))
    z = igm.apply_inverse(F, y)
    torch.cuda.synchronize()
    raw = buf.cpu().numpy().reshape(-1, 8)
    nst, next_ = raw[:, 0].sum(), raw[:, 1].sum()
    ts = raw[:, :8].astype(np.float64)
    ts = ts[ts[:, 3] > 0]
    t0 = ts[:, 2:8][ts[:, 2:8] > 0].min()
    ts -= t0
    ts /= 1.9  # cycles -> ns at ~1.9 GHz
    print(f"  cross-tile words used {next_}, stale at use {nst}")
    print(f"tile {tile}: segs {len(ts)} start {ts[0,3]/1e3:.1f}us end {ts[-1,4]/1e3:.1f}us")
    per = np.diff(ts[:, 3])
    print("  level period med %.0f mean %.0f ns | barrier wait %.0f | row %.0f | syncwarp+arrive %.0f | prefetch next %.0f" % (
        np.median(per), per.mean(), np.median(ts[:, 3] - ts[:, 2]), np.median(ts[:, 5] - ts[:, 3]),
        np.median(ts[:, 6] - ts[:, 5]), np.median(ts[:, 4] - ts[:, 6])))
    lead = ts[1:, 2] - ts[1:, 7]   # compute reaches level q  minus  loader issued level q
    print("  loader lead over compute: med %.0f ns, min %.0f; loader period med %.0f ns" % (
        np.median(lead), lead.min(), np.median(np.diff(ts[:, 7]))))
    for r in ts[5:8]:
        print("   ", " ".join(f"{x/1e3:8.2f}" for x in r))
lib.igm_debug_tri_trace(-1, None)
