"""Integer SpMV variants on a 27-point (config-4 family) or 7-point (config-2
family) matrix: one thread per row over CSR, the staged long-row kernel and
the sliced-ELL kernel (IGM_SPMV_STAGED / IGM_SPMV_SELL), timed with CUDA events through the Python call (adds ~30 us
per call), outputs compared by hash.

    python scripts/spmv27_bench.py [grid] [checked] [27|7]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 4:  # child: one mode
    import numpy as np
    import torch
    import paper_2009_07495_b200 as igm
    from workloads import gen
    g, checked = int(sys.argv[1]), int(sys.argv[2])
    rp, ci, v = gen.stencil27_rows(g, 5, 0, g) if sys.argv[3] == "27" else gen.upwind_3d_rows(g, 20.0, 0, g)
    n, nnz = len(rp) - 1, int(rp[-1])
    vals, _ = igm.row_scale_device(rp, ci, v, 32)
    comp, al, _ = igm.build_split_device(vals, 32, 1)
    S = igm.SplitMatrix(rp, ci, comp, al)
    x = torch.from_numpy(gen.uniform_int(7, n, -(1 << 30), 1 << 30)).cuda()
    dev = igm.Device.default()
    tr = igm.FxTrace(checked=bool(checked)) if checked else None
    for _ in range(3):
        out = igm.spmv(S, 0, x, trace=tr)
    st = torch.cuda.ExternalStream(dev.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        out = igm.spmv(S, 0, x, trace=tr)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    b = 12 * nnz + 4 * (n + 1) + 16 * n
    import hashlib
    print(f"sell={os.environ.get('IGM_SPMV_SELL', '1')} staged={os.environ.get('IGM_SPMV_STAGED', '1')} "
          f"{sys.argv[3]}-pt g={g} checked={checked}: {ms * 1e3:.1f} us, "
          f"{b / ms / 1e6:.0f} GB/s, sha {hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]}")
else:
    g = sys.argv[1] if len(sys.argv) > 1 else "160"
    chk = sys.argv[2] if len(sys.argv) > 2 else "1"
    kind = sys.argv[3] if len(sys.argv) > 3 else "27"
    for sell, staged in (("0", "0"), ("0", "1"), ("1", "1")):
        subprocess.run([sys.executable, __file__, g, chk, kind, "child"],
                       env=dict(os.environ, IGM_SPMV_SELL=sell, IGM_SPMV_STAGED=staged), check=True)
