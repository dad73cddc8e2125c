"""Time igm_norm2 (exact sequential FP64 chain, K8) on device-resident vectors
of config-2 size with different value distributions."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2009_07495_b200 as igm

n = 2097152
rng = np.random.default_rng(1)
dev = igm.Device(0)
cases = {
    "normal": rng.standard_normal(n),
    "uniform": rng.uniform(-1, 1, n),
    "const": np.full(n, 0.5),
    "tiny-then-big": np.concatenate([np.full(1000, 1e-150), rng.standard_normal(n - 1000)]),
}
for name, x in cases.items():
    t = torch.tensor(x, device="cuda")
    igm.norm2(t, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        r = igm.norm2(t, dev)
    e1.record()
    torch.cuda.synchronize()
    ref = 0.0
    print(f"{name:14s} {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us/call  value {r!r}")
