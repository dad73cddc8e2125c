"""Phase timeline of one k_arnoldi2 launch (Arnoldi step j) on config 2:
per pass, when CTAs start computing (v_i's buffer ready), finish, add their
sums and leave the grid barrier (globaltimer ns, igm_debug_arn_ts).

    python scripts/arn_ts.py [j] [grid]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2009_07495_b200 as igm  # noqa: E402
from paper_2009_07495_b200 import lib  # noqa: E402

j = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rp, ci, v, bh = bench.config2(g)
S, A, F, b, lower, upper, _ = bench.setup_b200(rp, ci, v, bh)
cfg = bench.solve_cfg(igm, max_ref=1)
igm.solve(S, A, b, cfg, precond=F)  # warm
slots = lib().igm_debug_arn_ts(j, None, 0)
igm.solve(S, A, b, cfg, precond=F)
G = 148
buf = (C.c_ulonglong * (G * slots))()
lib().igm_debug_arn_ts(j, buf, G * slots)
t = np.frombuffer(buf, dtype=np.uint64).reshape(G, slots).astype(np.int64)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 124].min()
rel = lambda col: (t[:, col] - t0) / 1e3  # us
print(f"step j={j}, {live.sum()} CTAs; times in us from the first CTA's start")
print(f"{'pass':>4} {'ready min/max':>16} {'comp.end min/max':>18} {'added max':>10} {'barrier min/max':>16}  "
      f"compute  reduce  barrier-wait  buffer-wait")
prev_bar = None
for i in range(j + 1):
    r0, c1, a2, b3 = rel(4 * i), rel(4 * i + 1), rel(4 * i + 2), rel(4 * i + 3)
    comp = np.median(c1 - r0)
    red = np.median(a2 - c1)
    bw = np.median(b3 - a2)
    buf_wait = np.median(r0 - prev_bar) if prev_bar is not None else float("nan")
    print(f"{i:4d} {r0.min():7.2f}/{r0.max():7.2f} {c1.min():8.2f}/{c1.max():8.2f} {a2.max():10.2f} "
          f"{b3.min():7.2f}/{b3.max():7.2f}  {comp:7.2f} {red:7.2f} {bw:12.2f} {buf_wait:12.2f}")
    prev_bar = b3
i = j + 1
c1, a2 = rel(4 * j + 5), rel(4 * j + 6)
print(f"norm pass: computed max {c1.max():.2f}, added max {a2.max():.2f}")
for k, name in ((120, "barrier before the scalar step"), (121, "scalar step done"), (122, "div barrier"),
                (125, "vec_div operands read"), (127, "vec_div rows written once"), (126, "vec_div rows written"), (123, "vec_div done")):
    x = rel(k)
    print(f"{name:32s} min {x.min():8.2f} max {x.max():8.2f}")
c = t[0, 100:111].tolist()
print("scalar step stamps (CTA 0, clock64 cycles from entry):", [x - c[0] if x else None for x in c])
