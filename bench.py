#!/usr/bin/env python
"""bench.py -- int-GMRES on one B200 (BASELINE.json metric, config 2 by default).

Workload (BASELINE.json configs[1]): 3D 7-point upwind convection-diffusion on
a 128^3 grid (n = 2,097,152, nnz = 14,581,760), beta = (20,20,20), b = A x*
with x* ~ U[-1,1) (seeded SplitMix64), alpha_a = 32, integer ILU(0), Q33.30,
preconditioned shift preset, GMRES(30), FP64 iterative refinement to 1e-10,
checked mode (the reference's default).  One step = one full solve from x = 0.

  value     = inner int-GMRES iterations / s over K timed solves, b and x
              resident in HBM (CUDA events on the library's stream)
  e2e       = the same through the public API with pinned HOST b / x: the
              H2D of b and the D2H of x are inside the timed region
  roofline  = the dominant kernel class of an instrumented solve, algorithmic
              bytes / its summed launch time vs measured HBM
  cpu_baseline = the reference library (oracle/_ref, built from
              /root/reference) on this host, one refinement cycle, 1 thread

``--impl reference`` times the reference's own CPU solver on the same config
(one refinement cycle = 30 iterations per step).

For N > 1 (torchrun) the bench runs the PARTITIONED configs instead of
replicas: value = iterations/s of ONE BASELINE config-4 solve (256^3 27-point
+ ILU(0)) row-block partitioned over the N GPUs (dist.solve_sharded: slab-
local setup, halo planes over NCCL P2P, per-pass sums through the library's
P2P mailboxes, global ILU hand-offs, x hashed against the reference golden),
scaling = strong, and kernel_microbench = the config-5 call on N GPUs.  The
1-GPU figure of that workload: `--gpus 1 --cfg4-sharded`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import gen  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- workload
def config2(g: int = 128):
    rp, ci, v = gen.upwind_3d(g, 20.0)
    n = len(rp) - 1
    xs = gen.uniform(gen.SEED_BASE ^ 2, n)
    bh = gen.spmv_np(rp, ci, v, xs)
    return rp, ci, v, bh


def setup_b200(rp, ci, v, bh, alpha=32):
    import paper_2009_07495_b200 as igm
    t0 = time.time()
    # device-side setup (bit-identical to the host code)
    vals, scale = igm.row_scale_device(rp, ci, v, alpha)
    b = bh / scale
    comp, al, _ = igm.build_split_device(vals, alpha, 1)
    lower, upper = igm.factorize_split_cast_device(rp, ci, vals)
    setup_s = time.time() - t0
    S = igm.SplitMatrix(rp, ci, comp, al)
    A = igm.CsrMatrixF(rp, ci, vals)
    F = igm.IluFactors(lower, upper)
    return S, A, F, b, lower, upper, setup_s


def solve_cfg(igm, tol=1e-10, m=30, max_ref=1000):
    return igm.RefineConfig(tol=tol, max_refinements=max_ref, m=m, frac_bits=30,
                            shifts=igm.ShiftPlan.default_preconditioned(30), s=0, checked=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- helpers
def peaks():
    try:
        with open(MEASURED) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return ws, rank, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def algorithmic_bytes(n, nnz, nnz_l, nnz_u, m_steps_dims, W=8):
    """SURVEY.md 8(d) per-class algorithmic bytes for one solve."""
    spmv = (W + 4) * nnz + 4 * (n + 1) + 2 * W * n
    ilu = (W + 4) * (nnz_l + nnz_u) + 8 * (n + 1) + 4 * W * n
    # MGS passes at step j: pass 0 (read w, v0), j fused passes (w, v_{i-1},
    # v_i read, w write), tail (w, v_j read, w write): (4j+5) W n
    mgs = sum((4 * j + 5) * W * n for dims in m_steps_dims for j in range(dims))
    # what k_arnoldi moves: the j+1 basis vectors and w read once, v_{j+1} written
    mgs_actual = sum((j + 3) * W * n for dims in m_steps_dims for j in range(dims))
    steps = sum(m_steps_dims)
    return {"spmv_int": spmv * steps, "ilu_int": ilu * steps, "mgs": mgs, "mgs_actual": mgs_actual,
            "vec_div": 2 * W * n * steps}


# ----------------------------------------------------------------- reference arm
def reference_solver():
    from oracle import ffi
    if ffi.ref_available():
        return ffi.Reference(), "reference"
    return ffi.Oracle(), "port"


def ref_setup(B, rp, ci, v, bh, alpha=32):
    A = B.csrf(rp, ci, v)
    vals, scale = B.row_scale(A, alpha)
    As = B.csrf(rp, ci, vals)
    b = bh / scale
    if isinstance(B, __import__("oracle.ffi", fromlist=["Reference"]).Reference):
        comp, al, _ = B.build_split(As, alpha, 1)
    else:
        comp, al, _ = B.build_split(vals, alpha, 1)
    sp = B.split(rp, ci, comp, al)
    lo, up = B.factorize_split_cast(As)
    il = B.ilu(lo, up)
    return sp, As, b, il


def ref_cycle(B, sp, As, b, il, max_ref=1, m=30):
    from oracle.ffi import Shifts
    x, rep = B.solve(sp, As, b, 1e-10, max_ref, m, 30, 0, Shifts(0, 0, 0, 0, 30, 0, 0, 0), checked=True,
                     precond=il)
    return rep


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


class pinned_core:
    """Pin this process to one host core (taskset equivalent) for a CPU sample."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = max(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def cpu_sample(rp, ci, v, bh):
    B, kind = reference_solver()
    sp, As, b, il = ref_setup(B, rp, ci, v, bh)
    with pinned_core() as pc:
        rep = ref_cycle(B, sp, As, b, il, 1)
    its = rep["total_inner_iterations"]
    model, total = host_cpu()
    return {"value": its / rep["wall_time_sec"], "unit": "iters/s", "cores": 1, "kind": kind,
            "host_cpu": model, "host_cores_total": total, "pinned_core": pc.core,
            "sample": f"1 refinement cycle ({its} int-GMRES iterations) of the config-2 solve, "
                      f"checked mode, single thread pinned to core {pc.core} (the reference has no "
                      f"threading); {rep['wall_time_sec']:.2f} s"}


def run_reference_cfg4(args):
    """The reference arm of `--gpus N > 1`: the B200 arm then runs config 4
    (run_b200_sharded), so the reference's own CPU solver is timed on the same
    system.  A whole config-4 solve takes the reference ~220 s, so each step
    is a bounded sample: one refinement cycle of GMRES(4) (4 inner iterations:
    SpMV + ILU(0) apply + MGS each; the MGS share is smaller than in a
    GMRES(30) cycle, which flatters the reference by ~15 %)."""
    g = args.cfg4_grid
    t0 = time.time()
    rp, ci, v = gen.stencil27_lean(g, gen.SEED_BASE ^ 4)
    n = len(rp) - 1
    bh = gen.spmv_np(rp, ci, v, gen.uniform(gen.SEED_BASE ^ 104, n))
    B, kind = reference_solver()
    sp, As, b, il = ref_setup(B, rp, ci, v, bh)
    del v, bh
    log(f"[bench] reference arm, config 4 at {g}^3: setup {time.time() - t0:.0f} s")
    m = 4
    for _ in range(args.warmup):
        ref_cycle(B, sp, As, b, il, 1, m)
    t, its = 0.0, 0
    for _ in range(args.steps):
        rep = ref_cycle(B, sp, As, b, il, 1, m)
        t += rep["wall_time_sec"]
        its += rep["total_inner_iterations"]
    val = its / t
    line = {"impl": "reference", "metric": "int-GMRES iters/s", "value": val, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded SplitMix64)",
            "config": {"workload": f"cfg4: 3D 27-pt {g}^3 (n={n}), integer ILU(0), GMRES(30), FP64 refinement to "
                                   f"1e-10, Q33.30, checked",
                       "step": f"one refinement cycle of GMRES({m}) ({m} inner iterations) of the reference solver"},
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": 1, "kind": kind,
                             "host_cpu": host_cpu()[0], "host_cores_total": host_cpu()[1],
                             "sample": f"each step = 1 refinement cycle of GMRES({m}) on the config-4 system; the "
                                       f"reference is single-threaded (no threads / OpenMP in proj/core)"},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    if ws > 1:
        return run_reference_cfg4(args)
    rp, ci, v, bh = config2(args.grid)
    B, kind = reference_solver()
    sp, As, b, il = ref_setup(B, rp, ci, v, bh)
    for _ in range(args.warmup):
        ref_cycle(B, sp, As, b, il, 1)
    t = 0.0
    its = 0
    for _ in range(args.steps):
        rep = ref_cycle(B, sp, As, b, il, 1)
        t += rep["wall_time_sec"]
        its += rep["total_inner_iterations"]
    val = its / t
    line = {"impl": "reference", "metric": "int-GMRES iters/s", "value": val, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded SplitMix64)",
            "config": {"workload": f"cfg2: 3D 7-pt upwind CD {args.grid}^3, ILU(0), GMRES(30), tol 1e-10",
                       "step": "one refinement cycle (30 iterations) of the reference solver"},
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": 1, "kind": kind,
                             "host_cpu": host_cpu()[0], "host_cores_total": host_cpu()[1],
                             "sample": "each step = 1 refinement cycle of the config-2 solve; the reference "
                                       "is single-threaded (no threads / OpenMP in proj/core)"},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- config 5
def run_cfg5(args, igm, dev, local, g=400, k=30):
    """BASELINE.json configs[4]: 400^3 7-pt operator (alpha_a = 16, A_0 only),
    one call = w = spmv(A, 0, v_30) then MGS of w against 30 int64 vectors
    uniform in [-2^40, 2^40) (dot b1=16, b2=0; axpy b1=16), unchecked."""
    import torch
    t0 = time.time()
    rp, ci, v = gen.upwind_3d_lean(g, 20.0)
    vals, _ = igm.row_scale(rp, ci, v, 16)
    del v
    comp, al, _ = igm.build_split(vals, 16, 1)
    del vals
    n, nnz = len(rp) - 1, int(rp[-1])
    S = igm.SplitMatrix(rp, ci, comp, al, device=dev)
    del comp, rp, ci
    dvc = f"cuda:{local}"
    seed = gen.SEED_BASE ^ 5
    basis = torch.empty((k, n), dtype=torch.int64, device=dvc)
    for i in range(k):
        basis[i] = gen.device_uniform_int40(n, seed, (i + 1) * n, dvc)
    vin = gen.device_uniform_int40(n, seed, 0, dvc)
    w = torch.empty(n, dtype=torch.int64, device=dvc)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    stream = torch.cuda.ExternalStream(dev.stream, device=dvc)
    for _ in range(max(args.warmup, 1)):
        igm.spmv_mgs(S, 0, vin, basis, k, 30, 16, 0, 16, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        igm.spmv_mgs(S, 0, vin, basis, k, 30, 16, 0, 16, w)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    igm.lib().igm_profile_enable(1)
    igm.spmv_mgs(S, 0, vin, basis, k, 30, 16, 0, 16, w)
    igm.lib().igm_profile_enable(0)
    kms = np.zeros(11)
    kcnt = np.zeros(11, dtype=np.uint64)
    igm.lib().igm_profile_collect(kms.ctypes.data_as(igm._capi.f64p), kcnt.ctypes.data_as(igm._capi.u64p))
    b_spmv = 12 * nnz + 4 * (n + 1) + 16 * n
    b_mgs = (4 * k + 1) * 8 * n
    hbm, src = peaks()
    mgs_gbs = b_mgs / (kms[3] / 1e3) / 1e9
    spmv_gbs = b_spmv / (kms[0] / 1e3) / 1e9
    call_gbs = (b_spmv + b_mgs) / (ms / 1e3) / 1e9
    del S, basis, vin, w
    torch.cuda.empty_cache()
    return {
        "workload": f"cfg5: SpMV (400^3 7-pt, alpha 16, s=0; n={n}, nnz={nnz}) + MGS against {k} int64 "
                    "vectors uniform in [-2^40,2^40), unchecked",
        "ms_per_call": ms, "bytes_per_call": b_spmv + b_mgs, "GB/s": round(call_gbs, 1),
        "frac": round(call_gbs / hbm, 4), "peak": hbm, "peak_source": src,
        "spmv": {"ms": round(float(kms[0]), 4), "GB/s": round(spmv_gbs, 1), "frac": round(spmv_gbs / hbm, 4),
                 "note": "read-dominated stream (sliced-ELL copy at this size): the denominator is the measured COPY "
                         "bandwidth (reads + writes), which a read-only stream can exceed"},
        "mgs": {"ms": round(float(kms[3]), 4), "launches": int(kcnt[3]), "GB/s": round(mgs_gbs, 1),
                "frac": round(mgs_gbs / hbm, 4), "bytes": b_mgs},
        "setup_s": round(setup_s, 1), "l2": "vectors 512 MB each, far larger than L2",
    }


def run_cfg5_sharded(args, igm, dev, local, rank, ws, g=400, k=30):
    """Config 5 row-block partitioned over the ws GPUs: each
    rank owns 400/ws z-planes (its slab of the operator, built locally), the
    SpMV input's boundary planes move to the neighbours (NCCL P2P), and each
    of the k MGS passes all-reduces one int64 accumulator (exact).  Strong
    scaling: the global problem is the 1-GPU config-5 call, word for word
    (vectors are drawn by global row index)."""
    import torch
    import torch.distributed as dist
    from paper_2009_07495_b200 import dist as D
    t0 = time.time()
    sl = D.make_slab(g, g * g, rank, ws)
    rp, ci, v, h0, own0, own1 = gen.upwind_3d_slab(g, 20.0, sl.z0, sl.z1)
    assert (h0, own0, own1) == (sl.h0, sl.own0, sl.own1)
    vals, _ = igm.row_scale(rp, ci, v, 16)
    del v
    comp, al, _ = igm.build_split(vals, 16, 1)
    del vals
    nnz_local = int(rp[-1])
    be = D.CudaSlabBackend(igm, dev)
    S = be.upload(rp, ci, comp, al)
    del comp, rp, ci
    dvc = f"cuda:{local}"
    n = g ** 3
    seed = gen.SEED_BASE ^ 5
    g0, g1 = sl.global_rows
    basis = torch.empty((k, sl.n_own), dtype=torch.int64, device=dvc)
    for i in range(k):
        basis[i] = gen.device_uniform_int40(sl.n_own, seed, (i + 1) * n + g0, dvc)
    vown = gen.device_uniform_int40(sl.n_own, seed, g0, dvc)
    work = dict(vext=torch.zeros(sl.next_, dtype=torch.int64, device=dvc),
                wext=torch.zeros(sl.next_, dtype=torch.int64, device=dvc),
                acc=torch.zeros(k, dtype=torch.int64, device=dvc))
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    call = lambda: D.spmv_mgs_sharded(be, sl, S, 0, vown, basis, k, 30, 16, 0, 16, dist, work)
    for _ in range(max(args.warmup, 1)):
        call()
    torch.cuda.synchronize()
    barrier(ws)
    stream = torch.cuda.ExternalStream(dev.stream, device=dvc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        call()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
    # global checksum of w and the h's: identical at every world size
    w, acc = call()
    torch.cuda.synchronize()
    wsum = torch.tensor([int(w.sum().item()) & ((1 << 63) - 1)], dtype=torch.int64, device=dvc)
    if ws > 1:
        dist.all_reduce(wsum)
    nnz = 7 * n - 6 * g * g
    b_spmv = 12 * nnz + 4 * (n + 1) + 16 * n
    b_mgs = (4 * k + 1) * 8 * n
    hbm, src = peaks()
    gbs = (b_spmv + b_mgs) / (ms / 1e3) / 1e9
    del S, basis, vown, work
    torch.cuda.empty_cache()
    return {
        "workload": f"cfg5 sharded: z-slabs of {g}^3 over {ws} GPU(s) ({sl.z1 - sl.z0} planes on rank {rank}), "
                    f"halo exchange (NCCL P2P) + per-pass int64 allreduce; SpMV + MGS against {k} vectors",
        "parallelism": f"z-slab x{ws}", "scaling": "strong", "ms_per_call": round(ms, 4),
        "bytes_per_call": b_spmv + b_mgs, "GB/s": round(gbs, 1), "GB/s_per_gpu": round(gbs / ws, 1),
        "frac_per_gpu": round(gbs / ws / hbm, 4), "peak": hbm, "peak_source": src,
        "h_acc_checksum": [int(x) for x in acc.cpu().tolist()][:3], "w_checksum_low63": int(wsum.item()),
        "rank0_local_nnz": nnz_local, "setup_s": round(setup_s, 1),
    }


def run_cfg4_sharded(args, igm, dev, local, rank, ws, g=256, m=30):
    """BASELINE config 4 (g^3 27-point + integer ILU(0), GMRES(30), refinement
    to 1e-10, checked) as ONE solve row-block partitioned over the ws GPUs
    (dist.solve_sharded): every rank builds its own planes only
    (plane-range generator, device row scaling / truncation layer, the ILU(0)
    plane relay -- dist.setup_slab_local), per step the halo planes move over
    NCCL P2P, the MGS / norm accumulators are summed through the library's
    P2P mailboxes (igm_mbox_*), the integer substitutions of the GLOBAL
    factors stream their boundary planes to the next rank pencil by pencil
    (dist.ZPipe, igm_dc_tri_piped: the 27-point wavefront's PIPE variant),
    norm2 is one rank-ordered FP64 chain.  Strong scaling: the global problem is the 1-GPU
    config, and the gathered x (every word) is hashed against the reference
    library's whole-solve golden at g = 256."""
    import hashlib
    import torch
    import torch.distributed as dist
    from paper_2009_07495_b200 import dist as D
    t0 = time.time()
    dvc = f"cuda:{local}"
    sl = D.make_slab(g, g * g, rank, ws)
    be = D.CudaSlabBackend(igm, dev)
    comm = D._Comm(sl, dist, be=be)
    seed = gen.SEED_BASE ^ 4
    rows_fn = lambda z0, z1: gen.stencil27_rows(g, seed, z0, z1)
    mats = D.setup_slab_local(be, sl, rows_fn, 32, comm, ilu=True)
    rp, ci_loc, _ = mats["rows"]
    _, _, v_own = rows_fn(sl.z0, sl.z1)  # unscaled rows: b = (A x*) / scale, the goldens' order
    n = g ** 3
    xs = gen.uniform(gen.SEED_BASE ^ 104, sl.next_, offset=sl.h0)
    b_own = gen.spmv_np(rp, ci_loc, v_own, xs) / mats["scale"]
    nnz_local = int(rp[-1])
    del v_own, xs
    mats.pop("rows")
    hb = torch.from_numpy(b_own).pin_memory()
    d_b = hb.to(dvc)
    cfg = igm.RefineConfig(tol=1e-10, max_refinements=100, m=m, frac_bits=30,
                           shifts=igm.ShiftPlan.default_preconditioned(30), checked=True)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    x, rep = None, None
    for _ in range(max(args.warmup, 1)):
        x, rep = D.solve_sharded(be, sl, mats, d_b, cfg, dist)
    stream = torch.cuda.ExternalStream(dev.stream, device=dvc)
    torch.cuda.synchronize()
    barrier(ws)
    l0 = dev.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            x, rep = D.solve_sharded(be, sl, mats, d_b, cfg, dist)
            its += rep.total_inner_iterations
        e1.record(stream)
        torch.cuda.synchronize()
    launches = dev.launches - l0
    ms = max_over_ranks(e0.elapsed_time(e1), ws)
    # e2e: the rank's rows of b from pinned host memory in, its rows of x out, per step
    hx = torch.empty(sl.n_own, dtype=torch.float64).pin_memory()
    barrier(ws)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_its = 0
    f0.record(stream)
    for _ in range(args.steps):
        with be.stream():
            d_b.copy_(hb, non_blocking=True)
        x, r2 = D.solve_sharded(be, sl, mats, d_b, cfg, dist)
        with be.stream():
            hx.copy_(x, non_blocking=True)
        e2e_its += r2.total_inner_iterations
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), ws)
    # the global x on rank 0, hashed against the reference's whole solve
    x_own = x.contiguous()
    parity = {"parity": None}
    if ws > 1:
        if rank == 0:
            parts = [x_own.cpu().numpy()]
            for r in range(1, ws):
                z0, z1 = D.plane_split(g, ws)[r]
                t = torch.empty((z1 - z0) * g * g, dtype=torch.float64, device=dvc)
                dist.recv(t, r)
                parts.append(t.cpu().numpy())
            xg = np.concatenate(parts)
        else:
            dist.send(x_own, 0)
            xg = None
    else:
        xg = x_own.cpu().numpy()
    if xg is not None:
        xh = hashlib.sha256(np.ascontiguousarray(xg).tobytes()).hexdigest()
        parity = {"parity": None, "x_sha256": xh[:16], "why": "goldens exist for g = 256 only"}
        try:
            with open(os.path.join(ROOT, "tests", "golden", "full_goldens.json")) as f:
                gold = json.load(f)["cfg4"]
            if g == gold["g"]:
                r = gold["solve"]["report"]
                same = (rep.inner_dims == r["inner_dims"] and rep.relres_history == r["relres_history"]
                        and rep.gamma_history == r["gamma_history"] and rep.overflow_total == r["overflow_total"])
                parity = {"parity": bool(xh == gold["solve"]["x"] and same), "x_sha256": xh[:16],
                          "golden_x_sha256": gold["solve"]["x"][:16], "report_equal": bool(same),
                          "against": "reference library whole solve (tests/golden/full_goldens.json cfg4)"}
        except (OSError, KeyError, ValueError) as exc:
            parity["why"] = f"no golden: {exc}"
    del mats, d_b
    torch.cuda.empty_cache()
    return {
        "workload": f"cfg4: 3D 27-pt {g}^3 (n={n}), integer ILU(0), GMRES({m}), FP64 refinement to 1e-10, Q33.30, "
                    f"checked; one solve on z-slabs over {ws} GPU(s) ({sl.z1 - sl.z0} planes on rank {rank})",
        "parallelism": f"z-slab x{ws}", "scaling": "strong",
        "value": its / (ms / 1e3), "unit": "iters/s", "ms_per_solve": ms / args.steps,
        "iterations_per_solve": rep.total_inner_iterations, "refinements": rep.refinements,
        "final_relres": rep.relres_history[-1], "overflows": rep.overflow_total,
        "e2e": {"value": e2e_its / (e2e_ms / 1e3), "unit": "iters/s", "h2d_bytes_per_step": int(8 * n),
                "d2h_bytes_per_step": int(8 * n)},
        "gpu_launches": int(launches), "parity": parity, "clocks": clk.summary(),
        "reductions": "igm_mbox (P2P mailboxes)" if comm.mb is not None else
                      ("none (1 GPU)" if ws == 1 else "torch.distributed all_reduce"),
        "rank0_local_nnz": nnz_local, "setup_s": round(setup_s, 1),
    }


def run_b200_sharded(args, ws, rank, local):
    """--gpus N > 1: the partitioned configs (BASELINE configs 4 and 5), not
    replicas of the 1-GPU config: value = iterations/s of ONE config-4 solve
    on N GPUs (strong scaling), kernel_microbench = the config-5 call on N
    GPUs.  The 1-GPU figure of the same workload: `--gpus 1 --cfg4-sharded`."""
    import paper_2009_07495_b200 as igm
    dev = igm.Device(local)
    igm.Device._default = dev
    c4 = run_cfg4_sharded(args, igm, dev, local, rank, ws, g=args.cfg4_grid)
    log(f"[bench] cfg4 sharded: {c4}")
    micro = None
    if not args.no_cfg5:
        try:
            micro = run_cfg5_sharded(args, igm, dev, local, rank, ws)
        except Exception as exc:
            micro = {"error": repr(exc)}
    if rank == 0:
        line = {
            "metric": "int-GMRES iters/s", "value": c4["value"], "unit": "iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": c4["ms_per_solve"],
            "time_to_solution_s": c4["ms_per_solve"] / 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded SplitMix64 matrix and x*, b = A x*)",
            "config": {"workload": c4["workload"], "refinements": c4["refinements"],
                       "iterations_per_solve": c4["iterations_per_solve"], "final_relres": c4["final_relres"],
                       "overflows": c4["overflows"], "parallelism": c4["parallelism"],
                       "reductions": c4["reductions"],
                       "l2": "inputs larger than L2 (matrix + ILU + basis ~ 19 GB over the ranks)",
                       "note": "N > 1 runs BASELINE config 4 (the partitioned config); the N = 1 default is "
                               "config 2, whose 1-GPU config-4 figure is `--gpus 1 --cfg4-sharded`"},
            "gpu_launches": c4["gpu_launches"], "e2e": c4["e2e"], "parity": c4["parity"],
            "kernel_microbench": micro, "clocks": c4["clocks"],
        }
        print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- e2e_cpp
def run_e2e_cpp(args, rp, ci, v, bh):
    """The drop-in boundary timed as a reference user calls it: build/e2e_cpp
    (scripts/e2e_cpp.cpp, written against include/intgmres/ and linked to
    libigm_b200.so) runs intgmres::solve on config 2 with host std::vector
    containers, b uploaded and x downloaded inside every timed call, the
    operators reused through the verified operator cache.  Its x is hashed
    against the reference golden."""
    import hashlib
    import subprocess
    import tempfile
    exe = os.path.join(ROOT, "build", "e2e_cpp")
    if not os.path.exists(exe):
        return {"error": "build/e2e_cpp not built"}
    with tempfile.TemporaryDirectory() as d:
        np.ascontiguousarray(rp, np.int32).tofile(os.path.join(d, "rp.bin"))
        np.ascontiguousarray(ci, np.int32).tofile(os.path.join(d, "ci.bin"))
        np.ascontiguousarray(v, np.float64).tofile(os.path.join(d, "v.bin"))
        np.ascontiguousarray(bh, np.float64).tofile(os.path.join(d, "bh.bin"))
        xo = os.path.join(d, "x.bin")
        p = subprocess.run([exe, d, str(args.steps), str(max(1, args.warmup)), xo], capture_output=True, text=True,
                           timeout=1200)
        try:
            rec = json.loads(p.stdout.strip().splitlines()[-1])
        except (ValueError, IndexError):
            return {"error": (p.stdout + p.stderr)[-400:]}
        if os.path.exists(xo):
            x = np.fromfile(xo, dtype=np.float64)
            xh = hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()
            try:
                with open(os.path.join(ROOT, "tests", "golden", "full_goldens.json")) as f:
                    gx = json.load(f)["cfg2"]["solve"]["x"]
                rec["parity"] = bool(xh == gx) if args.grid == 128 else None
            except (OSError, KeyError, ValueError):
                rec["parity"] = None
    rec.update({"value": rec.get("iters_per_s"), "unit": "iters/s",
                "call": "intgmres::solve(SplitMatrix, CsrMatrixF, std::vector<double> b, RefineConfig, &IluFactors) "
                        "from C++ (refine.hpp:67-70), host containers in and out"})
    return rec


# ----------------------------------------------------------------- parity
def parity_check(d_x, rep, grid):
    """The timed solve's x (every word) and report against the reference
    library's whole solve of the same system (tests/golden/full_goldens.json,
    made by tests/golden/make_full_goldens.py from oracle/_ref)."""
    import hashlib
    if grid != 128:
        return {"parity": None, "why": "goldens exist for the 128^3 config only"}
    try:
        with open(os.path.join(ROOT, "tests", "golden", "full_goldens.json")) as f:
            g = json.load(f)["cfg2"]["solve"]
    except (OSError, KeyError, ValueError) as exc:
        return {"parity": None, "why": f"no golden: {exc}"}
    x = d_x.cpu().numpy()
    xh = hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()
    r = g["report"]
    same_rep = (rep.inner_dims == r["inner_dims"] and rep.relres_history == r["relres_history"]
                and rep.gamma_history == r["gamma_history"] and rep.overflow_total == r["overflow_total"])
    return {"parity": bool(xh == g["x"] and same_rep), "x_sha256": xh[:16], "golden_x_sha256": g["x"][:16],
            "report_equal": bool(same_rep),
            "against": "reference library whole solve (tests/golden/full_goldens.json cfg2)"}


# ----------------------------------------------------------------- B200 arm
def measured_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture summary (profiles/traffic.json), or None"""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def roofline_line(breakdown, ab, n, levels, ms_step, refinements, hbm, src, micro):
    """The dominant kernel of the headline step: the integer ILU(0)
    substitution (k_tri_pencil, 2 launches per iteration).  achieved = its
    SURVEY.md 8(d) algorithmic bytes per launch / its average launch time
    (CUDA events around each launch on the library's stream, instrumented
    solve); traffic = ncu DRAM bytes per launch (profiles/traffic.json).
    Every other class is listed under `classes` with its own fraction; MGS
    (the persistent k_arnoldi step) is given against both the streaming
    formula and the bytes it actually moves (w stays on chip), and the whole
    cycle against BASELINE.md's 47.744 GB."""
    ilu = breakdown["ilu_int"]
    per_launch_ms = ilu["ms"] / ilu["launches"]
    bytes_launch = ab["ilu_int"] / ilu["launches"]
    achieved = bytes_launch / (per_launch_ms / 1e3) / 1e9
    step_share = ilu["ms"] / ms_step
    classes = {}
    for name in ("mgs", "spmv_int", "ilu_fp", "norm2_serial", "residual_fp", "x_update"):
        if name not in breakdown:
            continue
        e = dict(breakdown[name])
        e["share_of_step"] = round(breakdown[name]["ms"] / ms_step, 4)
        if name in ab:
            gbs = ab[name] / (e["ms"] / 1e3) / 1e9
            e["algorithmic_GB/s"] = round(gbs, 1)
            e["frac"] = round(gbs / hbm, 4)
        classes[name] = e
    if "mgs" in classes and "mgs_actual" in ab:
        classes["mgs"]["kernel"] = "k_arnoldi2 (register-resident w, TMA double-buffered basis slices)"
        gbs = ab["mgs_actual"] / (breakdown["mgs"]["ms"] / 1e3) / 1e9
        classes["mgs"]["actual_bytes_GB/s"] = round(gbs, 1)
        classes["mgs"]["frac_actual_bytes"] = round(gbs / hbm, 4)
        classes["mgs"]["note"] = ("frac uses the streaming formula (4k+3)Wn (SURVEY 8(d)); k_arnoldi keeps w on "
                                  "chip and moves (k+2)Wn per step (ncu: 374 MB at j=20 for k_arnoldi2, profiles/traffic.json), "
                                  "frac_actual_bytes divides those")
    cyc_ms = ms_step / max(1, refinements)
    cycle = {"bytes_per_cycle": 47.744e9, "ms_per_cycle": round(cyc_ms, 3),
             "floor_ms": round(47.744e9 / (hbm * 1e9) * 1e3, 3),
             "frac": round(47.744e9 / (cyc_ms / 1e3) / 1e9 / hbm, 4)}
    return {"bound": "hbm", "kernel": "k_tri_pencil2<checked,int,8> (ILU(0) substitution, warp-specialised pencil "
                                      "wavefront, bricks in 8-CTA clusters)",
            "achieved": round(achieved, 1), "peak": hbm, "peak_source": src, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": measured_traffic("k_tri_pencil2_cfg2"),
            "bytes_per_launch": int(bytes_launch), "us_per_launch": round(per_launch_ms * 1e3, 2),
            "launches_per_step": ilu["launches"], "share_of_step": round(step_share, 4),
            "levels": levels, "us_per_level": round(per_launch_ms * 1e3 / levels, 4),
            "latency_note": "a dependent wavefront of `levels` levels: bounded by per-level latency, "
                            "not by HBM (the 8(d) bytes are reported for comparability)",
            # the bound that does apply: `levels` dependent steps of the row recurrence (two 64-bit
            # shuffles -> three wrapping products -> exact reciprocal division), 240 cycles per step
            # alone in a warp (scripts/step_chain_bench.cu on this GPU) at the SM clock
            "latency_roofline": {"chain_cycles_per_level": 240, "sm_mhz": 1965,
                                 "floor_us": round(levels * 240 / 1965.0, 1),
                                 "achieved_us": round(per_launch_ms * 1e3, 2),
                                 "frac": round(levels * 240 / 1965.0 / (per_launch_ms * 1e3), 4)},
            "classes": classes, "cycle": cycle,
            "cfg5_mgs": (micro or {}).get("mgs")}


def run_b200(args, ws, rank, local):
    import torch
    import paper_2009_07495_b200 as igm
    from paper_2009_07495_b200._capi import KCLASS_NAMES

    dev = igm.Device(local)
    igm.Device._default = dev
    rp, ci, v, bh = config2(args.grid)
    n, nnz = len(rp) - 1, int(rp[-1])
    S, A, F, b, lower, upper, setup_s = setup_b200(rp, ci, v, bh)
    log(f"[bench] setup {setup_s:.2f}s n={n} nnz={nnz} levels fwd/bwd {F.levels(False)}/{F.levels(True)}")
    cfg = solve_cfg(igm)
    stream = torch.cuda.ExternalStream(dev.stream, device=f"cuda:{local}")
    d_b = torch.from_numpy(b).to(f"cuda:{local}")
    d_x = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}")
    torch.cuda.synchronize()

    # warm-up
    rep = None
    for _ in range(args.warmup):
        _, rep = igm.solve(S, A, d_b, cfg, precond=F, x_out=d_x)
    if rep is not None:
        log(f"[bench] warm-up solve: {rep.refinements} refinements, {rep.total_inner_iterations} iterations, "
            f"relres {rep.relres_history[-1]:.3e}, overflows {rep.overflow_total}")

    # timed region (device-resident)
    l0 = dev.launches
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            _, rep = igm.solve(S, A, d_b, cfg, precond=F, x_out=d_x)
            its += rep.total_inner_iterations
        e1.record(stream)
        torch.cuda.synchronize()
    launches = dev.launches - l0
    ms = e0.elapsed_time(e1)
    barrier(ws)
    ms = max_over_ranks(ms, ws)
    its_all = its * ws
    value = its_all / (ms / 1e3)

    # e2e through the public API: pinned host b in, host x out, per step
    hb = torch.from_numpy(b).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    barrier(ws)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_its = 0
    f0.record(stream)
    for _ in range(args.steps):
        _, r2 = igm.solve(S, A, hb.numpy(), cfg, precond=F, x_out=hx.numpy())
        e2e_its += r2.total_inner_iterations
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), ws)
    e2e_val = e2e_its * ws / (e2e_ms / 1e3)

    # e2e through the reference's own C++ API (intgmres::solve, host containers)
    e2e_cpp = None
    if rank == 0 and not args.no_e2e_cpp:
        e2e_cpp = run_e2e_cpp(args, rp, ci, v, bh)
        log(f"[bench] e2e_cpp: {e2e_cpp}")

    # instrumented solve: per-kernel-class device time -> roofline
    igm.lib().igm_profile_enable(1)
    _, rp_ = igm.solve(S, A, d_b, cfg, precond=F, x_out=d_x)
    igm.lib().igm_profile_enable(0)
    kms = np.zeros(11)
    kcnt = np.zeros(11, dtype=np.uint64)
    igm.lib().igm_profile_collect(kms.ctypes.data_as(igm._capi.f64p), kcnt.ctypes.data_as(igm._capi.u64p))
    ab = algorithmic_bytes(n, nnz, len(lower[1]), len(upper[1]), rp_.inner_dims)
    hbm, src = peaks()
    breakdown = {}
    for i, name in enumerate(KCLASS_NAMES):
        if kcnt[i]:
            e = {"ms": round(float(kms[i]), 4), "launches": int(kcnt[i])}
            if name in ab:
                e["GB/s"] = round(ab[name] / (kms[i] / 1e3) / 1e9, 1)
            breakdown[name] = e
    roof = roofline_line(breakdown, ab, n, F.levels(False), ms / args.steps, rep.refinements, hbm, src, None)
    parity = parity_check(d_x, rep, args.grid)

    del S, A, F, d_b, d_x, hb, hx
    torch.cuda.empty_cache()
    micro = None
    if not args.no_cfg5:
        try:
            micro = run_cfg5(args, igm, dev, local) if ws == 1 else \
                run_cfg5_sharded(args, igm, dev, local, rank, ws)
        except Exception as exc:
            micro = {"error": repr(exc)}
        log(f"[bench] cfg5 microbench: {micro}")
    if args.cfg4_sharded and ws == 1:
        try:
            c4 = run_cfg4_sharded(args, igm, dev, local, rank, ws, g=args.cfg4_grid)
        except Exception as exc:
            c4 = {"error": repr(exc)}
        log(f"[bench] cfg4 through the sharded driver at 1 GPU: {c4}")
        micro = micro if isinstance(micro, dict) else {}
        micro["cfg4_sharded_driver_1gpu"] = c4
    if args.cfg5_sharded and ws == 1 and not args.no_cfg5:
        try:
            micro["sharded_driver_1gpu"] = run_cfg5_sharded(args, igm, dev, local, rank, ws)
        except Exception as exc:
            micro["sharded_driver_1gpu"] = {"error": repr(exc)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(rp, ci, v, bh)
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "error": str(exc)}

    if micro and "mgs" in micro:
        roof["cfg5_mgs"] = micro["mgs"]
    if rank == 0:
        line = {
            "metric": "int-GMRES iters/s", "value": value, "unit": "iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "time_to_solution_s": ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded SplitMix64 x*, b = A x*)",
            "config": {"workload": f"cfg2: 3D 7-pt upwind CD {args.grid}^3 (n={n}, nnz={nnz}), integer ILU(0), "
                                   f"GMRES(30), FP64 refinement to 1e-10, Q33.30, checked",
                       "refinements": rep.refinements, "iterations_per_solve": rep.total_inner_iterations,
                       "final_relres": rep.relres_history[-1], "overflows": rep.overflow_total,
                       "overflow_count_exact": rep.overflow_exact,
                       "l2": "inputs larger than L2 (matrix + ILU + basis ~ 0.9 GB)",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "1 GPU"},
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": int(8 * n),
                    "d2h_bytes_per_step": int(8 * n)},
            "e2e_cpp": e2e_cpp,
            "roofline": roof,
            "parity": parity,
            "kernel_microbench": micro,
            "breakdown": breakdown,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--grid", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the config-5 kernel microbench")
    ap.add_argument("--no-e2e-cpp", action="store_true", help="skip the C++ drop-in API leg")
    ap.add_argument("--only-cfg5", action="store_true", help="run only the config-5 microbench (profiling)")
    ap.add_argument("--cfg4-sharded", action="store_true",
                    help="at 1 GPU, also run config 4 through the row-block partitioned solve driver")
    ap.add_argument("--cfg4-grid", type=int, default=256, help="grid of the partitioned config-4 solve")
    ap.add_argument("--cfg5-sharded", action="store_true",
                    help="at 1 GPU, also run the row-block partitioned config-5 driver")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    if args.only_cfg5:
        import paper_2009_07495_b200 as igm
        dev = igm.Device(local)
        igm.Device._default = dev
        print(json.dumps(run_cfg5(args, igm, dev, local)), flush=True)
        return 0
    if ws > 1:
        return run_b200_sharded(args, ws, rank, local)
    return run_b200(args, ws, rank, local)


if __name__ == "__main__":
    sys.exit(main())
