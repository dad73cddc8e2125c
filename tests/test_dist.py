"""Row-block (z-slab) sharding of the config-5 kernel:
partition / halo exchange / exact u64 allreduce over gloo with world_size 2
(CPU), against the single-process oracle.  The GPU parity of the same driver
at world_size 1 through the CUDA backend is in test_gpu_parity."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_07495_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plane_split_and_slab_csr():
    assert D.plane_split(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    with pytest.raises(ValueError):
        D.plane_split(2, 3)
    from workloads import gen
    g = 6
    rp, ci, v = gen.upwind_3d(g, 20.0)
    for world in (1, 2, 3):
        rows = []
        for r in range(world):
            sl = D.make_slab(g, g * g, r, world)
            lrp, lci, (lv,) = D.slab_csr(rp, ci, [v], sl)
            assert len(lrp) == sl.next_ + 1 and lrp[sl.own0] == 0
            for i in range(sl.own0, sl.own1):  # every own row maps back to the global row
                gi = sl.h0 + i
                a, b = rp[gi], rp[gi + 1]
                assert np.array_equal(lci[lrp[i]:lrp[i + 1]] + sl.h0, ci[a:b])
                assert np.array_equal(lv[lrp[i]:lrp[i + 1]], v[a:b])
            rows.append(sl.global_rows)
        assert rows[0][0] == 0 and rows[-1][1] == g ** 3
        assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    # the generator's slab form is the same local matrix
    for world in (2, 3):
        for r in range(world):
            sl = D.make_slab(g, g * g, r, world)
            a = D.slab_csr(rp, ci, [v], sl)
            b = gen.upwind_3d_slab(g, 20.0, sl.z0, sl.z1)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2][0], b[2])
            assert (b[3], b[4], b[5]) == (sl.h0, sl.own0, sl.own1)


def _worker(rank, world, port, g, k, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.dist_np import NumpySlabBackend
        from workloads import gen
        import paper_2009_07495_b200 as igm
        rp, ci, v = gen.upwind_3d(g, 20.0)
        vals, _ = igm.row_scale(rp, ci, v, 16)
        comp, al, _ = igm.build_split(vals, 16, 2)
        n = len(rp) - 1
        sl = D.make_slab(g, g * g, rank, world)
        lrp, lci, lcomp = D.slab_csr(rp, ci, comp, sl)
        be = NumpySlabBackend()
        m = be.upload(lrp, lci, lcomp, al)
        rng = np.random.default_rng(seed)
        vfull = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
        bfull = rng.integers(-(1 << 40), 1 << 40, (k, n), dtype=np.int64)
        g0, g1 = sl.global_rows
        v_own = torch.from_numpy(vfull[g0:g1].copy())
        b_own = torch.from_numpy(bfull[:, g0:g1].copy())
        work = dict(vext=torch.zeros(sl.next_, dtype=torch.int64), wext=torch.zeros(sl.next_, dtype=torch.int64),
                    acc=torch.zeros(k, dtype=torch.int64))
        w, acc = D.spmv_mgs_sharded(be, sl, m, 1, v_own, b_own, k, 30, 16, 0, 16, dist, work)
        parts = [None] * world
        dist.all_gather_object(parts, (g0, w.numpy().copy()))
        if rank == 0:
            wg = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
            q.put((wg, acc.numpy().copy(), vfull, bfull))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_spmv_mgs_matches_oracle(oracle, world):
    """World-size 2/3 gloo run of dist.spmv_mgs_sharded == the single-process
    reference sequence (spmv with a depth-1 split, then k x (fx_dot,
    fx_axpy_sub)) on every word of w and every h_i."""
    g, k, seed = 8, 5, 1234
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, g, k, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    wg, acc, vfull, bfull = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from workloads import gen
    import paper_2009_07495_b200 as igm
    rp, ci, v = gen.upwind_3d(g, 20.0)
    vals, _ = igm.row_scale(rp, ci, v, 16)
    comp, al, _ = oracle.build_split(vals, 16, 2)
    sp = oracle.split(rp, ci, comp, al)
    w = oracle.spmv(sp, 1, vfull)
    for i in range(k):
        h = oracle.fx_dot(w, bfull[i], 30, 16, 0)
        assert h == D.fx_dot_finalize(int(acc[i]), 30, 16, 0)
        w = oracle.fx_axpy_sub(w, h, bfull[i], 30, 16)
    assert np.array_equal(wg, w)


# ---------------------------------------------------------------------------
# the whole partitioned solve (dist.solve_sharded) vs the single-process oracle
def _problem(kind, g, oracle):
    from workloads import gen
    if kind == "27pt_ilu":
        rp, ci, v = gen.stencil27(g, 5)
    else:
        rp, ci, v = gen.upwind_3d(g, 20.0)
    n = len(rp) - 1
    A = oracle.csrf(rp, ci, v)
    ilu = kind.endswith("_ilu")
    alpha = 32 if ilu else 16
    vals, scale = oracle.row_scale(A, alpha)
    comp, al, _ = oracle.build_split(vals, alpha, 1 if ilu else 2)
    fac = oracle.factorize_split_cast(oracle.csrf(rp, ci, vals)) if ilu else None
    b = gen.spmv_np(rp, ci, v, gen.uniform(17, n)) / scale
    return rp, ci, vals, comp, al, fac, b


def _rows_fn(kind, g):
    from workloads import gen
    if kind == "27pt_ilu":
        return lambda z0, z1: gen.stencil27_rows(g, 5, z0, z1)
    return lambda z0, z1: gen.upwind_3d_rows(g, 20.0, z0, z1)


def _local_problem(be, sl, kind, g, comm):
    """the rank's inputs from its own planes only (dist.setup_slab_local)"""
    from workloads import gen
    mats = D.setup_slab_local(be, sl, _rows_fn(kind, g), 32, comm, ilu=True)
    rp, ci_loc, _ = mats["rows"]
    xs = gen.uniform(17, g ** 3)[sl.h0:sl.h0 + sl.next_]
    _, _, v = _rows_fn(kind, g)(sl.z0, sl.z1)
    return mats, gen.spmv_np(rp, ci_loc, v, xs) / mats["scale"]


@pytest.mark.parametrize("kind,g", [("7pt_ilu", 7), ("27pt_ilu", 6)])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_slab_local_ilu_equals_global_cut(oracle, kind, g, world):
    """dist.slab_ilu_local: every rank factorises its own planes from the
    previous rank's last plane of merged U rows (a relay of one plane of
    doubles) -- its extended-square integer factors are, array for array,
    what slab_factor cuts out of the oracle's global
    split_cast(factorize_ilu0(A)) (ilu.cpp:25-120); the own rows' scaling
    and truncation layer equal the global ones' slices."""
    from tests.dist_np import OracleSlabBackend
    rp, ci, vals, comp, al, fac, b = _problem(kind, g, oracle)
    be = OracleSlabBackend(oracle)
    rows = _rows_fn(kind, g)
    lu = None
    for r in range(world):
        sl = D.make_slab(g, g * g, r, world)
        g0, g1 = sl.global_rows
        a, e = int(rp[g0]), int(rp[g1])
        orp, oci, ov = rows(sl.z0, sl.z1)
        sv, sc = be.row_scale(orp, oci, ov, 32)
        assert np.array_equal(sv, vals[a:e])
        c1, a1, _ = be.build_split(sv, 32, 1)
        assert np.array_equal(np.atleast_2d(c1)[0], np.atleast_2d(comp)[0][a:e]) and list(a1) == list(al)
        halo = rows(sl.z0 - 1, sl.z0)[:2] if r > 0 else None
        lower, upper, lu = D.slab_ilu_local(sl, (orp, oci, sv), halo, lu, be.factorize)
        for got, want in ((lower, D.slab_factor(fac[0], sl)), (upper, D.slab_factor(fac[1], sl))):
            for x, y in zip(got, want):
                assert np.array_equal(np.asarray(x), np.asarray(y))
        assert (lu is None) == (r == world - 1)
    with pytest.raises(ValueError, match="does not match the pattern"):
        sl = D.make_slab(g, g * g, 1, 2)
        orp, oci, ov = rows(sl.z0, sl.z1)
        D.slab_ilu_local(sl, (orp, oci, be.row_scale(orp, oci, ov, 32)[0]), rows(sl.z0 - 1, sl.z0)[:2],
                         np.zeros(3), be.factorize)


def _solve_worker(rank, world, port, kind, g, m, s, q, pipe=False, local=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.ffi import Oracle
        from tests.dist_np import OracleSlabBackend
        import paper_2009_07495_b200 as igm
        O = Oracle()
        rp, ci, vals, comp, al, fac, b = _problem(kind, g, O)
        sl = D.make_slab(g, g * g, rank, world)
        be = OracleSlabBackend(O)
        be.pipe_emulate = pipe
        g0, g1 = sl.global_rows
        if local:  # nothing global on any rank: the planes, their scaling, the ILU relay
            mats, b_own = _local_problem(be, sl, kind, g, D._Comm(sl, dist, be=be))
        else:
            mats, b_own = D.shard_problem(be, sl, rp, ci, comp, al, vals, fac), b[g0:g1].copy()
        plan = igm.ShiftPlan.default_preconditioned(30) if fac is not None else igm.ShiftPlan.default_unpreconditioned(30)
        cfg = igm.RefineConfig(tol=1e-10, max_refinements=30, m=m, frac_bits=30, s=s, checked=True, shifts=plan)
        x, rep = D.solve_sharded(be, sl, mats, torch.from_numpy(b_own), cfg, dist)
        piped = sum(zp.calls for zp in be.__dict__.get("_zpipes", {}).values())
        parts = [None] * world
        dist.all_gather_object(parts, (g0, x.numpy().copy(), rep, piped))
        if pipe:
            be.pipe_close()
        if rank == 0:
            q.put(sorted(parts, key=lambda t: t[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,pipe,local", [
    ("27pt_ilu", 2, False, False), ("27pt_ilu", 3, False, False), ("7pt_plain", 2, False, False),
    ("7pt_ilu", 2, True, False), ("7pt_ilu", 3, True, False), ("27pt_ilu", 3, True, False),
    ("27pt_ilu", 3, False, True), ("7pt_ilu", 2, True, True)])
def test_sharded_solve_matches_oracle(oracle, kind, world, pipe, local):
    """World 2/3 gloo run of dist.solve_sharded (halo planes, exact u64 pass
    sums, relayed norm2 chain, rank-pipelined global ILU) against the
    single-process oracle solve: every x word, the relative-residual history,
    the inner dimensions and the gammas bit-identical.  pipe: the integer
    substitutions hand the boundary plane over dist.ZPipe's word protocol
    (tagged one-plane buffers opened by handle, epochs per call; emulated
    with shared-memory segments) instead of the NCCL/gloo plane relay.
    local: every rank builds its inputs from its own planes
    (dist.setup_slab_local: plane-range generator, local scaling, the ILU(0)
    relay of one plane of merged U rows) instead of cutting global arrays."""
    g, m = 6, 8
    s = 0 if kind.endswith("_ilu") else 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, kind, g, m, s, q, pipe, local))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.concatenate([p[1] for p in parts])
    rep = parts[0][2]
    assert all(p[2] == rep for p in parts)  # replicated report
    if pipe:  # every integer substitution pair went through the word protocol
        assert all(p[3] == parts[0][3] for p in parts) and parts[0][3] == rep.refinements * m  # one per Arnoldi step (the FP64 one is relayed)
    else:
        assert all(p[3] == 0 for p in parts)
    from oracle.ffi import Shifts
    from tests.cases import PRE, UNPRE
    rp, ci, vals, comp, al, fac, b = _problem(kind, g, oracle)
    sp, af = oracle.split(rp, ci, comp, al), oracle.csrf(rp, ci, vals)
    il = oracle.ilu(*fac) if fac is not None else None
    xo, ro = oracle.solve(sp, af, b, 1e-10, 30, m, 30, s, Shifts(*(PRE if fac is not None else UNPRE)),
                          precond=il)
    assert rep.converged and ro["converged"]
    assert rep.relres_history == ro["relres_history"]
    assert rep.inner_dims == ro["inner_dims"] and rep.gamma_history == ro["gamma_history"]
    assert rep.overflow_total == ro["overflow_total"] == 0
    assert np.array_equal(x, xo)


def run_sharded_threads(oracle, make_backend, kind, g, m, s, world, to_dev=lambda t: t, local=False):
    """dist.solve_sharded on `world` in-process ranks (tests/thread_comm.py);
    returns (x, reports, problem)."""
    from tests.thread_comm import run_ranks
    import paper_2009_07495_b200 as igm
    prob = _problem(kind, g, oracle)
    rp, ci, vals, comp, al, fac, b = prob
    plan = igm.ShiftPlan.default_preconditioned(30) if fac is not None else igm.ShiftPlan.default_unpreconditioned(30)
    cfg = igm.RefineConfig(tol=1e-10, max_refinements=30, m=m, frac_bits=30, s=s, checked=True, shifts=plan)

    def rank_fn(rank, comm):
        be = make_backend(rank)
        sl = D.make_slab(g, g * g, rank, world)
        g0, g1 = sl.global_rows
        if local:
            mats, b_own = _local_problem(be, sl, kind, g, D._Comm(sl, comm, be=be, mbox=False))
        else:
            mats, b_own = D.shard_problem(be, sl, rp, ci, comp, al, vals, fac), b[g0:g1].copy()
        x, rep = D.solve_sharded(be, sl, mats, to_dev(torch.from_numpy(b_own)), cfg, comm)
        return g0, x.cpu().numpy().copy(), rep

    parts = sorted(run_ranks(world, rank_fn), key=lambda t: t[0])
    return np.concatenate([p[1] for p in parts]), [p[2] for p in parts], prob


def check_sharded_vs_oracle(oracle, x, reps, prob, m, s):
    from oracle.ffi import Shifts
    from tests.cases import PRE, UNPRE
    rp, ci, vals, comp, al, fac, b = prob
    rep = reps[0]
    assert all(r == rep for r in reps)
    sp, af = oracle.split(rp, ci, comp, al), oracle.csrf(rp, ci, vals)
    il = oracle.ilu(*fac) if fac is not None else None
    xo, ro = oracle.solve(sp, af, b, 1e-10, 30, m, 30, s, Shifts(*(PRE if fac is not None else UNPRE)),
                          precond=il)
    assert rep.converged and ro["converged"] and rep.refinements >= 2
    assert rep.relres_history == ro["relres_history"]
    assert rep.inner_dims == ro["inner_dims"] and rep.gamma_history == ro["gamma_history"]
    assert rep.overflow_total == ro["overflow_total"]
    assert np.array_equal(x, xo)


def test_sharded_solve_thread_ranks_oracle_backend(oracle):
    """The in-process rank harness the GPU test uses (threads + host queues)
    gives the same bit-exact solve as the gloo processes."""
    from tests.dist_np import OracleSlabBackend
    x, reps, prob = run_sharded_threads(oracle, lambda r: OracleSlabBackend(oracle), "27pt_ilu", 6, 8, 0, 3)
    check_sharded_vs_oracle(oracle, x, reps, prob, 8, 0)
