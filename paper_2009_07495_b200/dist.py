"""Row-block (z-slab) partitioning of the int-GMRES kernels across the GPUs of
one box (north star: "rows are block-partitioned across
1/2/4/8 GPUs ... halos move over NVLink P2P or NCCL, and the int64 partial dot
products are combined with an NCCL allreduce, which is exact").

One process per GPU (torch.distributed, NCCL).  Rank p owns a contiguous run
of whole xy-planes (natural order has k outermost, so a plane run is a row
block).  Its matrix rows are stored over the *extended* local index space --
its own planes plus one halo plane on each side (7-point stencils reach one
plane) -- so the unmodified single-GPU SpMV kernel runs on it and each row's
CSR-order sum is the reference's (split.cpp:137-157): bit-identical.

Per call of the config-5 kernel (w = A v, then MGS of w against k basis
vectors, fxp.cpp:49-104):
  1. halo exchange: the first / last own plane of v goes to rank p-1 / p+1
     (batched NCCL P2P send/recv over NVLink);
  2. local SpMV over the extended vector, keep the own rows;
  3. for each pass i: the fused axpy_{i-1} + dot_i kernel on the own rows
     leaves a wrapping u64 partial accumulator, one all_reduce(SUM) of it
     (int64 two's complement addition == Z/2^64: exact in any order) gives
     every rank the reference's accumulator, from which the next pass
     re-derives h_i exactly as the single-GPU kernel does.
Nothing else is exchanged: vec_div / encode / x-update are local and the
Hessenberg scalars are replicated (§8(e)).

The local compute is a pluggable backend: `CudaSlabBackend` (the product:
C-ABI kernels on device tensors, NCCL) is the only one shipped here; the
CPU tests drive the same partition / halo / allreduce logic with a numpy
restatement of the per-element formulas over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class Slab:
    """Rank-local view of a row-block partition over whole planes."""
    rank: int
    world: int
    plane: int       # rows per plane (g*g)
    nplanes: int     # planes in the global grid
    z0: int          # own planes [z0, z1)
    z1: int
    h0: int          # first global row of the extended local space
    own0: int        # own rows [own0, own1) in local (extended) indices
    own1: int
    next_: int       # rows in the extended local space

    @property
    def n_own(self) -> int:
        return self.own1 - self.own0

    @property
    def global_rows(self) -> Tuple[int, int]:
        return self.z0 * self.plane, self.z1 * self.plane


def plane_split(nplanes: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced plane ranges [z0, z1) per rank."""
    if world < 1 or nplanes < world:
        raise ValueError(f"cannot split {nplanes} planes over {world} ranks")
    base, extra = divmod(nplanes, world)
    out, z = [], 0
    for p in range(world):
        c = base + (1 if p < extra else 0)
        out.append((z, z + c))
        z += c
    return out


def make_slab(nplanes: int, plane: int, rank: int, world: int) -> Slab:
    z0, z1 = plane_split(nplanes, world)[rank]
    zh0, zh1 = max(0, z0 - 1), min(nplanes, z1 + 1)
    return Slab(rank, world, plane, nplanes, z0, z1, zh0 * plane, (z0 - zh0) * plane, (z1 - zh0) * plane,
                (zh1 - zh0) * plane)


def slab_csr(row_ptr, col_idx, vals: Sequence[np.ndarray], slab: Slab):
    """Extended-square local CSR of a global CSR (one vals array per split
    component): own rows keep their entries (columns shifted into the local
    space; every column must fall inside the halo range), halo rows are empty."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    g0, g1 = slab.global_rows
    a, b = int(row_ptr[g0]), int(row_ptr[g1])
    cols = np.asarray(col_idx[a:b], dtype=np.int64) - slab.h0
    if cols.size and (cols.min() < 0 or cols.max() >= slab.next_):
        raise ValueError("slab_csr: a row reaches beyond the one-plane halo")
    rp = np.zeros(slab.next_ + 1, dtype=np.int32)
    rp[slab.own0 + 1:slab.own1 + 1] = (row_ptr[g0 + 1:g1 + 1] - a).astype(np.int32)
    rp[slab.own1 + 1:] = rp[slab.own1]
    return rp, cols.astype(np.int32), [np.asarray(v[a:b]) for v in vals]


def halo_ops(slab: Slab, own, ext, dist, group=None):
    """P2P ops of the halo exchange: own -> ext interior, first/last own plane
    to the neighbours, their boundary planes into ext's halo planes."""
    P = slab.plane
    ops = []
    if slab.rank > 0:
        ops.append(dist.P2POp(dist.isend, own[:P].contiguous(), slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, ext[:P], slab.rank - 1, group))
    if slab.rank < slab.world - 1:
        ops.append(dist.P2POp(dist.isend, own[-P:].contiguous(), slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, ext[slab.own1:slab.own1 + P], slab.rank + 1, group))
    return ops


def halo_exchange(slab: Slab, own, ext, dist, group=None) -> None:
    """Fill ext (extended local vector) from own rows + the neighbours' planes."""
    dst = ext[slab.own0:slab.own1]
    if dst.data_ptr() != own.data_ptr():
        dst.copy_(own)
    ops = halo_ops(slab, own, ext, dist, group)
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def fx_dot_finalize(acc: int, f: int, b1: int, b2: int) -> int:
    """fx_dot's final shift of the wrapped accumulator (fxp.cpp:63-65)."""
    a = ((int(acc) + (1 << 63)) % (1 << 64)) - (1 << 63)  # as int64
    e = f - b1 - b2
    if e >= 0:
        return a >> min(e, 63)
    s = -e
    if s >= 64:
        return 0
    v = (a << s) & ((1 << 64) - 1)
    return v - (1 << 64) if v >= (1 << 63) else v


class CudaSlabBackend:
    """The product backend: this rank's GPU through the C ABI."""

    def __init__(self, igm, device):
        import torch
        self.igm = igm
        self.dev = device
        self._torch = torch
        self._stream = torch.cuda.ExternalStream(device.stream, device=f"cuda:{device.index}")

    def stream(self):
        """torch ops (buffer zeroing, halo copies, NCCL) ordered on the
        library's stream, with the pass kernels that share their buffers"""
        return self._torch.cuda.stream(self._stream)

    def upload(self, rp, ci, comp, alphas):
        return self.igm.SplitMatrix(rp, ci, comp, alphas, device=self.dev)

    def spmv_c5(self, m, s, v_ext, out_ext):
        import ctypes as C
        # device pointers: enqueued on the library stream (== torch's current
        # stream inside stream()), returns synchronised
        self.igm._check(self.igm.lib().igm_spmv(self.dev.h, m.h, s, C.c_void_p(v_ext.data_ptr()),
                                                C.c_void_p(out_ext.data_ptr()), None))

    def mgs_pass_c5(self, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1):
        self.igm.mgs_pass(self.dev, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1)

    # ---- the partitioned solve (solve_sharded): igm_dstate + igm_dc_* entries
    def sync(self):
        self._torch.cuda.synchronize(self.dev.index)

    def zeros(self, shape, kind):
        dt = {"i64": self._torch.int64, "f64": self._torch.float64}[kind]
        with self.stream():
            return self._torch.zeros(shape, dtype=dt, device=f"cuda:{self.dev.index}")

    def host_i64(self, vals):
        return self._torch.tensor(vals, dtype=self._torch.int64, device=f"cuda:{self.dev.index}")

    def from_np(self, a):
        return self._torch.from_numpy(a).to(f"cuda:{self.dev.index}")

    def to_np(self, t):
        return t.cpu().numpy()

    # slab-local setup on the device (igm_*_dev: bit-identical to the host versions)
    def row_scale(self, rp, ci, v, alpha_a):
        return self.igm.row_scale_device(rp, ci, v, alpha_a, device=self.dev)

    def build_split(self, vals, alpha_a, max_components):
        return self.igm.build_split_device(vals, alpha_a, max_components, device=self.dev)

    def factorize(self, rp, ci, vals):
        return self.igm.factorize_split_cast_device(rp, ci, vals, device=self.dev, return_lu=True)

    def upload_rows(self, rp, ci, comp, alphas, fp_vals):
        """own rows x extended columns: SplitMatrix + CsrMatrixF (shared pattern)"""
        return (self.igm.SplitMatrix(rp, ci, comp, alphas, device=self.dev),
                self.igm.CsrMatrixF(rp, ci, fp_vals, device=self.dev))

    def upload_factors(self, lower, upper):
        return self.igm.IluFactors(lower, upper, device=self.dev)

    def state(self, m):
        return _DState(self, m)

    def view(self, st, which, j=0):
        return st.view(which, j)

    def _c(self, name, *args):
        self.igm._check(getattr(self.igm.lib(), name)(self.dev.h, *args))

    @staticmethod
    def _p(t):
        import ctypes as C
        return None if t is None else C.c_void_p(t.data_ptr())

    def reset(self, st):
        self._c("igm_dc_reset", st.h)

    def residual(self, st, a, x_ext, b, r):
        self._c("igm_dc_residual", st.h, a.h, self._p(x_ext), self._p(b), self._p(r))

    def norm2(self, st, v, start, out, mode):
        self._c("igm_dc_norm2", st.h, int(v.numel()), self._p(v), self._p(start), self._p(out), mode)

    def begin(self, st, f):
        self._c("igm_dc_begin", st.h, f)

    def scale(self, st, r, out):
        self._c("igm_dc_scale", st.h, int(r.numel()), self._p(r), self._p(out))

    def tri(self, st, fac, backward, src, dst, fp, j, checked):
        if fp:
            self._c("igm_dc_tri_fp", st.h, fac.h, 1 if backward else 0, self._p(src), self._p(dst))
        else:
            self._c("igm_dc_tri", st.h, fac.h, 1 if backward else 0, self._p(src), self._p(dst), j,
                    1 if checked else 0)

    # ---- pipelined substitutions: boundary planes streamed over CUDA IPC
    def pipe_auto(self, dist, group=None) -> bool:
        """P2P words between ranks need one process per GPU (NCCL ranks);
        IGM_DIST_PIPE=0 selects the plane relay"""
        import os
        if os.environ.get("IGM_DIST_PIPE", "1") == "0" or not hasattr(dist, "get_backend"):
            return False
        try:
            return dist.get_backend(group) == "nccl"
        except Exception:
            return False

    def pipe_capable(self, fac, slab) -> bool:
        """both local factors run the 7-point pencil wavefront on the slab's grid"""
        if fac is None:
            return False
        for bw in (False, True):
            info = fac.schedule_info(bw)
            gx, gy, gz = info["grid"]
            if fac.pencil_bricks(bw) <= 0 or gx * gy != slab.plane or gx * gy * gz != slab.next_:
                return False
        return True

    def pipe_alloc(self, nwords):
        import ctypes as C
        p = C.c_void_p()
        self._c("igm_dev_alloc", C.c_uint64(16 * nwords), C.byref(p))
        return p.value

    def pipe_handle(self, buf):
        import ctypes as C
        h = (C.c_ubyte * 64)()
        self.igm._check(self.igm.lib().igm_ipc_handle(C.c_void_p(buf), h))
        return np.frombuffer(bytes(h), dtype=np.int64).copy()

    def pipe_open(self, handle):
        import ctypes as C
        h = (C.c_ubyte * 64).from_buffer_copy(np.asarray(handle, dtype=np.int64).tobytes())
        p = C.c_void_p()
        self._c("igm_ipc_open", h, C.byref(p))
        return p.value

    def tri_piped(self, st, fac, backward, src, dst, j, checked, zimp, zexp, kexp, epoch):
        import ctypes as C
        self._c("igm_dc_tri_piped", st.h, fac.h, 1 if backward else 0, self._p(src), self._p(dst), j,
                1 if checked else 0, None if zimp is None else C.c_void_p(zimp),
                None if zexp is None else C.c_void_p(zexp), kexp, C.c_uint64(epoch))

    # ---- one-shot P2P mailbox reductions (igm_mbox_*): the per-pass sums
    def mbox_auto(self, dist, group=None) -> bool:
        """mailboxes are mapped between processes with CUDA IPC: one process
        per GPU (NCCL ranks); IGM_DIST_MBOX=0 keeps torch.distributed"""
        import os
        if os.environ.get("IGM_DIST_MBOX", "1") == "0" or not hasattr(dist, "get_backend"):
            return False
        try:
            return dist.get_backend(group) == "nccl"
        except Exception:
            return False

    def mbox_for(self, slab, comm, max_words=2048):
        """this rank's connected mailbox (cached): the IPC handles travel in
        one all_reduce of a zero-padded (world, 8) int64 table"""
        import ctypes as C
        cache = self.__dict__.setdefault("_mboxes", {})
        key = (slab.rank, slab.world, max_words)
        if key in cache:
            return cache[key]
        mb = C.c_void_p()
        self._c("igm_mbox_create", slab.rank, slab.world, max_words, C.byref(mb))
        h = (C.c_ubyte * 64)()
        self.igm._check(self.igm.lib().igm_mbox_handle(mb, h))
        mine = np.zeros((slab.world, 8), dtype=np.int64)
        mine[slab.rank] = np.frombuffer(bytes(h), dtype=np.int64)
        allh = self.host_i64(mine.ravel().tolist())
        comm.d.all_reduce(allh, op=comm.d.ReduceOp.SUM, group=comm.g)
        raw = allh.cpu().numpy().astype(np.int64).tobytes()
        # mapping a peer's buffer can fail (no P2P path between two devices):
        # the ranks agree on the outcome, and fall back to all_reduce together
        ok = 1
        try:
            self.igm._check(self.igm.lib().igm_mbox_connect_ipc(mb, (C.c_ubyte * len(raw)).from_buffer_copy(raw)))
        except Exception as exc:  # noqa: BLE001 -- any failure disables the mailboxes on every rank
            ok = 0
            import warnings
            warnings.warn(f"igm_mbox: cannot map the peers' mailboxes ({exc}); using torch.distributed all_reduce")
        flag = self.host_i64([ok])
        comm.d.all_reduce(flag, op=comm.d.ReduceOp.MIN, group=comm.g)
        if int(flag[0]) == 0:
            self.igm.lib().igm_mbox_free(mb)
            mb = None
        cache[key] = mb
        return mb

    def mbox_allreduce(self, mb, t, op):
        self._c("igm_mbox_allreduce", mb, self._p(t), int(t.numel()), op)

    def mbox_status(self, mb):
        self._c("igm_mbox_status", mb)

    def encode(self, st, r0, v0, f):
        self._c("igm_dc_encode", st.h, int(r0.numel()), self._p(r0), self._p(v0), f)

    def spmv(self, st, m, s, v_ext, out, j, checked):
        self._c("igm_dc_spmv", st.h, m.h, s, self._p(v_ext), self._p(out), j, 1 if checked else 0)

    def mgs_pass(self, st, j, i, w, vprev, vcur, f, sh, checked):
        import ctypes as C
        self._c("igm_dc_mgs_pass", st.h, int(w.numel()), j, i, self._p(w), self._p(vprev), self._p(vcur), f,
                C.byref(sh.c()), 1 if checked else 0)

    def step(self, st, j, f, sh, w, checked):
        import ctypes as C
        self._c("igm_dc_step", st.h, j, f, C.byref(sh.c()), self._p(w), 1 if checked else 0)

    def vec_div(self, st, j, w, vout, f, sh, checked):
        import ctypes as C
        self._c("igm_dc_vec_div", st.h, int(w.numel()), j, self._p(w), self._p(vout), f, C.byref(sh.c()),
                1 if checked else 0)

    def finish(self, st, f, basis, x):
        self._c("igm_dc_finish", st.h, f, int(x.numel()), self._p(basis), self._p(x))

    def fetch(self, st):
        import ctypes as C
        from . import _capi
        info = _capi.DcInfo()
        self._c("igm_dc_fetch", st.h, C.byref(info))
        return info


class _DevView:
    """__cuda_array_interface__ over a device buffer of the C library (no copy)."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class _DState:
    """igm_dstate: the rank's replicated per-cycle scalars + reduction slots."""

    def __init__(self, be, m):
        import ctypes as C
        self.be, self.m = be, m
        h = C.c_void_p()
        be.igm._check(be.igm.lib().igm_dstate_create(be.dev.h, m, C.byref(h)))
        self.h = h
        self._views = {}

    def view(self, which, j=0):
        import ctypes as C
        from . import _capi
        key = (which, j)
        if key not in self._views:
            code = {"red": _capi.IGM_DS_RED, "lcnt": _capi.IGM_DS_LCNT, "vcnt": _capi.IGM_DS_VCNT,
                    "rmax": _capi.IGM_DS_RMAX, "chain": _capi.IGM_DS_CHAIN}[which]
            ptr, nb = C.c_void_p(), C.c_int64()
            self.be.igm._check(self.be.igm.lib().igm_dstate_buffer(self.h, code, j, C.byref(ptr), C.byref(nb)))
            ts = "<f8" if which == "chain" else "<i8"
            self._views[key] = self.be._torch.as_tensor(_DevView(ptr.value, nb.value // 8, ts),
                                                        device=f"cuda:{self.be.dev.index}")
        return self._views[key]

    def __del__(self):
        try:
            self.be.igm.lib().igm_dstate_free(self.h)
        except Exception:
            pass


def spmv_mgs_sharded(backend, slab: Slab, m, s: int, v_own, basis_own, k: int, f: int, b1: int, b2: int,
                     a1: int, dist, work, group=None):
    """One config-5 call on this rank: returns (w_own, acc) where acc holds
    the k all-reduced accumulators (int64 tensor, wrapping sums).

    work: dict of reusable buffers {'vext': (next_,), 'wext': (next_,),
    'acc': (k,) int64} on the backend's device."""
    vext, wext, acc = work["vext"], work["wext"], work["acc"]
    with backend.stream():
        halo_exchange(slab, v_own, vext, dist, group)
        backend.spmv_c5(m, s, vext, wext)
        w = wext[slab.own0:slab.own1]
        acc.zero_()
        for i in range(k):
            backend.mgs_pass_c5(0 if i == 0 else 1, w, basis_own[i - 1] if i > 0 else None, basis_own[i],
                             acc[i - 1:i] if i > 0 else None, acc[i:i + 1], f, b1, b2, a1)
            if slab.world > 1:
                dist.all_reduce(acc[i:i + 1], op=dist.ReduceOp.SUM, group=group)
        backend.mgs_pass_c5(3, w, basis_own[k - 1], None, acc[k - 1:k], None, f, b1, b2, a1)
    return w, acc


# ===========================================================================
# The whole refinement solve on a row-block partition (SURVEY.md §8(e),
# BASELINE config 4: "rows block-partitioned along z at 1/2/4/8 GPUs with halo
# exchange and NCCL int64 dot allreduce").
#
# Every rank runs the reference's solve (refine.cpp:21-106) and cycle
# (gmres_int.cpp:42-196) over its own rows; the exchanges are exactly the
# data the sequential algorithm moves across a plane boundary:
#   * SpMV / FP residual: one halo plane per side (7- and 27-point stencils);
#   * MGS / norm passes: the wrapping u64 accumulators (+ the sum|t| words of
#     checked mode) summed over ranks -- Z/2^64 addition, exact in any order;
#     the per-step scalar work (h_ij, fx_norm, Givens, g) is then replicated;
#   * norm2 (split.cpp:45-49) is one sequential FP64 chain: rank p continues
#     it from rank p-1's running sum (a rank-ordered relay), the last rank
#     hands the total to all -- bit-identical to the single-chain order;
#   * gamma = max|r_i|: int64 MAX of the IEEE bits (non-negative doubles
#     order as integers);
#   * ILU(0) substitutions (ilu.cpp:122-180) stay the GLOBAL factors (a
#     block-Jacobi split would change the bits): forward solves run rank 0 ->
#     P-1, each rank starting once its lower neighbour's last plane of z has
#     arrived (placed in a unit halo row of its extended local factor: z = y /
#     1 exactly), backward solves run P-1 -> 0 the same way.  The DAG's
#     critical path is unchanged by P (§8(e)).
# Everything else (encode, vec_div, x update) is row-local.
# ===========================================================================
from dataclasses import field


def slab_rows(row_ptr, col_idx, vals: Sequence[np.ndarray], slab: Slab):
    """The rank's rows of a global CSR as a RECTANGULAR local CSR: own rows x
    extended columns (own planes + one halo plane per side).  Row order and
    each row's entry order are the global ones, so per-row CSR-order sums are
    the reference's."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    g0, g1 = slab.global_rows
    a, b = int(row_ptr[g0]), int(row_ptr[g1])
    cols = np.asarray(col_idx[a:b], dtype=np.int64) - slab.h0
    if cols.size and (cols.min() < 0 or cols.max() >= slab.next_):
        raise ValueError("slab_rows: a row reaches beyond the one-plane halo")
    rp = (row_ptr[g0:g1 + 1] - a).astype(np.int32)
    return rp, cols.astype(np.int32), [np.asarray(v[a:b]) for v in vals]


def slab_factor(factor, slab: Slab):
    """Extended-square local copy of one global ILU factor (row_ptr, col_idx,
    vals, diag_pos): own rows keep their entries (columns shifted into the
    local space), halo rows become unit rows (diagonal 1, no off-diagonals),
    so a substitution copies the neighbour's values placed in their rhs
    slots exactly (integer: trunc(y / 1) = y; FP64: y / 1.0 = y)."""
    rp, ci, v, dp = (np.asarray(a) for a in factor)
    rp = rp.astype(np.int64)
    g0, g1 = slab.global_rows
    a, b = int(rp[g0]), int(rp[g1])
    own_cols = ci[a:b].astype(np.int64) - slab.h0
    if own_cols.size and (own_cols.min() < 0 or own_cols.max() >= slab.next_):
        raise ValueError("slab_factor: a factor row reaches beyond the one-plane halo")
    nl, o0, o1 = slab.next_, slab.own0, slab.own1
    counts = np.ones(nl, dtype=np.int64)
    counts[o0:o1] = np.diff(rp[g0:g1 + 1])
    lrp = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(counts, out=lrp[1:])
    nnz = int(lrp[-1])
    lci = np.empty(nnz, dtype=np.int32)
    lv = np.empty(nnz, dtype=np.int64)
    ldp = np.empty(nl, dtype=np.int32)
    halo = np.r_[np.arange(0, o0), np.arange(o1, nl)].astype(np.int64)
    lci[lrp[halo]] = halo
    lv[lrp[halo]] = 1
    ldp[halo] = lrp[halo]
    s0 = int(lrp[o0])
    lci[s0:s0 + (b - a)] = own_cols
    lv[s0:s0 + (b - a)] = np.asarray(v[a:b], dtype=np.int64)
    ldp[o0:o1] = (np.asarray(dp[g0:g1], dtype=np.int64) - rp[g0:g1]) + lrp[o0:o1]
    return lrp.astype(np.int32), lci, lv, ldp


def shard_problem(be, slab: Slab, row_ptr, col_idx, comp, alphas, a_fp_vals, factors=None) -> dict:
    """The rank's inputs of solve_sharded from the global SplitMatrix (comp,
    alphas over row_ptr/col_idx), the FP64 matrix values on the same pattern,
    and optionally the global integer ILU factors (lower, upper)."""
    comp = [np.asarray(c) for c in np.atleast_2d(comp)]
    rp, ci, vals = slab_rows(row_ptr, col_idx, comp + [np.asarray(a_fp_vals)], slab)
    sp, af = be.upload_rows(rp, ci, np.stack(vals[:-1]), alphas, vals[-1])
    ilu = None
    if factors is not None:
        ilu = be.upload_factors(slab_factor(factors[0], slab), slab_factor(factors[1], slab))
    return dict(split=sp, csrf=af, ilu=ilu, ncomp=len(comp))


# ---- slab-local setup ("generate and factorise slab-locally") --
# A rank builds its rows, their scaling and the splitting's truncation layer
# from its own planes alone.  ILU(0) (ilu.cpp:25-120) eliminates row i with
# the rows j < i of its pattern, all within one plane below: the factors of a
# slab need the finished U rows (merged values, diagonal included) of the
# previous rank's last plane and nothing else.  So the factorisation is a
# rank-ordered relay of one plane of doubles, and every rank runs the
# unmodified factorisation on an extended matrix whose lower halo rows are
# those finished U rows (no entry left of the diagonal: nothing to eliminate,
# they pass through unchanged) and whose upper halo rows are unit rows.
def _u_part(rp, ci, row0):
    """mask of the entries on or right of the diagonal; rows are row0 + local index"""
    rows = np.repeat(np.arange(len(rp) - 1, dtype=np.int64) + row0, np.diff(rp))
    return np.asarray(ci, dtype=np.int64) >= rows


def slab_ilu_local(slab: Slab, own, halo_pattern, lu_in, factorize):
    """The rank's extended-square local integer factors -- array for array
    what slab_factor() cuts out of the global split_cast(factorize_ilu0(A))
    -- from its own rows only.

    own:          (row_ptr, col_idx GLOBAL, scaled vals) of the rank's rows
    halo_pattern: (row_ptr, col_idx GLOBAL) of plane z0-1's rows (None on rank 0)
    lu_in:        merged factor values of that plane's U part (diagonal
                  included), CSR order, from rank-1 (None on rank 0)
    factorize:    (row_ptr, col_idx, vals) -> (lower, upper, merged values)
    Returns (lower, upper, lu_out); lu_out = this rank's last plane in the
    same form for rank+1 (None on the last rank)."""
    P, o0, o1, nl = slab.plane, slab.own0, slab.own1, slab.next_
    g0, _ = slab.global_rows
    rp_o, ci_o, v_o = (np.asarray(a) for a in own)
    cnt = np.ones(nl, dtype=np.int64)
    cnt[o0:o1] = np.diff(rp_o)
    if o0:
        hrp, hci = (np.asarray(a) for a in halo_pattern)
        keep = _u_part(hrp, hci, g0 - P)
        cnt[:o0] = np.add.reduceat(keep.astype(np.int64), hrp[:-1].astype(np.int64))
        if lu_in is None or len(lu_in) != int(keep.sum()):
            raise ValueError("slab_ilu_local: the received plane does not match the pattern of plane z0-1")
    rp = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp[1:])
    nnz = int(rp[-1])
    ci = np.empty(nnz, dtype=np.int32)
    v = np.empty(nnz, dtype=np.float64)
    a, b = int(rp[o0]), int(rp[o1])
    if o0:
        ci[:a] = (hci[keep].astype(np.int64) - slab.h0).astype(np.int32)
        v[:a] = lu_in
    ci[a:b] = (ci_o.astype(np.int64) - slab.h0).astype(np.int32)
    v[a:b] = v_o
    up = np.arange(o1, nl, dtype=np.int64)
    ci[b:] = up.astype(np.int32)
    v[b:] = 1.0
    lower, upper, lu = factorize(rp.astype(np.int32), ci, v)
    lower, upper = [np.asarray(x) for x in lower], [np.asarray(x) for x in upper]
    lu = np.asarray(lu)
    lu_out = None
    if slab.rank < slab.world - 1:
        r0 = o1 - P
        k0, k1 = int(rp[r0]), int(rp[o1])
        lu_out = lu[k0:k1][_u_part(rp[r0:o1 + 1] - k0, ci[k0:k1], r0)].copy()
    # halo rows become unit rows (what slab_factor stores): L's already hold
    # the diagonal only; U's lower halo rows lose their off-diagonal entries
    lrp, lci, lv, ldp = lower
    lv = lv.copy()
    lv[lrp[:o0]] = 1
    urp, uci, uv, udp = (x.astype(np.int64) for x in upper)
    if o0:
        cut = int(urp[o0])
        urp2 = np.concatenate([np.arange(o0, dtype=np.int64), urp[o0:] - cut + o0])
        uci2 = np.concatenate([np.arange(o0, dtype=np.int64), uci[cut:]])
        uv2 = np.concatenate([np.ones(o0, dtype=np.int64), uv[cut:]])
        udp2 = np.concatenate([np.arange(o0, dtype=np.int64), udp[o0:] - cut + o0])
        upper = (urp2.astype(np.int32), uci2.astype(np.int32), uv2.astype(np.int64), udp2.astype(np.int32))
    else:
        upper = (urp.astype(np.int32), uci.astype(np.int32), uv.astype(np.int64), udp.astype(np.int32))
    return (lrp, lci, lv, ldp), upper, lu_out


def setup_slab_local(be, slab: Slab, rows_fn, alpha_a: int, comm, ilu: bool = True) -> dict:
    """solve_sharded's inputs built from the rank's own planes (no global
    array on any rank): row_scale (split.cpp:61-79) and the truncation layer
    of build_split (split.cpp:90-135; depth-0 splittings -- a deeper layer's
    scale is a global max) are row local; split_cast(factorize_ilu0(A))
    through the plane relay of slab_ilu_local.

    rows_fn(z0, z1) -> (row_ptr, col_idx GLOBAL, vals) of planes [z0, z1)
    be: backend with row_scale / build_split / factorize (device setup for
        CudaSlabBackend) and the upload methods; comm: send_np / recv_np.
    Returns solve_sharded's `mats` plus 'scale' (the own rows' row scaling,
    for scale_rhs) and 'rows' (row_ptr, local col_idx, scaled vals)."""
    rp, ci, v = rows_fn(slab.z0, slab.z1)
    vals, scale = be.row_scale(rp, ci, v, alpha_a)
    del v
    comp, alphas, _ = be.build_split(vals, alpha_a, 1)
    ci_loc = (np.asarray(ci, dtype=np.int64) - slab.h0).astype(np.int32)
    if ci_loc.size and (ci_loc.min() < 0 or ci_loc.max() >= slab.next_):
        raise ValueError("setup_slab_local: a row reaches beyond the one-plane halo")
    sp, af = be.upload_rows(rp, ci_loc, np.atleast_2d(comp), alphas, vals)
    fac = None
    if ilu:
        halo, lu_in = None, None
        if slab.rank > 0:
            hrp, hci, _ = rows_fn(slab.z0 - 1, slab.z0)
            halo = (hrp, hci)
            lu_in = comm.recv_np(int(_u_part(np.asarray(hrp), np.asarray(hci), (slab.z0 - 1) * slab.plane).sum()),
                                 slab.rank - 1)
        lower, upper, lu_out = slab_ilu_local(slab, (rp, ci, vals), halo, lu_in, be.factorize)
        if lu_out is not None:
            comm.send_np(lu_out, slab.rank + 1)
        fac = be.upload_factors(lower, upper)
    return dict(split=sp, csrf=af, ilu=fac, ncomp=1, scale=np.asarray(scale), rows=(rp, ci_loc, vals))


@dataclass
class ShardedReport:
    """SolveReport (refine.hpp:36-47) of a partitioned solve (identical on every rank)."""
    converged: bool = False
    refinements: int = 0
    total_inner_iterations: int = 0
    inner_dims: List[int] = field(default_factory=list)
    relres_history: List[float] = field(default_factory=list)
    gamma_history: List[float] = field(default_factory=list)
    overflow_per_restart: List[int] = field(default_factory=list)
    overflow_total: int = 0
    overflow_exact: bool = True


class _Comm:
    """The rank's exchanges (torch.distributed: NCCL on GPUs, gloo on CPU)."""

    def __init__(self, slab: Slab, dist, group=None, be=None, mbox=None):
        """mbox: reduce the small int64 sums through the library's P2P
        mailboxes (igm_mbox_*) instead of torch.distributed -- None: when
        the backend can (one process per GPU), False: never."""
        self.s, self.d, self.g = slab, dist, group
        self.rank, self.world = slab.rank, slab.world
        self.be, self.mb = be, None
        if (self.world > 1 and mbox is not False and be is not None and hasattr(be, "mbox_for")
                and (mbox is True or be.mbox_auto(dist, group))):
            self.mb = be.mbox_for(slab, self)

    def _native(self, t) -> bool:
        return (self.mb is not None and getattr(t, "is_cuda", False) and t.dtype == self.be._torch.int64
                and t.is_contiguous())

    def sum_(self, t):
        if self.world > 1:
            if self._native(t):
                self.be.mbox_allreduce(self.mb, t, 0)
            else:
                self.d.all_reduce(t, op=self.d.ReduceOp.SUM, group=self.g)

    def max_(self, t):
        if self.world > 1:
            if self._native(t):
                self.be.mbox_allreduce(self.mb, t, 1)
            else:
                self.d.all_reduce(t, op=self.d.ReduceOp.MAX, group=self.g)

    def check(self):
        """raises when a mailbox reduction gave up waiting for a peer"""
        if self.mb is not None:
            self.be.mbox_status(self.mb)

    def send(self, t, dst):
        self.d.send(t.contiguous(), dst, group=self.g)

    def recv(self, t, src):
        self.d.recv(t, src, group=self.g)

    def bcast(self, t, src):
        if self.world > 1:
            self.d.broadcast(t, src, group=self.g)

    def halo(self, own, ext):
        halo_exchange(self.s, own, ext, self.d, self.g)

    def send_np(self, a, dst):
        """a float64 host array to rank dst (setup relay); buffer, transfer
        and host copy all ordered on the backend's stream"""
        with self.be.stream():
            t = self.be.from_np(np.ascontiguousarray(a, dtype=np.float64))
            self.d.send(t, dst, group=self.g)
            self.be.sync()

    def recv_np(self, count, src):
        with self.be.stream():
            t = self.be.zeros(count, "f64")
            self.d.recv(t, src, group=self.g)
            return self.be.to_np(t)


def _validate_cycle(m: int, f: int, depth: int, ncomp: int, sh) -> None:
    """run_cycle's argument checks, same order and texts (gmres_int.cpp:47-52,
    fxp.hpp:24-27, fxp.cpp:106-127)."""
    if m < 1:
        raise ValueError("run_cycle: m must be >= 1")
    if depth < 0 or depth > ncomp - 1:
        raise ValueError("run_cycle: splitting depth out of range")
    if f < 0 or f > 62:
        raise ValueError("QFormat: frac_bits must be in [0, 62]")
    for name, b in (("dot_b1", sh.dot_b1), ("dot_b2", sh.dot_b2), ("axpy_b1", sh.axpy_b1),
                    ("norm_b1", sh.norm_b1), ("div_b1", sh.div_b1), ("div_b2", sh.div_b2),
                    ("givens_b2", sh.givens_b2), ("rot_b", sh.rot_b)):
        if b < 0 or b > 62:
            raise ValueError(f"ShiftPlan: {name} out of range")
    if sh.dot_b1 + sh.dot_b2 > f:
        raise ValueError("ShiftPlan: dot shifts exceed frac_bits")
    if sh.axpy_b1 > f:
        raise ValueError("ShiftPlan: axpy shift exceeds frac_bits")
    if 2 * (f - sh.norm_b1) > 62:
        raise ValueError("ShiftPlan: norm accumulator exceeds 62 fractional bits")
    if sh.div_b1 + sh.div_b2 > f + 62:
        raise ValueError("ShiftPlan: division shifts out of range")


class ZPipe:
    """The rank's side of the pipelined substitutions: the
    global ILU(0) wavefront crosses a slab boundary pencil by pencil instead
    of plane by plane.  Rank p owns two import buffers of one plane of
    16-byte words (value, epoch + natural idx): `fwd` written by rank p-1's
    forward wavefront as it finishes its last own plane, `bwd` by rank p+1's
    backward wavefront (its first own plane); the neighbours map them with
    CUDA IPC and store into them over NVLink.  In the rank-local solve order
    the import is plane 0 (the lower halo forward, the upper halo backward),
    the export is plane `kexp_*`.  Epochs are (call count) << 32, identical on
    every rank, so a word of an earlier substitution never matches.  Reuse of
    a buffer is ordered by the DAG itself: rank p writes epoch e+1 into
    p+1's `fwd` only after its own backward of call e, which needed p+1's
    backward of call e, which ran after p+1's forward of call e read epoch e."""

    def __init__(self, be, slab: Slab, comm):
        P = slab.plane
        rank, world = slab.rank, slab.world
        self.imp_fwd = be.pipe_alloc(P) if rank > 0 else None
        self.imp_bwd = be.pipe_alloc(P) if rank < world - 1 else None
        mine = np.zeros((world, 2, 8), dtype=np.int64)
        if self.imp_fwd is not None:
            mine[rank, 0] = be.pipe_handle(self.imp_fwd)
        if self.imp_bwd is not None:
            mine[rank, 1] = be.pipe_handle(self.imp_bwd)
        with be.stream():
            allh = be.host_i64(mine.ravel().tolist())
            comm.sum_(allh)
            allh = allh.cpu().numpy().reshape(world, 2, 8)
        # mapping a neighbour's buffer can fail (no P2P path): the ranks agree
        # on the outcome in _pipe_for and relay whole planes together instead
        self.ok = True
        self.exp_fwd = self.exp_bwd = None
        try:
            self.exp_fwd = be.pipe_open(allh[rank + 1, 0]) if rank < world - 1 else None
            self.exp_bwd = be.pipe_open(allh[rank - 1, 1]) if rank > 0 else None
        except Exception as exc:  # noqa: BLE001
            self.ok = False
            import warnings
            warnings.warn(f"ZPipe: cannot map the neighbour's import buffer ({exc}); relaying whole planes")
        self.kexp_fwd, self.kexp_bwd = self.planes(slab)
        self.calls = 0

    @staticmethod
    def planes(slab: Slab) -> Tuple[int, int]:
        """solve-order index of the exported plane, forward and backward (-1: none)"""
        P, nz = slab.plane, slab.next_ // slab.plane
        return (slab.own1 // P - 1 if slab.rank < slab.world - 1 else -1,
                nz - 1 - slab.own0 // P if slab.rank > 0 else -1)

    def next_epoch(self) -> int:
        self.calls += 1
        return self.calls << 32


def _pipe_for(be, slab: Slab, pre, comm, dist, group, pipe):
    """The rank's ZPipe (cached on the backend) when every rank can stream
    its boundary planes, else None (the plane relay)."""
    if slab.world == 1 or pre is None or pipe is False or not hasattr(be, "tri_piped"):
        return None
    if pipe is None and not be.pipe_auto(dist, group):
        return None
    with be.stream():
        bad = be.host_i64([0 if be.pipe_capable(pre, slab) else 1])
        comm.max_(bad)
        if int(bad[0]):
            return None
    cache = be.__dict__.setdefault("_zpipes", {})
    key = (slab.rank, slab.world, slab.z0, slab.z1, slab.plane, slab.nplanes)
    if key not in cache:
        zp = ZPipe(be, slab, comm)
        with be.stream():
            bad = be.host_i64([0 if getattr(zp, "ok", True) else 1])
            comm.max_(bad)
            cache[key] = None if int(bad[0]) else zp
    return cache[key]


def solve_sharded(be, slab: Slab, mats: dict, b_own, cfg, dist, group=None, s_schedule=None,
                  pipe=None, mbox=None):
    """solve() (refine.cpp:21-106, fixed-point engine) on this rank's rows.

    be:   rank-local backend (CudaSlabBackend: the product's kernels through
          the C ABI; tests drive the same code with a CPU restatement)
    mats: {'split': own rows x ext cols SplitMatrix, 'csrf': the same for
          A_fp, 'ilu': extended-square local factors or None, 'ncomp': int}
    b_own: the rank's rows of b; cfg: RefineConfig-like (tol,
          max_refinements, m, frac_bits, s, checked, shifts).
    pipe: stream the integer substitutions' boundary planes pencil by pencil
          (ZPipe) -- None: when the backend and every rank can, False: relay.
    mbox: sum the per-pass accumulators / counters through the library's P2P
          mailboxes (igm_mbox_*) -- None: when one process drives each GPU
          (NCCL ranks), False: torch.distributed all_reduce.
    Returns (x_own, ShardedReport); every rank returns the same report."""
    comm = _Comm(slab, dist, group, be, mbox)
    be.sync()  # inputs produced on other streams are complete
    n, nx, P = slab.n_own, slab.next_, slab.plane
    o0, o1 = slab.own0, slab.own1
    rank, world = slab.rank, slab.world
    M = max(cfg.m, 1)
    f, sh, checked = cfg.frac_bits, cfg.shifts, bool(cfg.checked)
    pre = mats.get("ilu")
    st = be.state(M)
    x_ext = be.zeros(nx, "f64")
    x_own = x_ext[o0:o1]
    r = be.zeros(n, "f64")
    t_ext = be.zeros(nx, "f64")
    u_ext = be.zeros(nx, "f64")
    r0 = be.zeros(n, "f64")
    basis = be.zeros((M + 1, n), "i64")
    v_ext = be.zeros(nx, "i64")
    y_ext = be.zeros(nx, "i64")
    z_ext = be.zeros(nx, "i64")
    q_ext = be.zeros(nx, "i64")
    w_plain = be.zeros(n, "i64")
    chain = be.view(st, "chain")

    def norm2_relay(v, mode):
        """norm2 (split.cpp:45-49) over the global vector: one sequential chain
        through the ranks in order, then finished (sqrt) on every rank."""
        with be.stream():
            if rank > 0:
                comm.recv(chain[1:2], rank - 1)
            be.norm2(st, v, chain[1:2] if rank > 0 else None, chain[0:1], 5)
            if rank < world - 1:
                comm.send(chain[0:1], rank + 1)
            chain[2:3].copy_(chain[0:1])
            comm.bcast(chain[2:3], world - 1)
            be.norm2(st, v[:0], chain[2:3], None, mode)

    zp = _pipe_for(be, slab, pre, comm, dist, group, pipe)

    def tri_pipeline(fac_fp, src_ext, mid_ext, dst_ext, j=0):
        """forward (ranks in order) then backward (reverse order) substitution
        of the global factors; src_ext's own rows hold the rhs.  Integer
        substitutions stream the boundary planes word by word when the ranks
        can (ZPipe); otherwise, and for the FP64 one, whole planes are relayed."""
        if zp is not None and not fac_fp:
            e = zp.next_epoch()
            with be.stream():
                be.tri_piped(st, pre, False, src_ext, mid_ext, j, checked, zp.imp_fwd, zp.exp_fwd, zp.kexp_fwd, e)
                be.tri_piped(st, pre, True, mid_ext, dst_ext, j, checked, zp.imp_bwd, zp.exp_bwd, zp.kexp_bwd, e)
            return
        with be.stream():
            if rank > 0:
                comm.recv(src_ext[:o0], rank - 1)
            be.tri(st, pre, False, src_ext, mid_ext, fac_fp, j, checked)
            if rank < world - 1:
                comm.send(mid_ext[o1 - P:o1], rank + 1)
                comm.recv(mid_ext[o1:], rank + 1)
            be.tri(st, pre, True, mid_ext, dst_ext, fac_fp, j, checked)
            if rank > 0:
                comm.send(dst_ext[o0:o0 + P], rank - 1)

    def fetch():
        """synchronise, read the scalars; a device error on any rank is raised on all"""
        err = None
        try:
            info = be.fetch(st)
        except (ArithmeticError, ValueError, RuntimeError, OverflowError) as e:
            err, info = e, None
        with be.stream():
            code = be.host_i64([0 if err is None else _err_code(err)])
            comm.max_(code)
            c = int(code[0])
        comm.check()
        if c:
            if err is not None:
                raise err
            raise _ERR_TYPES.get(c, RuntimeError)("error raised on another rank")
        return info

    rep = ShardedReport()
    with be.stream():
        be.reset(st)
    norm2_relay(b_own, 1)  # ||b|| (residual_fp's denominator)

    def residual():
        with be.stream():
            comm.halo(x_own, x_ext)
            be.residual(st, mats["csrf"], x_ext, b_own, r)
            comm.max_(be.view(st, "rmax"))
        norm2_relay(r, 2)
        return fetch()

    info = residual()
    relnorm = info.relnorm
    rep.relres_history.append(relnorm)
    ncomp = mats["ncomp"]
    k = 0
    while k < cfg.max_refinements and relnorm >= cfg.tol:
        gamma = info.gamma
        if gamma == 0.0:
            break
        depth = s_schedule(k) if s_schedule is not None else cfg.s
        _validate_cycle(cfg.m, f, depth, ncomp, sh)
        # ---- one int-GMRES(m) cycle on b_k = r / gamma, x0 = 0
        with be.stream():
            be.begin(st, f)
            if pre is not None:
                be.scale(st, r, t_ext[o0:o1])
        if pre is not None:
            tri_pipeline(True, t_ext, u_ext, t_ext)
            r0_own = t_ext[o0:o1]
        else:
            with be.stream():
                be.scale(st, r, r0)
            r0_own = r0
        norm2_relay(r0_own, 3)
        with be.stream():
            be.encode(st, r0_own, basis[0], f)
        for j in range(M):
            with be.stream():
                comm.halo(basis[j], v_ext)
                if pre is not None:
                    be.spmv(st, mats["split"], depth, v_ext, y_ext[o0:o1], j, checked)
            if pre is not None:
                tri_pipeline(False, y_ext, z_ext, q_ext, j)
                w = q_ext[o0:o1]
            else:
                with be.stream():
                    be.spmv(st, mats["split"], depth, v_ext, w_plain, j, checked)
                w = w_plain
            with be.stream():
                red = be.view(st, "red", j)
                for i in range(j + 2):
                    be.mgs_pass(st, j, i, w, basis[i - 1] if i > 0 else None, basis[i] if i <= j else None,
                                f, sh, checked)
                    comm.sum_(red[3 * i:3 * i + 3])
                if checked:
                    comm.sum_(be.view(st, "lcnt", j))
                be.step(st, j, f, sh, w, checked)
                be.vec_div(st, j, w, basis[j + 1], f, sh, checked)
        with be.stream():
            if checked:
                comm.sum_(be.view(st, "vcnt"))
            be.finish(st, f, basis, x_own)
        info = fetch()
        dim = info.dim
        if info.add_inexact:
            rep.overflow_exact = False
        if dim == 0:
            break
        rep.refinements = k + 1
        rep.total_inner_iterations += dim
        rep.inner_dims.append(dim)
        rep.gamma_history.append(gamma)
        rep.overflow_per_restart.append(int(info.overflows))
        rep.overflow_total += int(info.overflows)
        info = residual()
        relnorm = info.relnorm
        rep.relres_history.append(relnorm)
        k += 1
    rep.converged = relnorm < cfg.tol
    return x_own, rep


_ERR_TYPES = {1: ValueError, 2: ArithmeticError, 3: OverflowError, 4: RuntimeError}


def _err_code(e) -> int:
    for code, t in ((3, OverflowError), (2, ArithmeticError), (1, ValueError), (4, RuntimeError)):
        if isinstance(e, t):
            return code
    return 4
