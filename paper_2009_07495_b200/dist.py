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
    ext[slab.own0:slab.own1].copy_(own)
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

    def spmv(self, m, s, v_ext, out_ext):
        import ctypes as C
        # device pointers: enqueued on the library stream (== torch's current
        # stream inside stream()), returns synchronised
        self.igm._check(self.igm.lib().igm_spmv(self.dev.h, m.h, s, C.c_void_p(v_ext.data_ptr()),
                                                C.c_void_p(out_ext.data_ptr()), None))

    def mgs_pass(self, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1):
        self.igm.mgs_pass(self.dev, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1)


def spmv_mgs_sharded(backend, slab: Slab, m, s: int, v_own, basis_own, k: int, f: int, b1: int, b2: int,
                     a1: int, dist, work, group=None):
    """One config-5 call on this rank: returns (w_own, acc) where acc holds
    the k all-reduced accumulators (int64 tensor, wrapping sums).

    work: dict of reusable buffers {'vext': (next_,), 'wext': (next_,),
    'acc': (k,) int64} on the backend's device."""
    vext, wext, acc = work["vext"], work["wext"], work["acc"]
    with backend.stream():
        halo_exchange(slab, v_own, vext, dist, group)
        backend.spmv(m, s, vext, wext)
        w = wext[slab.own0:slab.own1]
        acc.zero_()
        for i in range(k):
            backend.mgs_pass(0 if i == 0 else 1, w, basis_own[i - 1] if i > 0 else None, basis_own[i],
                             acc[i - 1:i] if i > 0 else None, acc[i:i + 1], f, b1, b2, a1)
            if slab.world > 1:
                dist.all_reduce(acc[i:i + 1], op=dist.ReduceOp.SUM, group=group)
        backend.mgs_pass(3, w, basis_own[k - 1], None, acc[k - 1:k], None, f, b1, b2, a1)
    return w, acc
