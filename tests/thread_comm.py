"""In-process stand-in for torch.distributed (TEST INFRASTRUCTURE ONLY): the
ranks of a partitioned solve run as Python threads of one process, each with
its own library context (stream), and exchange data through host queues.

Used by the GPU tests to run dist.solve_sharded at world size 2/3 through the
CUDA backend on the single GPU the test box has.  No kernel ever waits on
another rank: every exchange is a host-side copy (tensor.cpu() synchronises
the sending stream, copy_ enqueues on the receiving one), so the ranks'
kernels are ordinary independent launches."""
import queue
import threading

import torch


class _Op:
    SUM = "sum"
    MAX = "max"


class P2POp:
    def __init__(self, op, tensor, peer, group=None):
        self.op, self.tensor, self.peer = op, tensor, peer


class _Done:
    def wait(self):
        pass


class World:
    def __init__(self, size):
        self.size = size
        self.q = {(a, b): queue.Queue() for a in range(size) for b in range(size)}
        self.slots = [None] * size
        self.bar = threading.Barrier(size)

    def rank_view(self, rank):
        return RankComm(self, rank)


class RankComm:
    ReduceOp = _Op
    P2POp = P2POp

    def __init__(self, world, rank):
        self.w, self.rank = world, rank

    def isend(self, *a):  # placeholders (identity markers for P2POp.op)
        raise NotImplementedError

    def irecv(self, *a):
        raise NotImplementedError

    def send(self, t, dst, group=None):
        self.w.q[(self.rank, dst)].put(t.detach().cpu().clone())

    def recv(self, t, src, group=None):
        t.copy_(self.w.q[(src, self.rank)].get(timeout=300))

    def batch_isend_irecv(self, ops):
        for o in ops:
            if o.op == self.isend:
                self.send(o.tensor, o.peer)
        for o in ops:
            if o.op == self.irecv:
                self.recv(o.tensor, o.peer)
        return [_Done()]

    def all_reduce(self, t, op=_Op.SUM, group=None):
        self.w.slots[self.rank] = t.detach().cpu().clone()
        self.w.bar.wait()
        parts = list(self.w.slots)
        self.w.bar.wait()
        acc = parts[0].clone()
        for p in parts[1:]:
            acc = acc + p if op == _Op.SUM else torch.maximum(acc, p)
        t.copy_(acc)

    def broadcast(self, t, src, group=None):
        if self.rank == src:
            self.w.slots[src] = t.detach().cpu().clone()
        self.w.bar.wait()
        v = self.w.slots[src]
        self.w.bar.wait()
        t.copy_(v)


def run_ranks(size, fn):
    """fn(rank, comm) in `size` threads; returns the per-rank results (re-raises)."""
    w = World(size)
    out, errs = [None] * size, []

    def body(r):
        try:
            out[r] = fn(r, w.rank_view(r))
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errs.append(e)
            w.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out
