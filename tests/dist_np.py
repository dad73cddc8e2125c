"""numpy restatement of the per-element config-5 formulas (TEST
INFRASTRUCTURE ONLY): a CPU backend for paper_2009_07495_b200.dist so the
multi-rank partition / halo / allreduce logic is exercised over gloo and
checked against the single-process oracle (fxp.cpp:49-104, split.cpp:137-157)."""
import numpy as np


def asr(x, s):
    return np.right_shift(x, min(int(s), 63))


class NumpySlabBackend:
    def stream(self):
        import contextlib
        return contextlib.nullcontext()

    def upload(self, rp, ci, comp, alphas):
        return dict(rp=np.asarray(rp, np.int64), ci=np.asarray(ci, np.int64), comp=[np.asarray(c, np.int64) for c in comp],
                    alphas=list(alphas))

    def spmv_c5(self, m, s, v_ext, out_ext):
        v = v_ext.numpy()
        rp, ci = m["rp"], m["ci"]
        n = len(rp) - 1
        out = np.zeros(n, np.int64)
        with np.errstate(over="ignore"):
            for l in range(s + 1):
                prod = m["comp"][l] * v[ci]  # wrapping int64
                part = np.zeros(n, np.int64)
                rows = np.repeat(np.arange(n), np.diff(rp))
                np.add.at(part, rows, prod)  # order-free mod 2^64
                out = out + asr(part, m["alphas"][l])
        out_ext.copy_(__import__("torch").from_numpy(out))

    def mgs_pass_c5(self, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1):
        from paper_2009_07495_b200.dist import fx_dot_finalize
        wn = w.numpy()
        with np.errstate(over="ignore"):
            if mode != 0:
                h = fx_dot_finalize(int(hacc.numpy()[0]), f, b1, b2)
                hs = np.int64(h >> min(a1, 63))
                d = asr(hs * vprev.numpy(), f - a1)
                wn[:] = wn - d
            if mode != 3:
                t = asr(wn, b1) * asr(vcur.numpy(), b2)
                acc_out.numpy()[0] += np.sum(t, dtype=np.int64)


# ---------------------------------------------------------------------------
# CPU restatement of the rank-local pieces of dist.solve_sharded (TEST
# INFRASTRUCTURE ONLY): each method is the per-rank computation the matching
# igm_dc_* entry performs, written with the oracle's scalar/vector functions
# and IEEE-exact numpy / Python float arithmetic, so the partition, halo,
# relay, pipeline and allreduce logic of solve_sharded can run over gloo on
# CPU and be compared with the single-process oracle solve.
import math
from types import SimpleNamespace

import torch

MASK = (1 << 64) - 1


def _i64(v):
    v &= MASK
    return v - (1 << 64) if v >= (1 << 63) else v


def _asr(x, s):
    return x >> min(s, 63)


def _wshl(x, s):
    return 0 if s >= 64 else _i64(x << s)


class OracleSlabBackend:
    def __init__(self, oracle):
        self.O = oracle

    # plumbing
    def stream(self):
        import contextlib
        return contextlib.nullcontext()

    def sync(self):
        pass

    def zeros(self, shape, kind):
        return torch.zeros(shape, dtype=torch.int64 if kind == "i64" else torch.float64)

    def host_i64(self, vals):
        return torch.tensor(vals, dtype=torch.int64)

    def from_np(self, a):
        return torch.from_numpy(a)

    def to_np(self, t):
        return t.numpy()

    # slab-local setup: the oracle's row_scale / build_split; the factorisation
    # with its merged values is the product's HOST setup function (no GPU)
    def row_scale(self, rp, ci, v, alpha_a):
        return self.O.row_scale(self.O.csrf(rp, ci, v), alpha_a)

    def build_split(self, vals, alpha_a, max_components):
        return self.O.build_split(vals, alpha_a, max_components)

    def factorize(self, rp, ci, vals):
        import paper_2009_07495_b200 as igm
        return igm.factorize_split_cast(rp, ci, vals, return_lu=True)

    def upload_rows(self, rp, ci, comp, alphas, fp_vals):
        return (SimpleNamespace(sp=self.O.split(rp, ci, comp, alphas), ncomp=len(comp)),
                self.O.csrf(rp, ci, fp_vals))

    def upload_factors(self, lower, upper):
        n = len(lower[0]) - 1
        eye = (np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.ones(n, np.int64),
               np.arange(n, dtype=np.int32))
        return SimpleNamespace(fwd=self.O.ilu(lower, eye), bwd=self.O.ilu(eye, upper))

    def state(self, m):
        K = 11 * 6
        return SimpleNamespace(m=m, red=torch.zeros((m, 3 * (m + 2)), dtype=torch.int64),
                               lcnt=torch.zeros((m, K), dtype=torch.int64), vcnt=torch.zeros(m * K, dtype=torch.int64),
                               rmax=torch.zeros(1, dtype=torch.int64), chain=torch.zeros(4, dtype=torch.float64),
                               err=None, stop=0, dim=0, nbasis=1, do_vecdiv=0, hnext=0, r0n=0.0, nb=0.0, nr=0.0,
                               relnorm=0.0, hess=[[0] * (m + 1) for _ in range(m)], g=[0] * (m + 1), cs=[0] * m,
                               sn=[0] * m)

    def view(self, st, which, j=0):
        return {"red": lambda: st.red[j], "lcnt": lambda: st.lcnt[j], "vcnt": lambda: st.vcnt,
                "rmax": lambda: st.rmax, "chain": lambda: st.chain}[which]()

    @staticmethod
    def _over(st):
        return st.stop or st.err is not None

    @staticmethod
    def _fail(st, exc):
        if st.err is None:
            st.err = exc
        st.stop = 1

    # refinement pieces
    def reset(self, st):
        st.err, st.stop, st.nb, st.nr, st.relnorm = None, 0, 0.0, 0.0, 0.0
        st.rmax.zero_()

    def residual(self, st, a, x_ext, b, r):
        rr, _ = self.O.residual_fp(a, x_ext.numpy(), b.numpy())
        r.numpy()[:] = rr
        st.rmax[0] = int(np.float64(np.max(np.abs(rr)) if len(rr) else 0.0).view(np.int64))

    def norm2(self, st, v, start, out, mode):
        if mode == 3 and self._over(st):
            return
        acc = float(start[0]) if start is not None else 0.0
        for x in v.numpy().tolist():
            acc = acc + x * x
        if mode == 5:
            out[0] = acc
            return
        rt = math.sqrt(acc)
        if mode == 1:
            st.nb = rt
        elif mode == 2:
            st.nr = rt
            st.relnorm = rt if st.nb == 0.0 else rt / st.nb
        else:
            st.r0n = rt
            if rt == 0.0:
                st.stop = 1

    def begin(self, st, f):
        st.red.zero_(); st.lcnt.zero_(); st.vcnt.zero_()
        m = st.m
        st.hess = [[0] * (m + 1) for _ in range(m)]
        st.g, st.cs, st.sn = [0] * (m + 1), [0] * m, [0] * m
        st.g[0] = 1 << f
        st.stop, st.dim, st.nbasis, st.do_vecdiv, st.r0n = 0, 0, 1, 0, 0.0

    def scale(self, st, r, out):
        if self._over(st):
            return
        gamma = np.int64(int(st.rmax[0])).view(np.float64)
        out.numpy()[:] = r.numpy() / gamma

    def tri(self, st, fac, backward, src, dst, fp, j, checked):
        if self._over(st):
            return
        il = fac.bwd if backward else fac.fwd
        if fp:
            dst.numpy()[:] = self.O.apply_inverse_fp(il, src.numpy())
        else:
            from oracle.ffi import PyTrace
            t = PyTrace() if checked else None
            dst.numpy()[:] = self.O.apply_inverse(il, src.numpy(), t)
            if t is not None:
                st.lcnt[j][1 * 6 + 3] += t.total

    # ---- pipelined substitutions (dist.ZPipe), emulated: the "device
    # buffers" are shared-memory segments of one plane of (value, tag) words,
    # the "IPC handle" is the segment name; the import waits for every tag
    # of the plane, the export writes values then tags -- the CUDA kernel's
    # word protocol with the plane as the unit
    pipe_emulate = False

    def pipe_auto(self, dist, group=None):
        return self.pipe_emulate

    def pipe_capable(self, fac, slab):
        if fac is None:
            return False
        fac.slab = slab
        return True

    def _pipe_view(self, key):
        shm = self._shm[key]
        return np.ndarray((shm.size // 16, 2), dtype=np.int64, buffer=shm.buf)

    def pipe_alloc(self, nwords):
        from multiprocessing import shared_memory
        shm = shared_memory.SharedMemory(create=True, size=16 * nwords)
        self.__dict__.setdefault("_shm", {})
        self.__dict__.setdefault("_own_shm", []).append(shm)
        key = len(self._shm) + 1
        self._shm[key] = shm
        self._pipe_view(key)[:] = 0
        return key

    def pipe_handle(self, key):
        name = self._shm[key].name.encode()
        assert len(name) <= 64
        return np.frombuffer(name.ljust(64, b"\0"), dtype=np.int64).copy()

    def pipe_open(self, handle):
        from multiprocessing import shared_memory
        name = np.asarray(handle, dtype=np.int64).tobytes().rstrip(b"\0").decode()
        shm = shared_memory.SharedMemory(name=name)
        self.__dict__.setdefault("_shm", {})
        key = len(self._shm) + 1
        self._shm[key] = shm
        return key

    def pipe_close(self):
        for shm in self.__dict__.get("_shm", {}).values():
            shm.close()
        for shm in self.__dict__.get("_own_shm", []):
            shm.unlink()
        self._shm, self._own_shm = {}, []

    def tri_piped(self, st, fac, backward, src, dst, j, checked, zimp, zexp, kexp, epoch):
        import time
        if st.stop and st.err is None:  # the replicated stop (errors can be rank-local: run on)
            return
        P, nx = fac.slab.plane, fac.slab.next_
        y = src.numpy().copy()
        tags = epoch + np.arange(P, dtype=np.int64)
        if zimp is not None:
            buf = self._pipe_view(zimp)
            t0 = time.time()
            while not np.array_equal(buf[:, 1], tags):
                if time.time() - t0 > 120:
                    raise RuntimeError("tri_piped: import timed out")
                time.sleep(0.0005)
            if backward:
                y[nx - P:] = buf[:, 0]
            else:
                y[:P] = buf[:, 0]
        il = fac.bwd if backward else fac.fwd
        from oracle.ffi import PyTrace
        t = PyTrace() if checked else None
        dst.numpy()[:] = self.O.apply_inverse(il, y, t)
        if t is not None:
            st.lcnt[j][1 * 6 + 3] += t.total
        if zexp is not None:
            z = (nx // P - 1 - kexp) if backward else kexp
            buf = self._pipe_view(zexp)
            buf[:, 0] = dst.numpy()[z * P:(z + 1) * P]
            buf[:, 1] = tags

    def encode(self, st, r0, v0, f):
        if self._over(st):
            return
        from oracle.ffi import CheckerError
        out = v0.numpy()
        for i, x in enumerate(r0.numpy().tolist()):
            try:
                out[i] = self.O.encode(x / st.r0n, f)
            except CheckerError as e:
                out[i] = 0
                self._fail(st, OverflowError(e.msg))

    def spmv(self, st, m, s, v_ext, out, j, checked):
        if self._over(st):
            return
        from oracle.ffi import PyTrace
        t = PyTrace() if checked else None
        out.numpy()[:] = self.O.spmv(m.sp, s, v_ext.numpy(), t)
        if t is not None:
            st.lcnt[j][0] += t.total

    def mgs_pass(self, st, j, i, w, vprev, vcur, f, sh, checked):
        if self._over(st):
            return
        from paper_2009_07495_b200.dist import fx_dot_finalize
        red = st.red[j].numpy()
        wn = w.numpy()
        if i > 0:
            h = fx_dot_finalize(int(red[3 * (i - 1)]), f, sh.dot_b1, sh.dot_b2)
            wn[:] = self.O.fx_axpy_sub(wn, h, vprev.numpy(), f, sh.axpy_b1)
        with np.errstate(over="ignore"):
            if i <= j:
                t = np.right_shift(wn, min(sh.dot_b1, 63)) * np.right_shift(vcur.numpy(), min(sh.dot_b2, 63))
            else:
                q = np.right_shift(wn, min(sh.norm_b1, 63))
                t = q * q
            red[3 * i] += np.sum(t, dtype=np.int64)

    def step(self, st, j, f, sh, w, checked):
        st.do_vecdiv = 0
        if self._over(st):
            return
        O = self.O
        red = [int(x) for x in st.red[j].numpy()]
        col = st.hess[j]
        for i in range(j + 1):
            col[i] = fx_dot_finalize_int(red[3 * i], f, sh.dot_b1, sh.dot_b2)
        nsum = red[3 * (j + 1)]
        if nsum < 0:
            return self._fail(st, ArithmeticError("fx_norm: accumulator wrapped negative"))
        hnext = _wshl(O.isqrt(nsum), sh.norm_b1)
        col[j + 1] = hnext
        happy = hnext == 0
        if not happy:
            if _asr(hnext, sh.div_b2) == 0:
                return self._fail(st, ArithmeticError("fx_div: shifted divisor is zero"))
            st.do_vecdiv, st.hnext, st.nbasis = 1, hnext, j + 2
        for i in range(j):
            c, s, hi, hn = st.cs[i], st.sn[i], col[i], col[i + 1]
            a = O.fx_mul(c, hi, f, 0, sh.givens_b2, f)
            b = O.fx_mul(s, hn, f, 0, sh.givens_b2, f)
            d = O.fx_mul(c, hn, f, 0, sh.givens_b2, f)
            q = O.fx_mul(s, hi, f, 0, sh.givens_b2, f)
            col[i], col[i + 1] = O.fx_add(a, b), O.fx_sub(d, q)
        from oracle.ffi import CheckerError
        try:
            tmp = O.fx_norm(np.array([col[j], col[j + 1]], np.int64), f, sh.norm_b1)
        except CheckerError as e:
            return self._fail(st, ArithmeticError(e.msg))
        if tmp == 0:
            st.stop = 1
            return
        try:
            c = O.fx_div(col[j], tmp, f, sh.div_b1, sh.div_b2)
            s = O.fx_div(col[j + 1], tmp, f, sh.div_b1, sh.div_b2)
        except CheckerError as e:
            return self._fail(st, ArithmeticError(e.msg))
        st.cs[j], st.sn[j] = c, s
        col[j], col[j + 1] = tmp, 0
        g_old = st.g[j]
        neg_s = O.fx_sub(0, s)
        st.g[j + 1] = O.fx_mul(neg_s, g_old, f, sh.rot_b, sh.rot_b, f)
        st.g[j] = O.fx_mul(c, g_old, f, sh.rot_b, sh.rot_b, f)
        st.dim = j + 1
        if happy:
            st.stop = 1

    def vec_div(self, st, j, w, vout, f, sh, checked):
        if not st.do_vecdiv:
            return
        out = vout.numpy()
        for l, x in enumerate(w.numpy().tolist()):
            out[l] = self.O.fx_div(x, st.hnext, f, sh.div_b1, sh.div_b2)

    def finish(self, st, f, basis, x):
        if st.err is not None or st.dim == 0:
            return
        dim, sc = st.dim, 2.0 ** -f
        dec = lambda raw: float(np.float64(raw)) * sc
        y = [0.0] * dim
        for i in range(dim - 1, -1, -1):
            acc = dec(st.g[i])
            for jj in range(i + 1, dim):
                acc = acc - dec(st.hess[jj][i]) * y[jj]
            rii = dec(st.hess[i][i])
            if rii == 0.0:
                return self._fail(st, RuntimeError("solve_hessenberg: zero diagonal"))
            y[i] = acc / rii
        wts = [st.r0n * yy for yy in y]
        gamma = np.int64(int(st.rmax[0])).view(np.float64)
        b = basis.numpy()
        acc = np.zeros(b.shape[1])
        for jj in range(dim):
            acc = acc + wts[jj] * (b[jj].astype(np.float64) * sc)
        xn = x.numpy()
        xn[:] = xn + gamma * acc

    def fetch(self, st):
        if st.err is not None:
            raise st.err
        return SimpleNamespace(dim=st.dim, stop=st.stop, nbasis=st.nbasis, add_inexact=0, r0_norm=st.r0n,
                               relnorm=st.relnorm, nb=st.nb, nr=st.nr,
                               gamma=float(np.int64(int(st.rmax[0])).view(np.float64)),
                               overflows=int(st.lcnt.sum()) + int(st.vcnt.sum()))


def fx_dot_finalize_int(acc, f, b1, b2):
    from paper_2009_07495_b200.dist import fx_dot_finalize
    return fx_dot_finalize(acc, f, b1, b2)
