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

    def spmv(self, m, s, v_ext, out_ext):
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

    def mgs_pass(self, mode, w, vprev, vcur, hacc, acc_out, f, b1, b2, a1):
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
