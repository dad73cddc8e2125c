"""Randomised equivalence of the CPU restatement and the reference library
(mirrors the reference's oracle-equivalence suites, test_fxp.cpp:237-318,
test_split.cpp:122-151, test_ilu.cpp:127-149), including checked-mode traces."""
import numpy as np
import pytest

from oracle.ffi import CheckerError, PyTrace, Shifts
from tests.cases import CASES, build_case

I64_MIN, I64_MAX = np.iinfo(np.int64).min, np.iinfo(np.int64).max


def _both(fn_o, fn_r):
    try:
        a = ("ok", fn_o())
    except CheckerError as e:
        a = ("err", e.code)
    try:
        b = ("ok", fn_r())
    except CheckerError as e:
        b = ("err", e.code)
    return a, b


def test_scalar_ops_random(oracle, reference):
    rng = np.random.default_rng(20260821)
    for _ in range(4000):
        f = int(rng.integers(2, 63))
        a, b = (int(x) for x in rng.integers(I64_MIN, I64_MAX, 2, dtype=np.int64))
        b1, b2 = int(rng.integers(0, 30)) % f, int(rng.integers(0, 30)) % f
        t1, t2 = PyTrace(), PyTrace()
        x, y = _both(lambda: oracle.fx_mul(a, b, f, b1, b2, f, t1), lambda: reference.fx_mul(a, b, f, b1, b2, f, t2))
        assert x == y and t1.total == t2.total
        t1, t2 = PyTrace(), PyTrace()
        x, y = _both(lambda: oracle.fx_div(a, b, f, b1, b2, t1), lambda: reference.fx_div(a, b, f, b1, b2, t2))
        assert x == y and t1.total == t2.total and t1.events == t2.events
        assert oracle.fx_add(a, b) == reference.fx_add(a, b)
        assert oracle.fx_sub(a, b) == reference.fx_sub(a, b)


def test_isqrt_sqrt_random(oracle, reference):
    rng = np.random.default_rng(7)
    for v in rng.integers(0, 2 ** 63, 3000, dtype=np.uint64):
        assert oracle.isqrt(int(v) * 2 + 1) == reference.isqrt(int(v) * 2 + 1)
    for v in rng.integers(0, I64_MAX, 2000, dtype=np.int64):
        assert oracle.fx_sqrt(int(v), 30, 30) == reference.fx_sqrt(int(v), 30, 30)


def test_vector_kernels_random(oracle, reference):
    rng = np.random.default_rng(99)
    for _ in range(200):
        n = int(rng.integers(1, 65))
        v = rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64)
        w = rng.integers(I64_MIN, I64_MAX, n, dtype=np.int64)
        b1, b2 = int(rng.integers(0, 30)), int(rng.integers(0, 30))
        t1, t2 = PyTrace(), PyTrace()
        assert oracle.fx_dot(v, w, 30, b1, b2, t1) == reference.fx_dot(v, w, 30, b1, b2, t2)
        assert t1.total == t2.total and t1.events == t2.events
        h = int(rng.integers(I64_MIN, I64_MAX))
        t1, t2 = PyTrace(), PyTrace()
        assert np.array_equal(oracle.fx_axpy_sub(w, h, v, 30, b1, t1), reference.fx_axpy_sub(w, h, v, 30, b1, t2))
        assert t1.events == t2.events
        u = rng.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
        nb1 = 16 + int(rng.integers(0, 14))
        assert oracle.fx_norm(u, 30, nb1) == reference.fx_norm(u, 30, nb1)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_16", "split_s3", "ilu_random"])
def test_operators_full_range(oracle, reference, name):
    co, cr = build_case(name, oracle), build_case(name, reference)
    for s in range(co["ncomp"]):
        t1, t2 = PyTrace(), PyTrace()
        assert np.array_equal(oracle.spmv(co["sp"], s, co["v_full"], t1), reference.spmv(cr["sp"], s, cr["v_full"], t2))
        assert t1.total == t2.total and t1.events == t2.events
    if co.get("ilu"):
        for y in (co["y_int"], co["v_full"]):
            t1, t2 = PyTrace(), PyTrace()
            assert np.array_equal(oracle.apply_inverse(co["il"], y, t1), reference.apply_inverse(cr["il"], y, t2))
            assert t1.total == t2.total and t1.events == t2.events


def test_overflow_trace_matches(oracle, reference):
    """test_refine.cpp:392-426: no dot guard shift -> wrap events (and maybe a throw)."""
    from workloads import gen
    rp, ci, v = gen.laplacian2d(8)
    res = []
    for B in (oracle, reference):
        A = B.csrf(rp, ci, v)
        vals, scale = B.row_scale(A, 16)
        af = B.csrf(rp, ci, vals)
        comp, al, _ = (B.build_split(af, 16, 10) if B.prefix == "ref_" else B.build_split(vals, 16, 10))
        sp = B.split(rp, ci, comp, al)
        b = np.ones(len(rp) - 1) / scale
        t = PyTrace(cap_events=1024)
        try:
            x, rep = B.solve(sp, af, b, 1e-8, 3, 6, 30, len(al) - 1, Shifts(0, 0, 16, 16, 16, 14, 16, 0), trace=t)
            out = ("ok", rep["overflow_total"])
        except CheckerError as e:
            out = ("err", e.code)
        res.append((out, t.total, t.events[:50]))
    assert res[0] == res[1]
    assert res[0][1] > 0
