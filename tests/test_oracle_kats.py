"""The CPU restatement (oracle/igm_oracle.c) against the reference's own
known-answer tests (tests/golden/kats.json, each value citing its source)."""
import math

import numpy as np
import pytest

from oracle.ffi import CheckerError, PyTrace, Shifts

F = 30


def raw(x):
    return int(round(x * (1 << F)))


def test_encode(oracle, kats):
    for k in kats["encode"]:
        assert oracle.encode(k["x"], k["f"]) == k["raw"], k["cite"]
    for k in kats["encode_overflow"]:
        x = float(k["x"])
        with pytest.raises(CheckerError) as e:
            oracle.encode(x, k["f"])
        assert e.value.code == 3, k["cite"]
    assert oracle.encode(float(2 ** 33 - 1), 30) == (2 ** 33 - 1) << 30  # test_fxp.cpp:45


def test_decode_roundtrip(oracle):
    rng = np.random.default_rng(11)
    for x in rng.uniform(-1000, 1000, 500):
        back = oracle.decode(oracle.encode(float(x), 30), 30)
        assert abs(back - x) < 2.0 ** -30  # test_fxp.cpp:52-62
    assert oracle.decode(oracle.encode(0.5, 30), 30) == 0.5
    assert oracle.decode(oracle.encode(-2.25, 30), 30) == -2.25


def test_fx_mul_div(oracle, kats):
    for k in kats["fx_mul"]:
        assert oracle.fx_mul(k["a"], k["b"], k["f"], k["b1"], k["b2"], k["out"]) == k["raw"], k["cite"]
    for k in kats["fx_mul_invalid"]:
        with pytest.raises(CheckerError) as e:
            oracle.fx_mul(k["a"], k["b"], k["f"], k["b1"], k["b2"], k["out"])
        assert e.value.code == 1, k["cite"]
    for k in kats["fx_div"]:
        assert oracle.fx_div(k["a"], k["b"], k["f"], k["b1"], k["b2"]) == k["raw"], k["cite"]
    for k in kats["fx_div_domain"]:
        with pytest.raises(CheckerError) as e:
            oracle.fx_div(k["a"], k["b"], k["f"], k["b1"], k["b2"])
        assert e.value.code == 2, k["cite"]


def test_isqrt_and_sqrt(oracle, kats):
    for v, r in kats["isqrt"]:
        assert oracle.isqrt(v) == r, kats["isqrt_cite"]
    for v in range(0, 70000, 7):  # test_fxp.cpp:117 (against math.isqrt here)
        assert oracle.isqrt(v) == math.isqrt(v)
    for k in kats["fx_sqrt"]:
        assert oracle.fx_sqrt(k["a"], k["fin"], k["out"]) == k["raw"], k["cite"]
    for k in kats["fx_sqrt_errors"]:
        with pytest.raises(CheckerError) as e:
            oracle.fx_sqrt(k["a"], k["fin"], k["out"])
        assert e.value.code == (2 if k["kind"] == "domain" else 1), k["cite"]


def test_vector_kats(oracle, kats):
    for k in kats["fx_dot"]:
        v = [raw(x) for x in k["v"]]
        w = [raw(x) for x in k["w"]]
        assert oracle.fx_dot(v, w, F, k["b1"], k["b2"]) == raw(k["value"]), k["cite"]
    for k in kats["fx_norm"]:
        assert oracle.fx_norm([raw(x) for x in k["v"]], F, k["b1"]) == raw(k["value"]), k["cite"]
    k = kats["fx_norm_wrap"]
    with pytest.raises(CheckerError) as e:
        oracle.fx_norm(k["raw"], F, k["b1"])
    assert e.value.code == 2
    k = kats["fx_axpy_sub"]
    w = oracle.fx_axpy_sub([raw(x) for x in k["w"]], raw(k["h"]), [raw(x) for x in k["v"]], F, k["b1"])
    assert [x / (1 << F) for x in w] == k["result"], k["cite"]


def test_checked_wrap(oracle, kats):
    k = kats["add_wrap"]
    t = PyTrace(checked=True)
    assert oracle.fx_add(k["a"], k["b"], t) == k["raw"]
    assert t.total == k["events"] and t.events[0][1] == "add"
    silent = PyTrace(checked=False)
    assert oracle.fx_add(k["a"], k["b"], silent) == k["raw"] and silent.total == 0


def test_shift_plans(oracle, kats):
    p = kats["shift_presets"]
    assert oracle.shifts_validate(Shifts(*p["unpreconditioned"]), 30) == 0
    assert oracle.shifts_validate(Shifts(*p["preconditioned"]), 30) == 0
    for k in kats["shift_invalid"]:
        assert oracle.shifts_validate(Shifts(*k["plan"]), k["f"]) == 1, k["cite"]
    for k in kats["shift_valid"]:
        assert oracle.shifts_validate(Shifts(*k["plan"]), k["f"]) == 0, k["cite"]


def test_setup_kats(oracle, kats):
    k = kats["row_scale"]
    a = oracle.csrf(k["row_ptr"], k["col_idx"], k["vals"])
    vals, scale = oracle.row_scale(a, k["alpha"])
    assert list(scale) == k["scale"] and list(vals) == k["scaled"], k["cite"]
    k = kats["build_split"]
    comp, al, ex = oracle.build_split(k["vals"], k["alpha"], k["max"])
    assert comp.tolist() == k["comps"] and al == k["alphas"] and ex == k["exact"], k["cite"]
    k = kats["split_cast"]
    lo, up = oracle.factorize_split_cast(oracle.csrf(k["row_ptr"], k["col_idx"], k["vals"]))
    assert lo[2].tolist() == k["lower"] and up[2].tolist() == k["upper"], k["cite"]
    assert lo[3].tolist() == k["diag_pos_lower"] and up[3].tolist() == k["diag_pos_upper"]


def test_givens_hessenberg_gamma(oracle, kats):
    import ctypes as C
    k = kats["solve_hessenberg"]
    r = np.array(k["r"])
    g = np.array(k["g"])
    y = np.zeros(k["dim"])
    fn = oracle.fn("solve_hessenberg")
    f64p = C.POINTER(C.c_double)
    assert fn(r.ctypes.data_as(f64p), k["ld"], k["dim"], g.ctypes.data_as(f64p), y.ctypes.data_as(f64p)) == 0
    assert y.tolist() == k["y"], k["cite"]
    k = kats["rotation"]
    col = np.array([raw(x) for x in k["col"]], dtype=np.int64)
    c = np.array([raw(k["c"])], dtype=np.int64)
    s = np.array([raw(k["s"])], dtype=np.int64)
    i64p = C.POINTER(C.c_int64)
    assert oracle.fn("apply_stored_rotations")(col.ctypes.data_as(i64p), 1, c.ctypes.data_as(i64p),
                                               s.ctypes.data_as(i64p), k["givens_b2"], F, None) == 0
    assert [x / (1 << F) for x in col] == k["result"], k["cite"]
    k = kats["gamma_scale"]
    rr = np.array(k["r"])
    bk = np.zeros(3)
    gm = C.c_double()
    assert oracle.fn("gamma_scale")(C.c_int64(3), rr.ctypes.data_as(f64p), C.byref(gm), bk.ctypes.data_as(f64p)) == 0
    assert gm.value == k["gamma"] and bk.tolist() == k["b_k"], k["cite"]


def test_cyclic_permutation_happy_breakdown(oracle):
    """test_gmres_cycle.cpp:167-190: A e_j = e_{j+1 mod n}, exact in fixed point."""
    n = 8
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.array([(i - 1) % n for i in range(n)], dtype=np.int32)  # row i has A[i, i-1] = 1
    comp, al, ex = oracle.build_split(np.ones(n), 16, 2)
    sp = oracle.split(rp, ci, comp, al)
    b = np.zeros(n)
    b[0] = 1.0
    out = oracle.run_cycle(sp, n + 4, 30, 0, Shifts(16, 0, 16, 16, 16, 14, 16, 0), b, np.zeros(n))
    assert out["dim"] == n and out["n_basis"] == n


def test_zero_rhs(oracle):
    """test_gmres_cycle.cpp:192-204 / test_refine.cpp:372-380."""
    from workloads import gen
    rp, ci, v = gen.laplacian2d(3)
    comp, al, _ = oracle.build_split(v, 16, 4)
    sp = oracle.split(rp, ci, comp, al)
    out = oracle.run_cycle(sp, 5, 30, 0, Shifts(16, 0, 16, 16, 16, 14, 16, 0), np.zeros(9), np.zeros(9))
    assert out["dim"] == 0 and out["r0_norm"] == 0.0 and not out["x"].any()
