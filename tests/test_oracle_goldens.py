"""The CPU restatement against golden outputs of the REFERENCE library
(tests/golden/ref_goldens.json, made by tests/golden/make_goldens.py)."""
import hashlib

import numpy as np
import pytest

from oracle.ffi import PyTrace, Shifts
from tests.cases import CASES, build_case


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(CASES))
def test_case_against_reference_goldens(oracle, goldens, name):
    g = goldens["cases"][name]
    c = build_case(name, oracle)
    sh = Shifts(*c["shifts"])
    if "setup" in g:
        assert h(c["vals"]) == g["setup"]["scaled"]
        assert h(c["comp"]) == g["setup"]["comp"] and c["alphas"] == g["setup"]["alphas"]
        if "ilu" in g["setup"]:
            assert [h(a) for a in c["ilu_arrays"]] == g["setup"]["ilu"]
    if "spmv" in g:
        for s, hv in g["spmv"].items():
            assert h(oracle.spmv(c["sp"], int(s), c["v_full"])) == hv
    if "apply_inverse" in g:
        assert h(oracle.apply_inverse(c["il"], c["y_int"])) == g["apply_inverse"]
        assert h(oracle.apply_inverse_fp(c["il"], c["y_fp"])) == g["apply_inverse_fp"]
    if "cycle" in g:
        cy = oracle.run_cycle(c["sp"], c["m"], 30, c["s"], sh, c["b"], np.zeros(c["n"]), precond=c.get("il"))
        for k in ("dim", "r0_norm", "n_basis"):
            assert cy[k] == g["cycle"][k], k
        for k in ("basis", "hess", "g", "cos_raw", "sin_raw", "x"):
            assert h(cy[k]) == g["cycle"][k], k
    if "solve" in g:
        tr = PyTrace()
        x, rep = oracle.solve(c["sp"], c["af"], c["b"], c["tol"], c["max_ref"], c["m"], 30, c["s"], sh,
                              precond=c.get("il"), trace=tr)
        rep.pop("wall_time_sec")
        assert rep == g["solve"]["report"]
        assert h(x) == g["solve"]["x"]
        assert tr.total == g["solve"]["trace_total"]
