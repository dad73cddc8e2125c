"""Generate tests/golden/ref_goldens.json from the REFERENCE library itself.

Runs only in the build container, where oracle/_ref/libintgmres_ref.so has been
compiled from /root/reference (oracle/Makefile).  The committed JSON pins the
CPU restatement and the CUDA path on machines without the reference (the GPU
box).  Inputs come from workloads/gen.py (seeded SplitMix64), so every consumer
regenerates identical arrays.

    python tests/golden/make_goldens.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.ffi import PyTrace, Reference, Shifts  # noqa: E402
from tests.cases import CASES, build_case  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = Reference()
    out = {"_source": "reference library (oracle/_ref, built from /root/reference/proj/core) on the "
                      "inputs of tests/cases.py; regenerate with tests/golden/make_goldens.py",
           "cases": {}}
    for name in CASES:
        c = build_case(name, R)
        rec = {}
        sh = Shifts(*c["shifts"])
        if c.get("cycle"):
            cy = R.run_cycle(c["sp"], c["m"], 30, c["s"], sh, c["b"], np.zeros(c["n"]), precond=c.get("il"))
            rec["cycle"] = {"dim": cy["dim"], "r0_norm": cy["r0_norm"], "n_basis": cy["n_basis"],
                            "basis": h(cy["basis"]), "hess": h(cy["hess"]), "g": h(cy["g"]),
                            "cos_raw": h(cy["cos_raw"]), "sin_raw": h(cy["sin_raw"]), "x": h(cy["x"])}
        if c.get("solve"):
            tr = PyTrace()
            x, rep = R.solve(c["sp"], c["af"], c["b"], c["tol"], c["max_ref"], c["m"], 30, c["s"], sh,
                             checked=True, precond=c.get("il"), trace=tr)
            rep.pop("wall_time_sec")
            rec["solve"] = {"x": h(x), "report": rep, "trace_total": tr.total}
        if c.get("spmv"):
            rec["spmv"] = {str(s): h(R.spmv(c["sp"], s, c["v_full"])) for s in range(c["ncomp"])}
        if c.get("ilu_apply"):
            rec["apply_inverse"] = h(R.apply_inverse(c["il"], c["y_int"]))
            rec["apply_inverse_fp"] = h(R.apply_inverse_fp(c["il"], c["y_fp"]))
        if c.get("setup"):
            rec["setup"] = {"scaled": h(c["vals"]), "comp": h(c["comp"]), "alphas": c["alphas"]}
            if c.get("il") is not None:
                rec["setup"]["ilu"] = [h(a) for a in c["ilu_arrays"]]
        out["cases"][name] = rec
        print(name, "done", flush=True)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_goldens.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
