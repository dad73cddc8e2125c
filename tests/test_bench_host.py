"""Host-side legs of bench.py that run without a GPU: the reference arm
(`--impl reference`), which times the reference library / the oracle port on
the box's host cores (N = 1: config 2; N > 1: config 4, the partitioned arm's
workload).  Small grids here; the JSON contract is what is checked."""
import argparse
import io
import json
import contextlib

import pytest


def _line(fn, *a):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert fn(*a) == 0
    return json.loads(buf.getvalue().strip().splitlines()[-1])


def test_reference_arm_config2_contract():
    import bench
    args = argparse.Namespace(gpus=1, steps=1, warmup=0, grid=12, cfg4_grid=10)
    d = _line(bench.run_reference, args, 1, 0)
    assert d["impl"] == "reference" and d["metric"] == "int-GMRES iters/s" and d["unit"] == "iters/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "cfg2" in d["config"]["workload"]


def test_reference_arm_multi_gpu_runs_config4_on_rank0_only():
    import bench
    args = argparse.Namespace(gpus=2, steps=1, warmup=0, grid=12, cfg4_grid=10)
    d = _line(bench.run_reference, args, 2, 0)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert "cfg4" in d["config"]["workload"] and d["value"] > 0
    # the other ranks exit 0 without work and without a line
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert bench.run_reference(args, 2, 1) == 0
    assert buf.getvalue() == ""
