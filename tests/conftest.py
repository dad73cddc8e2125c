import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import ffi
    ffi.ensure_built()
    return ffi.Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import ffi
    if not ffi.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return ffi.Reference()


@pytest.fixture(scope="session")
def goldens():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "ref_goldens.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kats():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def product_lib():
    so = os.path.join(ROOT, "paper_2009_07495_b200", "libigm_b200.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-C", ROOT, "paper_2009_07495_b200/libigm_b200.so"], check=True)
    import paper_2009_07495_b200 as igm
    return igm.lib()


@pytest.fixture(scope="session")
def igm(product_lib):
    import paper_2009_07495_b200 as igm
    return igm
