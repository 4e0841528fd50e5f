import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_npz(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    if "spec" in d:
        d["spec"] = json.loads(str(d["spec"]))
    return d


def load_json(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def have_reference_build():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgeodock_ref.so"))


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    if not have_reference_build():
        pytest.skip("oracle/_ref not built (make -C oracle ref needs /root/reference)")
    from oracle import Oracle
    return Oracle("reference")
