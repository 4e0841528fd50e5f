"""GPU: the C++ drop-in adapter (integration/) with the reference's exact signatures, checked
bit-for-bit against the unmodified reference's dock_ligand / run_screening in one C++ process."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "integration", "_build", "adapter_test")


def test_cpp_adapter_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/adapter_test not built (make -C integration needs /root/reference)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER TEST PASSED" in r.stdout
