"""The reference's own C++ call sites on the B200 path (GPU).

tests/cpp/dropin_test.cpp ports proj/tests/test_accelerated.cpp:131-186, :223-244
and acceptance criteria 1-2 (proj/tests/acceptance.cpp:70-131) with only the
solver calls swapped for include/dlb_dolb.hpp (dlb_dolb::collide_and_stream,
dlb_dolb::build_device_run / DeviceRun). It is compiled by build() against the
unmodified reference headers and objects plus libdlb_b200.so, in the build
container (the reference tree is not on the GPU box), and shipped as a binary.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin_test")


def test_reference_call_sites_on_device():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} is not built: run build() where /root/reference is present")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in checks passed" in r.stdout
    for line in ("criterion 1", "criterion 2", "golden_dump", "hybrid", "dispatch_error"):
        assert line in r.stdout
