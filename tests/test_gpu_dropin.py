"""The drop-in boundary end to end: the reference's own C++ types and CPU functions
(proj/src, unmodified) next to dash::b200 (include/dash_b200.hpp -> libdashcu.so)
in one binary, integration/dropin_test.cpp (built into oracle/_ref by
`make -C oracle dropin`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (reference sources absent)")
def test_reference_api_through_the_b200_library():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
