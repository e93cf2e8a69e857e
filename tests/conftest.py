import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference compiled in place)")


def pytest_collection_modifyitems(config, items):
    from oracle_ffi import ref_available
    skip_ref = pytest.mark.skip(reason="oracle/_ref not built (reference sources absent)")
    for it in items:
        if "ref" in it.keywords and not ref_available():
            it.add_marker(skip_ref)


@pytest.fixture
def knob():
    """Set a libdashcu kernel-variant knob for one test (dashcu_set_knob); restored after."""
    import paper_2505_17218_b200 as D
    touched = []

    def set_(name, value):
        touched.append(name)
        D.set_knob(name, value)
    yield set_
    for name in touched:
        D.set_knob(name, None)
