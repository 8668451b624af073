import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The package refuses to import without its library (no CPU fallback exists), and the
# built .so is not in git: build it once if this checkout has none yet (nvcc
# cross-compiles sm_100a without a GPU).
if not os.path.exists(os.path.join(ROOT, "paper_2510_12872_b200", "lib", "libkvcomm.so")):
    import importlib.util
    _spec = importlib.util.spec_from_file_location("_kvcomm_build",
                                                   os.path.join(ROOT, "paper_2510_12872_b200", "build.py"))
    _mod = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(_mod)
    _mod.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
