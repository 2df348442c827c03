"""The guard build (make guard -> libbpdec_guard.so, csrc/devmem.hpp): the
bounds-checking stand-in for compute-sanitizer.  Its self-test proves the
mechanism on the device (poisoned allocations, an out-of-bounds write caught,
no false positive); scripts/guard_tests.sh runs the GPU suites against it."""
import ctypes as C
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GUARD = os.path.join(ROOT, "paper_2507_03509_b200", "libbpdec_guard.so")


def test_guard_library_exports_selftest():
    if not os.path.exists(GUARD):
        pytest.skip("guard build not present (make guard)")
    lib = C.CDLL(GUARD)
    assert hasattr(lib, "bpdec_guard_selftest")
    assert hasattr(lib, "bpdec_decode_batch")


@pytest.mark.gpu
def test_guard_selftest_on_device():
    assert os.path.exists(GUARD), "make guard"
    code = ("import ctypes, sys; l = ctypes.CDLL(sys.argv[1]); rc = l.bpdec_guard_selftest(); "
            "print('selftest', rc); sys.exit(rc)")
    r = subprocess.run([sys.executable, "-c", code, GUARD], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
