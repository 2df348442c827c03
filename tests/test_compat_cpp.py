"""The reference-shaped C++ host layer (include/bpdec/etdec_compat.hpp) built
against libbpdec.so and run as a standalone program."""
import os
import subprocess

import pytest

from conftest import ROOT


def _build():
    subprocess.run(["make", "-s", "-C", ROOT, "compat_test"], check=True)
    return os.path.join(ROOT, "build", "compat_test")


def test_compat_host():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only variant (expects no GPU)")
    r = subprocess.run([_build()], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_compat_gpu():
    r = subprocess.run([_build(), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compat_test (gpu) OK" in r.stdout
