"""The C++ host API (include/refsig/gpu.hpp) on the SPEC known answers."""
import os
import subprocess

import pytest

from tests.conftest import REPO

pytestmark = pytest.mark.gpu


def test_cpp_api_check_binary():
    exe = os.path.join(REPO, "paper_1810_03099_b200", "lib", "refsig_gpu_cpp_check")
    assert os.path.exists(exe), "build the C++ check (make)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "gpu_api_check OK" in r.stdout
