"""The C-ABI library loads and exports every symbol include/refsig_gpu.h
declares; the product fails loudly without a device. CPU only (no compute)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1810_03099_b200 as R
from tests.conftest import REPO, have_gpu


def declared(header):
    src = open(os.path.join(REPO, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(refsig_gpu_\w+|mrcgen_\w+)\s*\(", src)))


def test_gpu_library_exports_header_symbols():
    lib = ctypes.CDLL(R.library_path())
    names = declared("refsig_gpu.h")
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # the Python binding declares a signature for every exported entry point
    assert sorted(R.SIGNATURES) == names


def test_generator_library_exports_header_symbols():
    lib = ctypes.CDLL(os.path.join(REPO, "paper_1810_03099_b200", "lib", "libmrcgen.so"))
    for n in declared("mrcgen.h"):
        assert hasattr(lib, n), n


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.skipif(have_gpu(), reason="checks the no-device behaviour")
def test_no_device_fails_loudly():
    with pytest.raises(R.RefsigRuntimeError):
        R.Context(0)


def test_version_string():
    lib = R.load_library()
    assert b"sm_100a" in lib.refsig_gpu_version()
