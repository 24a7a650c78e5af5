import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full configs[1] sizes)")


def _ensure_built():
    need = [os.path.join(REPO, "paper_1810_03099_b200", "lib", "librefsig_gpu.so"),
            os.path.join(REPO, "paper_1810_03099_b200", "lib", "libmrcgen.so"),
            os.path.join(REPO, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-j8", "all"], cwd=REPO, check=True, stdout=subprocess.DEVNULL)
    ref = os.path.join(REPO, "oracle", "_ref", "librefshim.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "ref"], cwd=REPO, check=True, stdout=subprocess.DEVNULL)


_ensure_built()


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(os.path.join(GOLDEN, "corpus_small.npz")))


@pytest.fixture(scope="session")
def golden_text():
    return dict(np.load(os.path.join(GOLDEN, "text_small.npz")))


@pytest.fixture(scope="session")
def spec_examples():
    import json
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_ctx_factory():
    # No skip: a gpu-marked test on a box without a usable device is a failure.
    import paper_1810_03099_b200 as R

    ctxs = []

    def make():
        c = R.Context(0)
        ctxs.append(c)
        return c

    yield make
    for c in ctxs:
        c.close()
