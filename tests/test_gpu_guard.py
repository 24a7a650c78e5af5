"""Out-of-bounds-write guard over every kernel (tools/sanitize_run.py under
REFSIG_CANARY=1: a 4 KB guard region past every device buffer, checked by
refsig_gpu_debug_check). compute-sanitizer is closed on the GPU pool; this
is the in-tree substitute for its memcheck of writes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_within_its_buffers():
    env = dict(os.environ, REFSIG_CANARY="1")
    r = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sanitize run done" in r.stdout
