"""compute-sanitizer memcheck, racecheck and synccheck over small invocations
of every kernel (tools/sanitize_driver.py, which also checks each result
against the oracle): no error may be reported."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([CS, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_driver.py")], cwd=ROOT, capture_output=True,
                       text=True, timeout=1500)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "compute-sanitizer is closed" in out:
        # the GPU pool's wrapper refuses sanitizer runs (they have left GPUs
        # needing a reset); the clean runs are recorded in profiles/r2_sanitize_summary.txt
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out
