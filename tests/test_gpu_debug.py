"""The AUGSCHED_DEBUG build (device checks of the SURVEY §8(c).4 invariants:
sum of grants <= B, ledger non-negative and, in the simulator, inside the
capacity, the dynamic limit inside its clamp) runs parity workloads of every
path without a check firing (tools/debug_parity.py in a subprocess that
loads the debug library through AUGSCHED_LIB)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_build_parity_without_invariant_failures():
    from paper_2512_04013_b200 import _build
    lib = _build.build_debug()
    env = dict(os.environ, AUGSCHED_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_parity.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "debug parity ok" in r.stdout
